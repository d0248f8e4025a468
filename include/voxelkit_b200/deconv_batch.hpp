// Batch extension of the reference's deconvolution API.
//
// richardson_lucy_batch(observed[], psf, rule, flat_init) returns exactly what
// calling voxelkit::deconv::richardson_lucy (deconv.hpp:97-103) on each
// volume in order would return, and throws what that loop would throw first.
// Same-shape volumes share one plan (one pair of OTFs) and run on its
// concurrent batch lanes (vk_rl_run_batch); the BASELINE batch configs (C3:
// 64 volumes, C5: 4096 fields) go through this call.  Implemented in
// paper_2510_14143_b200/host/deconv_b200.cpp.
#pragma once

#include <vector>

#include "voxelkit/deconv.hpp"
#include "voxelkit/image.hpp"

namespace voxelkit::deconv {

std::vector<RlResult> richardson_lucy_batch(const std::vector<NdImage>& observed, const NdImage& psf,
                                            const StoppingRule& rule = {}, bool flat_init = false);

}  // namespace voxelkit::deconv
