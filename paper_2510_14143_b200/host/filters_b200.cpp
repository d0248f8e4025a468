// Registry binding of filters::fft_convolve on the B200 path.
//
// The reference registers "fft_convolve" for both backend tags
// (src/filters.cpp:316-323) over fft_convolve_impl (:174-264, an FFTW
// r2c/c2r in double).  register_filter_ops_b200 (called by the drop-in's
// register_deconv_ops, which the registry runs after register_filter_ops,
// registry.cpp:87-93) replaces both entries with vk_fft_convolve: linear mode
// on good_size(A + K - 1) with the centred crop, circular mode on the image
// grid (any extent: 5-smooth grids directly, others as the periodic
// extension through the linear path).  filters::fft_convolve and every other
// caller (the CLI's blur, tools/voxelkit_main.cpp:424) then run on the GPU
// unchanged.  Errors keep the reference's types and messages: ShapeMismatch
// on rank mismatch, KernelTooLarge in circular mode.
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "voxelkit/errors.hpp"
#include "voxelkit/image.hpp"
#include "voxelkit/registry.hpp"
#include "vk_rl.h"

namespace voxelkit::detail {

namespace {

int conv_device() {
  const char* e = std::getenv("VOXELKIT_DEVICE");
  return e ? std::atoi(e) : 0;
}

std::string strip(const char* msg, const char* name) {
  const std::string m = msg ? msg : "";
  const std::string p = std::string(name) + ": ";
  return m.rfind(p, 0) == 0 ? m.substr(p.size()) : m;
}

NdImage gpu_fft_convolve(const NdImage& img, const NdImage& kernel, bool circular) {
  if (img.rank() != kernel.rank()) throw ShapeMismatch("fft_convolve: rank mismatch");  // filters.cpp:176-177
  const NdImage a = img.as_f32();
  const NdImage k = kernel.as_f32();
  const std::vector<std::uint64_t> sh(a.shape().begin(), a.shape().end()), ks(k.shape().begin(), k.shape().end());
  std::vector<float> out(a.size());
  const vk_status st = vk_fft_convolve(conv_device(), static_cast<int>(sh.size()), sh.data(), a.f32_values().data(),
                                       static_cast<int>(ks.size()), ks.data(), k.f32_values().data(),
                                       circular ? 1 : 0, out.data());
  if (st == VK_ERR_SHAPE) throw ShapeMismatch(strip(vk_last_error(), "ShapeMismatch"));
  if (st == VK_ERR_KERNEL_TOO_LARGE) throw KernelTooLarge(strip(vk_last_error(), "KernelTooLarge"));
  if (st != VK_OK) throw Error(vk_last_error());
  return NdImage::f32_like(a, std::move(out));
}

}  // namespace

void register_filter_ops_b200(ExecutionRegistry& reg) {
  using ConvSig = NdImage(const NdImage&, const NdImage&, bool);
  reg.add<ConvSig>("fft_convolve", BackendId::reference, gpu_fft_convolve);
  reg.add<ConvSig>("fft_convolve", BackendId::accelerated, gpu_fft_convolve);
}

}  // namespace voxelkit::detail
