// TEST INFRASTRUCTURE — oracle only.  Never linked into the product.
//
// A flat C wrapper over the UNMODIFIED reference library (built from
// /root/reference/proj/src with -Dvoxelkit=vkref by oracle/Makefile into
// oracle/_ref/libvkref.so) so tests, golden-fixture generation and bench.py's
// CPU baseline can call the reference's own code through ctypes.  Every
// function forwards to the reference API it names:
//   vkref_richardson_lucy -> deconv::richardson_lucy  (proj/src/deconv.cpp:304-431)
//   vkref_rl_step         -> deconv::rl_step (dispatch) (proj/src/deconv.cpp:196-200)
//   vkref_fft_convolve    -> filters::fft_convolve       (proj/src/filters.cpp:175-264)
//   vkref_gaussian_psf    -> synth::gaussian_psf         (proj/src/synth.cpp:226-258)
//   vkref_generate_blobs  -> synth::generate_blobs       (proj/src/synth.cpp:199-224)
//   vkref_si_psnr         -> metrics::si_psnr            (proj/src/metrics.cpp:67-101)
//   vkref_good_size       -> fftx::good_size             (proj/src/fft_plan.cpp:41-49)
//   vkref_single_image_frc-> metrics::single_image_frc   (proj/src/metrics.cpp:241-264)
//   vkref_ssim            -> metrics::ssim (as shipped)  (proj/src/metrics.cpp:103-144)
//   vkref_gaussian        -> filters::gaussian           (proj/src/filters.cpp:78-140)
//   vkref_write_volume    -> io::write_volume (f32 / u16)  (proj/src/io.cpp:53-81)
//   vkref_read_volume     -> io::read_volume              (proj/src/io.cpp:83-158)
// Exceptions are mapped to the same status codes the product C-ABI uses
// (include/vk_rl.h) so error-parity tests compare like with like.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "voxelkit/deconv.hpp"
#include "voxelkit/errors.hpp"
#include "voxelkit/filters.hpp"
#include "voxelkit/image.hpp"
#include "voxelkit/io.hpp"
#include "voxelkit/metrics.hpp"
#include "voxelkit/synth.hpp"
#include "fft_plan.hpp"

using namespace voxelkit;

namespace {

enum {
  OK = 0,
  E_ARG = 1,
  E_SHAPE = 2,
  E_NEGATIVE = 3,
  E_UNNORMALIZED = 4,
  E_DEGENERATE = 5,
  E_TOO_SMALL = 6,
  E_ODD = 7,
  E_KERNEL_TOO_LARGE = 11,
  E_BAD_MAGIC = 12,
  E_HEADER_MISMATCH = 13,
  E_TRUNCATED = 14,
  E_PLACEMENT = 15,
  E_EVEN_EXTENT = 16,
  E_OTHER = 99,
};

Shape to_shape(int rank, const std::uint64_t* s) {
  Shape out(rank);
  for (int i = 0; i < rank; ++i) out[i] = static_cast<std::size_t>(s[i]);
  return out;
}

NdImage make(int rank, const std::uint64_t* s, const float* v, bool accel) {
  Shape sh = to_shape(rank, s);
  std::vector<float> data(v, v + shape_volume(sh));
  NdImage img = NdImage::f32(sh, std::move(data));
  return accel ? img.with_backend(BackendId::accelerated) : img;
}

int fail(const std::exception& e, int code, char* err, int errlen) {
  if (err && errlen > 0) {
    std::strncpy(err, e.what(), static_cast<std::size_t>(errlen - 1));
    err[errlen - 1] = 0;
  }
  return code;
}

#define VKREF_CATCH                                                        \
  catch (const ShapeMismatch& e) { return fail(e, E_SHAPE, err, errlen); } \
  catch (const NegativeInput& e) { return fail(e, E_NEGATIVE, err, errlen); } \
  catch (const UnnormalizedPsf& e) { return fail(e, E_UNNORMALIZED, err, errlen); } \
  catch (const DegenerateReference& e) { return fail(e, E_DEGENERATE, err, errlen); } \
  catch (const TooSmall& e) { return fail(e, E_TOO_SMALL, err, errlen); } \
  catch (const OddExtent& e) { return fail(e, E_ODD, err, errlen); }       \
  catch (const KernelTooLarge& e) { return fail(e, E_KERNEL_TOO_LARGE, err, errlen); } \
  catch (const BadMagic& e) { return fail(e, E_BAD_MAGIC, err, errlen); } \
  catch (const HeaderMismatch& e) { return fail(e, E_HEADER_MISMATCH, err, errlen); } \
  catch (const TruncatedPayload& e) { return fail(e, E_TRUNCATED, err, errlen); } \
  catch (const PlacementFailure& e) { return fail(e, E_PLACEMENT, err, errlen); } \
  catch (const EvenExtent& e) { return fail(e, E_EVEN_EXTENT, err, errlen); } \
  catch (const Error& e) { return fail(e, E_ARG, err, errlen); }           \
  catch (const std::exception& e) { return fail(e, E_OTHER, err, errlen); }

}  // namespace

extern "C" {

std::uint64_t vkref_good_size(std::uint64_t n) { return fftx::good_size(n); }

int vkref_richardson_lucy(int rank, const std::uint64_t* shape, const float* observed,
                          int psf_rank, const std::uint64_t* psf_shape, const float* psf, int metric,
                          double rel_tol, int patience, int max_iters, int flat_init,
                          int accelerated, float* estimate_out, double* metric_values,
                          double* wall_s, double* loglik, int* iters_run, int* stop_reason,
                          std::uint64_t* fft_shape, char* err, int errlen) {
  try {
    NdImage obs = make(rank, shape, observed, accelerated != 0);
    NdImage k = make(psf_rank, psf_shape, psf, false);
    deconv::StoppingRule rule;
    rule.metric = static_cast<deconv::StopMetric>(metric);
    rule.rel_tol = rel_tol;
    rule.patience = patience;
    rule.max_iters = max_iters;
    deconv::RlResult r = deconv::richardson_lucy(obs, k, rule, flat_init != 0);
    const auto ev = r.estimate.f32_values();
    std::memcpy(estimate_out, ev.data(), ev.size() * sizeof(float));
    const int n = static_cast<int>(r.trace.records.size());
    for (int i = 0; i < n; ++i) {
      if (metric_values) metric_values[i] = r.trace.records[i].value;
      if (wall_s) wall_s[i] = r.trace.records[i].wall_time_s;
      if (loglik) loglik[i] = r.trace.log_likelihood[i];
    }
    *iters_run = n;
    *stop_reason = r.trace.stop_reason == "converged" ? 1 : 0;
    for (int a = 0; a < rank; ++a) fft_shape[a] = r.trace.fft_shape[a];
    return OK;
  }
  VKREF_CATCH
}

int vkref_rl_step(int rank, const std::uint64_t* shape, const float* estimate,
                  const float* observed, const std::uint64_t* psf_shape, const float* psf,
                  int accelerated, float* out, char* err, int errlen) {
  try {
    NdImage e = make(rank, shape, estimate, accelerated != 0);
    NdImage o = make(rank, shape, observed, accelerated != 0);
    NdImage k = make(rank, psf_shape, psf, accelerated != 0);
    NdImage r = deconv::rl_step(e, o, k);
    const auto v = r.f32_values();
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return OK;
  }
  VKREF_CATCH
}

int vkref_fft_convolve(int rank, const std::uint64_t* shape, const float* img,
                       const std::uint64_t* kshape, const float* kernel, int circular,
                       float* out, char* err, int errlen) {
  try {
    NdImage a = make(rank, shape, img, false);
    NdImage k = make(rank, kshape, kernel, false);
    NdImage r = filters::fft_convolve(a, k, circular != 0);
    const auto v = r.f32_values();
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return OK;
  }
  VKREF_CATCH
}

int vkref_gaussian_psf(int rank, const std::uint64_t* shape, const double* sigmas, int nsig,
                       float* out, char* err, int errlen) {
  try {
    std::vector<double> s(sigmas, sigmas + nsig);
    NdImage r = synth::gaussian_psf(to_shape(rank, shape), s);
    const auto v = r.f32_values();
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return OK;
  }
  VKREF_CATCH
}

int vkref_generate_blobs(const std::uint64_t* shape3, std::uint64_t n_objects, double rmin,
                         double rmax, std::uint64_t seed, double noise, float* out, char* err,
                         int errlen) {
  try {
    synth::SynthSpec spec;
    spec.shape = to_shape(3, shape3);
    spec.n_objects = n_objects;
    spec.radius_min = rmin;
    spec.radius_max = rmax;
    spec.seed = seed;
    spec.noise_sigma = noise;
    synth::BlobVolume b = synth::generate_blobs(spec);
    const auto v = b.intensity.f32_values();
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return OK;
  }
  VKREF_CATCH
}

int vkref_si_psnr(int rank, const std::uint64_t* shape, const float* x, const float* ref,
                  double* value, char* err, int errlen) {
  try {
    *value = metrics::si_psnr(make(rank, shape, x, false), make(rank, shape, ref, false));
    return OK;
  }
  VKREF_CATCH
}

int vkref_single_image_frc(int rank, const std::uint64_t* shape, const float* x,
                           double spacing, double* value, char* err, int errlen) {
  try {
    *value = metrics::single_image_frc(make(rank, shape, x, false), spacing);
    return OK;
  }
  VKREF_CATCH
}

// metrics::ssim as shipped (proj/src/metrics.cpp:103-144).  It reads the
// smoothed moments through spans of destroyed temporaries (:128-132), so the
// value is only trustworthy while the allocator has not reused those blocks;
// callers cross-check it against vkref_gaussian-based recomputation.
int vkref_ssim(int rank, const std::uint64_t* shape, const float* x, const float* ref,
               double* value, char* err, int errlen) {
  try {
    *value = metrics::ssim(make(rank, shape, x, false), make(rank, shape, ref, false));
    return OK;
  }
  VKREF_CATCH
}

// filters::gaussian (proj/src/filters.cpp:78-140), sigma per axis.
int vkref_gaussian(int rank, const std::uint64_t* shape, const float* x, double sigma,
                   double truncate, float* out, char* err, int errlen) {
  try {
    const NdImage g = filters::gaussian(make(rank, shape, x, false),
                                        std::vector<double>(rank, sigma), truncate);
    const auto v = g.f32_values();
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return OK;
  }
  VKREF_CATCH
}

#ifdef VKREF_HAVE_IO
// elem 0 = f32, 1 = u16, 2 = u32, 3 = bool; spacing may be NULL.
int vkref_write_volume(const char* path, int elem, int rank, const std::uint64_t* shape,
                       const void* data, const double* spacing, char* err, int errlen) {
  try {
    const Shape sh = to_shape(rank, shape);
    const std::size_t n = shape_volume(sh);
    NdImage img;
    if (elem == 0) {
      const float* p = static_cast<const float*>(data);
      img = NdImage::f32(sh, std::vector<float>(p, p + n));
    } else if (elem == 1) {
      const std::uint16_t* p = static_cast<const std::uint16_t*>(data);
      img = NdImage::u16(sh, std::vector<std::uint16_t>(p, p + n));
    } else if (elem == 2) {
      const std::uint32_t* p = static_cast<const std::uint32_t*>(data);
      img = NdImage::labels(sh, std::vector<std::uint32_t>(p, p + n));
    } else {
      const std::uint8_t* p = static_cast<const std::uint8_t*>(data);
      img = NdImage::boolean(sh, std::vector<std::uint8_t>(p, p + n));
    }
    if (spacing) img = img.with_spacing(std::vector<double>(spacing, spacing + rank));
    io::write_volume(path, img);
    return OK;
  }
  VKREF_CATCH
}

// Reads into f32 (as_f32); shape/rank/elem/spacing reported.
int vkref_read_volume(const char* path, int* elem, int* rank, std::uint64_t* shape, int* has_spacing,
                      double* spacing, float* out, std::uint64_t out_cap, char* err, int errlen) {
  try {
    const NdImage img = io::read_volume(path);
    *elem = img.elem() == Elem::f32 ? 0 : img.elem() == Elem::u16 ? 1 : img.elem() == Elem::u32_label ? 2 : 3;
    *rank = static_cast<int>(img.rank());
    for (std::size_t a = 0; a < img.rank() && a < 4; ++a) shape[a] = img.shape()[a];
    *has_spacing = img.spacing() ? 1 : 0;
    if (img.spacing())
      for (std::size_t a = 0; a < img.rank() && a < 4; ++a) spacing[a] = (*img.spacing())[a];
    if (out) {
      const auto v = img.as_f32().f32_values();
      std::memcpy(out, v.data(), std::min<std::uint64_t>(out_cap, v.size()) * sizeof(float));
    }
    return OK;
  }
  VKREF_CATCH
}
#endif

}  // extern "C"
