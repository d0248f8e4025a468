// TEST INFRASTRUCTURE — the C++ drop-in (voxelkit::deconv on the B200, via
// paper_2510_14143_b200/host/deconv_b200.cpp + libvkrl.so) against the
// unmodified reference (vkref::, via oracle/ref_capi.cpp) in one process, on
// identical inputs.  Exit code 0 iff every check passes.  Run by
// tests/test_dropin.py (-m gpu).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "voxelkit/core_ops.hpp"
#include "voxelkit/deconv.hpp"
#include "voxelkit/errors.hpp"
#include "voxelkit/filters.hpp"
#include "voxelkit/image.hpp"
#include "voxelkit/io.hpp"
#include "voxelkit/synth.hpp"
#include "voxelkit_b200/deconv_batch.hpp"
#include <fstream>
#include <iterator>

extern "C" {
int vkref_richardson_lucy(int rank, const std::uint64_t* shape, const float* observed, int psf_rank,
                          const std::uint64_t* psf_shape, const float* psf, int metric, double rel_tol,
                          int patience, int max_iters, int flat_init, int accelerated, float* estimate_out,
                          double* metric_values, double* wall_s, double* loglik, int* iters_run, int* stop_reason,
                          std::uint64_t* fft_shape, char* err, int errlen);
int vkref_rl_step(int rank, const std::uint64_t* shape, const float* estimate, const float* observed,
                  const std::uint64_t* psf_shape, const float* psf, int accelerated, float* out, char* err,
                  int errlen);
int vkref_fft_convolve(int rank, const std::uint64_t* shape, const float* img, const std::uint64_t* kshape,
                       const float* kernel, int circular, float* out, char* err, int errlen);
int vkref_write_volume(const char* path, int elem, int rank, const std::uint64_t* shape, const void* data,
                       const double* spacing, char* err, int errlen) __attribute__((weak));
}

using namespace voxelkit;

namespace {

int failures = 0;

void report(bool ok, const std::string& name, const std::string& detail = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : ": ", detail.c_str());
  if (!ok) ++failures;
}

double rel_l2(std::span<const float> a, std::span<const float> b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double d = (double)a[i] - (double)b[i];
    num += d * d;
    den += (double)b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

struct RefRun {
  int rc = 0;
  std::string err;
  std::vector<float> est;
  std::vector<double> metric, ll;
  int iters = 0, reason = 0;
  std::vector<std::uint64_t> fft;
};

RefRun ref_rl(const NdImage& obs, const NdImage& psf, const deconv::StoppingRule& r, bool flat) {
  RefRun out;
  const NdImage o = obs.as_f32(), k = psf.as_f32();
  std::vector<std::uint64_t> s(o.shape().begin(), o.shape().end()), ks(k.shape().begin(), k.shape().end());
  const int cap = std::max(r.max_iters, 1);
  out.est.resize(o.size());
  out.metric.resize(cap);
  out.ll.resize(cap);
  std::vector<double> wall(cap);
  out.fft.resize(s.size());
  char err[512] = {0};
  out.rc = vkref_richardson_lucy((int)s.size(), s.data(), o.f32_values().data(), (int)ks.size(), ks.data(),
                                 k.f32_values().data(), (int)r.metric, r.rel_tol, r.patience, r.max_iters, flat, 0,
                                 out.est.data(), out.metric.data(), wall.data(), out.ll.data(), &out.iters,
                                 &out.reason, out.fft.data(), err, 512);
  out.err = err;
  return out;
}

NdImage blurred_blobs(const Shape& shape, std::size_t n, std::uint64_t seed, const NdImage& psf) {
  synth::SynthSpec spec;
  spec.shape = shape;
  spec.n_objects = n;
  spec.radius_min = 3;
  spec.radius_max = 5;
  spec.seed = seed;
  const NdImage truth = synth::generate_blobs(spec).intensity;
  return vmax(filters::fft_convolve(truth, psf, false), 0.0f);  // tools/voxelkit_main.cpp:424
}

void compare_rl(const std::string& name, const NdImage& obs, const NdImage& psf, int iters, bool flat) {
  deconv::StoppingRule rule{deconv::StopMetric::si_psnr_vs_input, 1e-300, iters, iters};
  deconv::StoppingRule one{deconv::StopMetric::si_psnr_vs_input, 1e-300, 1, 1};
  const RefRun r1 = ref_rl(obs, psf, one, flat);
  const RefRun rn = ref_rl(obs, psf, rule, flat);
  const deconv::RlResult g1 = deconv::richardson_lucy(obs, psf, one, flat);
  const deconv::RlResult gn = deconv::richardson_lucy(obs, psf, rule, flat);
  const double e1 = rel_l2(g1.estimate.f32_values(), r1.est), en = rel_l2(gn.estimate.f32_values(), rn.est);
  char buf[256];
  std::snprintf(buf, sizeof buf, "relL2 iter1 %.2e, iter%d %.2e", e1, iters, en);
  report(r1.rc == 0 && rn.rc == 0 && e1 <= 1e-4 && en <= 1e-3, name + " estimate", buf);
  bool shape_ok = gn.trace.fft_shape.size() == rn.fft.size();
  for (std::size_t a = 0; shape_ok && a < rn.fft.size(); ++a) shape_ok = gn.trace.fft_shape[a] == rn.fft[a];
  report(shape_ok, name + " trace.fft_shape");
  bool trace_ok = (int)gn.trace.records.size() == rn.iters && gn.trace.stop_reason == (rn.reason ? "converged" : "max_iters");
  for (int i = 0; trace_ok && i < rn.iters; ++i) {
    trace_ok = gn.trace.records[i].iter == i + 1 && gn.trace.records[i].metric_name == "si_psnr_vs_input" &&
               std::abs(gn.trace.records[i].value - rn.metric[i]) <= 1e-3 * std::abs(rn.metric[i]) &&
               std::abs(gn.trace.log_likelihood[i] - rn.ll[i]) <= 1e-5 * std::abs(rn.ll[i]) &&
               gn.trace.records[i].wall_time_s > 0;
  }
  report(trace_ok, name + " trace records / log_likelihood / stop_reason");
  report(gn.estimate.shape() == obs.shape() && gn.estimate.backend() == obs.backend(), name + " result metadata");
}

// The reference's DEFAULT rule (frc_resolution) end to end: trace values
// (resolution, inf = unresolved), iterations and stop reason.
void compare_default_rule(const std::string& name, const NdImage& obs, const NdImage& psf, int max_iters) {
  deconv::StoppingRule rule;  // {frc_resolution, 1e-3, 3, 100}
  rule.max_iters = max_iters;
  const RefRun rn = ref_rl(obs, psf, rule, false);
  const deconv::RlResult gn = deconv::richardson_lucy(obs, psf, rule, false);
  bool ok = rn.rc == 0 && (int)gn.trace.records.size() == rn.iters &&
            gn.trace.stop_reason == (rn.reason ? "converged" : "max_iters");
  for (int i = 0; ok && i < rn.iters; ++i) {
    const double a = gn.trace.records[i].value, b = rn.metric[i];
    ok = gn.trace.records[i].metric_name == "frc_resolution" &&
         (std::isinf(b) ? std::isinf(a) : std::abs(a - b) <= 1e-3 * std::abs(b));
  }
  char buf[128];
  std::snprintf(buf, sizeof buf, "%d vs %d iterations, relL2 %.2e", (int)gn.trace.records.size(), rn.iters,
                rel_l2(gn.estimate.f32_values(), rn.est));
  report(ok && rel_l2(gn.estimate.f32_values(), rn.est) <= 1e-3, name + " default rule (frc)", buf);
}

template <class Exc>
void expect_error(const std::string& name, const NdImage& obs, const NdImage& psf, deconv::StoppingRule rule) {
  const RefRun r = ref_rl(obs, psf, rule, false);
  try {
    deconv::richardson_lucy(obs, psf, rule, false);
    report(false, name, "no exception");
  } catch (const Exc& e) {
    report(std::string(e.what()) == r.err, name, std::string(e.what()) + " | ref: " + r.err);
  } catch (const std::exception& e) {
    report(false, name, std::string("wrong type: ") + e.what());
  }
}

}  // namespace

int main() {
  // 3D phantom, odd Gaussian PSF
  const NdImage psf3 = synth::gaussian_psf({7, 7, 7}, {1.0});
  compare_rl("blobs3d", blurred_blobs({20, 48, 48}, 4, 7, psf3), psf3, 6, false);
  compare_rl("blobs3d_flat", blurred_blobs({20, 48, 48}, 4, 9, psf3), psf3, 4, true);
  compare_default_rule("blobs3d", blurred_blobs({20, 48, 48}, 4, 17, psf3), psf3, 12);
  // fast-kernel grid (W = 96 x 288 x 288, the C1 grid) at the C1 size
  const NdImage psf15 = synth::gaussian_psf({15, 15, 15}, {1.75});
  compare_rl("c1", blurred_blobs({64, 256, 256}, 60, 1, psf15), psf15, 3, false);
  // 2D and the accelerated backend tag
  {
    std::vector<float> v(40 * 52);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = 0.2f + 0.001f * (float)((i * 7919) % 997);
    const NdImage img = NdImage::f32({40, 52}, v).with_backend(BackendId::accelerated);
    compare_rl("img2d_accel", img, synth::gaussian_psf({9, 9}, {1.5}), 5, false);
  }
  // u16 input is promoted like the reference (image.hpp as_f32)
  {
    std::vector<std::uint16_t> v(12 * 30 * 30);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = (std::uint16_t)(100 + (i * 31) % 900);
    compare_rl("u16", NdImage::u16({12, 30, 30}, v), synth::gaussian_psf({5, 5, 5}, {1.0}), 3, false);
  }

  // errors: same type and what() as the reference
  const std::vector<float> good(4 * 6 * 6, 0.5f);
  std::vector<float> ramp(good);
  for (std::size_t i = 0; i < ramp.size(); ++i) ramp[i] += 0.01f * (float)i;
  const NdImage obs = NdImage::f32({4, 6, 6}, ramp);
  const NdImage gpsf = synth::gaussian_psf({3, 3, 3}, {1.0});
  deconv::StoppingRule base{deconv::StopMetric::si_psnr_vs_input, 1e-3, 3, 3};
  expect_error<Error>("err rel_tol", obs, gpsf, {base.metric, 0.0, 3, 3});
  expect_error<Error>("err patience", obs, gpsf, {base.metric, 1e-3, 0, 3});
  expect_error<Error>("err max_iters", obs, gpsf, {base.metric, 1e-3, 3, 0});
  expect_error<ShapeMismatch>("err rank", obs, synth::gaussian_psf({3, 3}, {1.0}), base);
  {
    std::vector<float> neg(ramp);
    neg[17] = -1e-3f;
    expect_error<NegativeInput>("err negative observed", NdImage::f32({4, 6, 6}, neg), gpsf, base);
    std::vector<float> k(gpsf.f32_values().begin(), gpsf.f32_values().end());
    for (float& x : k) x *= 1.01f;
    expect_error<UnnormalizedPsf>("err unnormalized psf", obs, NdImage::f32({3, 3, 3}, k), base);
    k[0] = -1e-4f;
    expect_error<NegativeInput>("err negative psf", obs, NdImage::f32({3, 3, 3}, k), base);
    expect_error<NegativeInput>("err order (observed before psf)", NdImage::f32({4, 6, 6}, neg),
                                NdImage::f32({3, 3, 3}, k), base);
  }
  expect_error<DegenerateReference>("err degenerate", NdImage::f32({4, 6, 6}, good), gpsf, base);

  // rl_step: registry dispatch for both backend tags, and the transforms form
  {
    std::vector<float> e(6 * 14 * 18), o(e.size());
    for (std::size_t i = 0; i < e.size(); ++i) {
      e[i] = 0.1f + 0.001f * (float)((i * 131) % 1000);
      o[i] = 0.1f + 0.001f * (float)((i * 211) % 1000);
    }
    const NdImage k = synth::gaussian_psf({3, 5, 5}, {0.8, 1.2, 1.2});
    std::vector<std::uint64_t> s{6, 14, 18}, ks{3, 5, 5};
    std::vector<float> ref(e.size());
    char err[256];
    vkref_rl_step(3, s.data(), e.data(), o.data(), ks.data(), k.f32_values().data(), 0, ref.data(), err, 256);
    for (BackendId b : {BackendId::reference, BackendId::accelerated}) {
      const NdImage E = NdImage::f32({6, 14, 18}, e).with_backend(b);
      const NdImage Ob = NdImage::f32({6, 14, 18}, o).with_backend(b);
      const NdImage out = deconv::rl_step(E, Ob, k.with_backend(b));
      report(rel_l2(out.f32_values(), ref) <= 1e-5 && out.backend() == b,
             std::string("rl_step dispatch ") + to_string(b));
    }
    deconv::RlTransforms t({6, 14, 18}, k, 1);
    const NdImage out = deconv::rl_step(NdImage::f32({6, 14, 18}, e), NdImage::f32({6, 14, 18}, o), t);
    report(rel_l2(out.f32_values(), ref) <= 1e-5 && t.fft_shape() == Shape{8, 18, 24}, "rl_step transforms");
    try {
      deconv::rl_step(NdImage::f32({2, 2, 2}, std::vector<float>(8, 1.f)),
                      NdImage::f32({2, 2, 2}, std::vector<float>(8, 1.f)), t);
      report(false, "rl_step transforms shape error");
    } catch (const ShapeMismatch& ex) {
      report(std::string(ex.what()) == "ShapeMismatch: rl_step: transforms were prepared for [6,14,18]",
             "rl_step transforms shape error", ex.what());
    }
  }
  // richardson_lucy_batch: element-wise identical to richardson_lucy
  {
    const NdImage k = synth::gaussian_psf({5, 5, 5}, {1.0});
    std::vector<NdImage> vols;
    for (int i = 0; i < 3; ++i) vols.push_back(blurred_blobs({20, 48, 40}, 4, 40 + i, k));
    deconv::StoppingRule rule{deconv::StopMetric::si_psnr_vs_input, 1e-300, 4, 4};
    const auto batch = deconv::richardson_lucy_batch(vols, k, rule, false);
    bool ok = batch.size() == vols.size();
    double worst = 0;
    for (std::size_t i = 0; ok && i < vols.size(); ++i) {
      const deconv::RlResult one = deconv::richardson_lucy(vols[i], k, rule, false);
      const auto a = batch[i].estimate.f32_values(), b = one.estimate.f32_values();
      ok = std::equal(a.begin(), a.end(), b.begin()) && batch[i].trace.records.size() == one.trace.records.size() &&
           batch[i].trace.stop_reason == one.trace.stop_reason && batch[i].trace.fft_shape == one.trace.fft_shape;
      for (std::size_t r = 0; ok && r < one.trace.records.size(); ++r)
        ok = batch[i].trace.records[r].value == one.trace.records[r].value &&
             batch[i].trace.log_likelihood[r] == one.trace.log_likelihood[r];
      const RefRun ref = ref_rl(vols[i], k, rule, false);
      worst = std::max(worst, rel_l2(a, ref.est));
    }
    char buf[96];
    std::snprintf(buf, sizeof buf, "worst relL2 vs reference %.2e", worst);
    report(ok && worst <= 1e-3, "richardson_lucy_batch == per-volume richardson_lucy", buf);
    // the first failing volume's exception, as the per-volume loop throws it
    std::vector<float> bad(vols[1].f32_values().begin(), vols[1].f32_values().end());
    bad[5] = -1.f;
    vols[1] = NdImage::f32({20, 48, 40}, bad);
    try {
      deconv::richardson_lucy_batch(vols, k, rule, false);
      report(false, "richardson_lucy_batch error", "no exception");
    } catch (const NegativeInput& e) {
      report(std::string(e.what()) == "NegativeInput: observed image must be nonnegative",
             "richardson_lucy_batch error", e.what());
    }
  }
  // filters::fft_convolve through the registry (both tags) on the GPU vs the reference
  {
    struct Case {
      Shape a, k;
      bool circ;
    };
    const Case cases[] = {{{20, 33, 40}, {5, 4, 7}, false}, {{16, 18, 20}, {3, 3, 5}, true},
                          {{7, 11, 13}, {3, 4, 5}, true}, {{50, 61}, {9, 8}, false}};
    for (const Case& c : cases) {
      std::size_t n = 1, kn = 1;
      for (auto v : c.a) n *= v;
      for (auto v : c.k) kn *= v;
      std::vector<float> a(n), k(kn), ref(n);
      for (std::size_t i = 0; i < n; ++i) a[i] = std::sin(0.37f * (float)i) + 0.1f * (float)(i % 7);
      for (std::size_t i = 0; i < kn; ++i) k[i] = 0.5f + std::cos(0.9f * (float)i);
      std::vector<std::uint64_t> s(c.a.begin(), c.a.end()), ks(c.k.begin(), c.k.end());
      char err[256];
      vkref_fft_convolve((int)s.size(), s.data(), a.data(), ks.data(), k.data(), c.circ, ref.data(), err, 256);
      for (BackendId b : {BackendId::reference, BackendId::accelerated}) {
        const NdImage out = filters::fft_convolve(NdImage::f32(c.a, a).with_backend(b), NdImage::f32(c.k, k).with_backend(b), c.circ);
        char buf[96];
        std::snprintf(buf, sizeof buf, "relL2 %.2e", rel_l2(out.f32_values(), ref));
        report(rel_l2(out.f32_values(), ref) <= 1e-5 && out.backend() == b,
               std::string("fft_convolve registry ") + to_string(b) + (c.circ ? " circular " : " linear ") +
                   shape_to_string(c.a),
               buf);
      }
    }
    try {
      filters::fft_convolve(NdImage::f32({4, 4}, std::vector<float>(16, 1.f)),
                            NdImage::f32({5, 3}, std::vector<float>(15, 1.f)), true);
      report(false, "fft_convolve KernelTooLarge", "no exception");
    } catch (const KernelTooLarge& e) {
      report(std::string(e.what()) == "KernelTooLarge: circular convolution needs kernel <= image",
             "fft_convolve KernelTooLarge", e.what());
    }
  }
  // io::write_volume / read_volume (io_b200.cpp over vk_io.h): round trip, and
  // byte-identical to the reference writer when it is linked in
  {
    std::vector<float> v(3 * 4 * 5);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = 0.25f * (float)i - 3.f;
    const NdImage img = NdImage::f32({3, 4, 5}, v).with_spacing({2.0, 0.5, 0.125});
    const std::string ours = "/tmp/vk_dropin_io_ours.ndiv", theirs = "/tmp/vk_dropin_io_ref.ndiv";
    io::write_volume(ours, img);
    const NdImage back = io::read_volume(ours);
    const auto bv = back.f32_values();
    bool ok = back.shape() == img.shape() && back.spacing() && *back.spacing() == *img.spacing() &&
              std::equal(bv.begin(), bv.end(), v.begin());
    if (vkref_write_volume) {
      const std::uint64_t sh[3] = {3, 4, 5};
      const double sp[3] = {2.0, 0.5, 0.125};
      char err[256];
      vkref_write_volume(theirs.c_str(), 0, 3, sh, v.data(), sp, err, 256);
      std::ifstream fa(ours, std::ios::binary), fb(theirs, std::ios::binary);
      const std::string A((std::istreambuf_iterator<char>(fa)), {}), B((std::istreambuf_iterator<char>(fb)), {});
      ok = ok && A == B;
    }
    report(ok, "io write/read round trip (byte-identical to the reference writer)");
    try {
      io::read_volume("/tmp/vk_dropin_io_missing.ndiv");
      report(false, "io read missing file");
    } catch (const Error& e) {
      report(std::string(e.what()) == "cannot open '/tmp/vk_dropin_io_missing.ndiv'", "io read missing file",
             e.what());
    }
  }
  // trace CSV (deconv.cpp:85-96)
  {
    deconv::IterationTrace tr;
    tr.records.push_back({1, "si_psnr_vs_input", 12.5, 0.25});
    tr.records.push_back({2, "frc_resolution", INFINITY, 0.5});
    std::ostringstream os;
    tr.to_csv(os);
    report(os.str() == "iter,metric,value,wall_time_s\n1,si_psnr_vs_input,12.5,0.25\n2,frc_resolution,inf,0.5\n",
           "trace csv");
  }
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
