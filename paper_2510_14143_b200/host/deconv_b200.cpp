// Drop-in replacement for the reference's src/deconv.cpp.
//
// Implements the unchanged public header voxelkit/deconv.hpp
// (reference proj/include/voxelkit/deconv.hpp:28-103) on top of the C ABI
// in include/vk_rl.h, whose kernels run on the B200.  Link this translation
// unit instead of src/deconv.cpp (and libvkrl.so) and every caller —
// tools/voxelkit_main.cpp:436 (CLI `deconvolve`) and registry dispatch of
// "rl_step" (src/deconv.cpp:196-200) — runs on the GPU with no other change.
//
// Behaviour kept from the reference, line by line:
//   * validation order and exception types/messages (deconv.cpp:306-326),
//     re-thrown from vk_status codes; no exception crosses the C ABI;
//   * RlTransforms semantics (deconv.cpp:98-176): PSF spectra built once,
//     fft_shape = good_size(shape + psf - 1), "one run at a time";
//   * rl_step shape checks and messages (deconv.cpp:178-194);
//   * IterationTrace contents and CSV format (deconv.cpp:85-96, 346-430);
//   * "rl_step" registered for BOTH backend tags (deconv.cpp:437-449).  The
//     tag is metadata here: both run the same GPU kernel (no multi-backend
//     dispatch, no CPU fallback).
// The GPU is selected by VOXELKIT_DEVICE (default 0).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <ostream>
#include <string>
#include <vector>

#include "voxelkit/deconv.hpp"
#include "voxelkit/errors.hpp"
#include "voxelkit/image.hpp"
#include "voxelkit/registry.hpp"
#include "voxelkit_b200/deconv_batch.hpp"
#include "vk_rl.h"

namespace voxelkit::deconv {

namespace {

int device() {
  const char* e = std::getenv("VOXELKIT_DEVICE");
  return e ? std::atoi(e) : 0;
}

// Strips the "Name: " prefix the C ABI reports (it equals what()); the typed
// exception constructors add it back (errors.hpp:30-34).
std::string body(const char* msg, const char* name) {
  const std::string m = msg ? msg : "";
  const std::string p = std::string(name) + ": ";
  return m.rfind(p, 0) == 0 ? m.substr(p.size()) : m;
}

[[noreturn]] void rethrow(vk_status st) {
  const char* m = vk_last_error();
  switch (st) {
    case VK_ERR_SHAPE: throw ShapeMismatch(body(m, "ShapeMismatch"));
    case VK_ERR_NEGATIVE: throw NegativeInput(body(m, "NegativeInput"));
    case VK_ERR_UNNORMALIZED_PSF: throw UnnormalizedPsf(body(m, "UnnormalizedPsf"));
    case VK_ERR_DEGENERATE_REF: throw DegenerateReference(body(m, "DegenerateReference"));
    case VK_ERR_TOO_SMALL: throw TooSmall(body(m, "TooSmall"));
    case VK_ERR_ODD_EXTENT: throw OddExtent(body(m, "OddExtent"));
    default: throw Error(m ? m : "vk_rl failure");
  }
}

void check(vk_status st) {
  if (st != VK_OK) rethrow(st);
}

std::vector<std::uint64_t> u64(const Shape& s) { return {s.begin(), s.end()}; }

// Caller-side buffers of one vk_trace.
struct TraceBuf {
  std::vector<double> metric, wall, ll;
  vk_trace tr{};
  explicit TraceBuf(int max_iters) {
    const int cap = max_iters > 0 ? max_iters : 1;
    metric.resize(cap);
    wall.resize(cap);
    ll.resize(cap);
    tr.capacity = cap;
    tr.metric = metric.data();
    tr.wall_s = wall.data();
    tr.log_likelihood = ll.data();
  }
};

// The C ABI's stopping rule; FRC uses the x spacing of the observed image
// (deconv.cpp:286-287).
vk_stop_rule c_rule(const StoppingRule& rule, const NdImage& obs) {
  const double spacing = obs.spacing() ? obs.spacing()->back() : 0.0;
  return vk_stop_rule{static_cast<int>(rule.metric), rule.rel_tol, rule.patience, rule.max_iters, spacing};
}

RlResult assemble(const NdImage& obs, const StoppingRule& rule, std::vector<float> est, const TraceBuf& t) {
  RlResult res;
  res.estimate = NdImage::f32_like(obs, std::move(est));
  for (int i = 0; i < t.tr.iters_run; ++i) {
    res.trace.records.push_back({i + 1, to_string(rule.metric), t.metric[i], t.wall[i]});
    res.trace.log_likelihood.push_back(t.ll[i]);
  }
  res.trace.fft_shape.assign(t.tr.fft_shape, t.tr.fft_shape + obs.rank());
  res.trace.stop_reason = t.tr.stop_reason == 1 ? "converged" : "max_iters";
  return res;
}

}  // namespace

const char* to_string(StopMetric m) {
  switch (m) {
    case StopMetric::si_psnr_vs_input: return "si_psnr_vs_input";
    case StopMetric::ssim_vs_prev: return "ssim_vs_prev";
    case StopMetric::frc_resolution: return "frc_resolution";
  }
  return "?";
}

void IterationTrace::to_csv(std::ostream& out) const {
  out << "iter,metric,value,wall_time_s\n";
  for (const auto& r : records) {
    out << r.iter << "," << r.metric_name << ",";
    if (std::isinf(r.value)) {
      out << (r.value > 0 ? "inf" : "-inf");
    } else {
      out << r.value;
    }
    out << "," << r.wall_time_s << "\n";
  }
}

struct RlTransforms::Impl {
  vk_rl_plan plan = nullptr;
  Shape image_shape;
  Shape work_shape;
  ~Impl() {
    if (plan) vk_rl_plan_destroy(plan);
  }
};

RlTransforms::RlTransforms(const Shape& image_shape, const NdImage& psf, int /*threads*/)
    : impl_(std::make_unique<Impl>()) {
  const NdImage k = psf.as_f32();
  if (k.rank() != image_shape.size()) throw ShapeMismatch("psf rank must match the image rank");
  const auto sh = u64(image_shape);
  const auto ks = u64(k.shape());
  check(vk_rl_plan_create(device(), static_cast<int>(sh.size()), sh.data(), static_cast<int>(ks.size()),
                          ks.data(), k.f32_values().data(), /*pad_replicate=*/0, &impl_->plan));
  impl_->image_shape = image_shape;
  int rank = 0;
  std::uint64_t w[VK_MAX_RANK] = {};
  check(vk_rl_plan_shapes(impl_->plan, &rank, nullptr, nullptr, w));
  impl_->work_shape.assign(w, w + rank);
}
RlTransforms::~RlTransforms() = default;

const Shape& RlTransforms::image_shape() const { return impl_->image_shape; }
const Shape& RlTransforms::fft_shape() const { return impl_->work_shape; }

NdImage rl_step(const NdImage& estimate, const NdImage& observed, RlTransforms& transforms) {
  require_same_shape(estimate, observed, "rl_step");
  if (estimate.shape() != transforms.image_shape())
    throw ShapeMismatch("rl_step: transforms were prepared for " + shape_to_string(transforms.image_shape()));
  const NdImage e = estimate.as_f32();
  const NdImage o = observed.as_f32();
  std::vector<float> out(e.size());
  check(vk_rl_step(transforms.impl_->plan, e.f32_values().data(), o.f32_values().data(), out.data()));
  return NdImage::f32_like(estimate, std::move(out));
}

NdImage rl_step(const NdImage& estimate, const NdImage& observed, const NdImage& psf) {
  return dispatch<NdImage(const NdImage&, const NdImage&, const NdImage&)>("rl_step", estimate, observed, psf);
}

RlResult richardson_lucy(const NdImage& observed, const NdImage& psf, const StoppingRule& rule, bool flat_init) {
  const NdImage obs = observed.as_f32();
  const NdImage k = psf.as_f32();
  const auto sh = u64(obs.shape());
  const auto ks = u64(k.shape());
  TraceBuf t(rule.max_iters);
  const vk_stop_rule r = c_rule(rule, obs);
  std::vector<float> est(obs.size());
  // one-shot call: the C ABI keeps the plan (OTFs, work buffers) cached for
  // the next call on the same shape and PSF
  check(vk_richardson_lucy(device(), static_cast<int>(sh.size()), sh.data(), obs.f32_values().data(),
                           static_cast<int>(ks.size()), ks.data(), k.f32_values().data(), &r, flat_init ? 1 : 0,
                           est.data(), &t.tr));
  return assemble(obs, rule, std::move(est), t);
}

std::vector<RlResult> richardson_lucy_batch(const std::vector<NdImage>& observed, const NdImage& psf,
                                            const StoppingRule& rule, bool flat_init) {
  std::vector<RlResult> out;
  const auto sequential = [&] {
    out.clear();
    for (const NdImage& o : observed) out.push_back(richardson_lucy(o, psf, rule, flat_init));
    return out;
  };
  if (observed.size() < 2) return sequential();
  const NdImage k = psf.as_f32();
  std::vector<NdImage> obs;
  obs.reserve(observed.size());
  for (const NdImage& o : observed) obs.push_back(o.as_f32());
  const vk_stop_rule r = c_rule(rule, obs[0]);
  for (const NdImage& o : obs)  // one plan serves volumes of one shape (and one FRC spacing)
    if (o.shape() != obs[0].shape() || c_rule(rule, o).spacing != r.spacing || k.rank() != o.rank())
      return sequential();
  const auto sh = u64(obs[0].shape());
  const auto ks = u64(k.shape());
  const int n = static_cast<int>(obs.size());
  std::vector<std::vector<float>> est(n, std::vector<float>(obs[0].size()));
  std::vector<TraceBuf> tb;
  tb.reserve(n);
  std::vector<vk_trace> trs(n);
  std::vector<const float*> ip(n);
  std::vector<float*> op(n);
  for (int i = 0; i < n; ++i) {
    tb.emplace_back(rule.max_iters);
    trs[i] = tb[i].tr;
    ip[i] = obs[i].f32_values().data();
    op[i] = est[i].data();
  }
  // one cached plan, volumes on its concurrent batch lanes
  const vk_status st =
      vk_richardson_lucy_batch(device(), static_cast<int>(sh.size()), sh.data(), n, ip.data(),
                               static_cast<int>(ks.size()), ks.data(), k.f32_values().data(), &r, flat_init ? 1 : 0,
                               op.data(), trs.data());
  // any failure: the per-volume loop throws exactly what the reference would
  if (st != VK_OK) return sequential();
  for (int i = 0; i < n; ++i) {
    tb[i].tr = trs[i];
    out.push_back(assemble(obs[i], rule, std::move(est[i]), tb[i]));
  }
  return out;
}

}  // namespace voxelkit::deconv

namespace voxelkit::detail {

void register_filter_ops_b200(ExecutionRegistry& reg);  // host/filters_b200.cpp

void register_deconv_ops(ExecutionRegistry& reg) {
  // The registry is filled register_filter_ops first, register_deconv_ops
  // last (registry.cpp:87-93) and add() replaces an entry, so this puts
  // "fft_convolve" on the GPU for both tags too (filters.cpp:316-323).
  register_filter_ops_b200(reg);
  using StepSig = NdImage(const NdImage&, const NdImage&, const NdImage&);
  auto step = [](const NdImage& estimate, const NdImage& observed, const NdImage& psf) {
    deconv::RlTransforms transforms(estimate.shape(), psf.as_f32(), 1);
    return deconv::rl_step(estimate, observed, transforms);
  };
  reg.add<StepSig>("rl_step", BackendId::reference, step);
  reg.add<StepSig>("rl_step", BackendId::accelerated, step);
}

}  // namespace voxelkit::detail
