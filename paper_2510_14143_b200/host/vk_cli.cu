// voxelkit_b200 — the reference CLI's `deconvolve` subcommand on the B200
// path.
//
// Mirrors `voxelkit deconvolve` (/root/reference/proj/tools/voxelkit_main.cpp:
// flags :538-561, run_deconvolve :398-472, exit codes :42-66): the same
// options and defaults, the same outputs (estimate.ndiv, trace.csv,
// summary.json) and the same stdout line.  Everything heavy runs on the GPU
// through the C ABI: the input volume streams from the file into device
// memory (vk_volume_read_device), a synthetic input is generated and blurred
// on the device (vk_generate_blobs + vk_conv_run_device), the deconvolution
// runs on device buffers (vk_rl_run_device) and the estimate streams back to
// the file (vk_volume_write_device).  Only the si_psnr figures of the summary
// (synthetic mode) are computed on the host, from one D2H copy of each image.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <limits>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "../../include/vk_io.h"
#include "../../include/vk_rl.h"

namespace {

constexpr int kOk = 0, kIoError = 2, kBadStructure = 4, kBadNumeric = 5, kUsage = 106;

struct CliError {
  int status;  // vk_status
  std::string msg;
};

void check(vk_status st) {
  if (st != VK_OK) throw CliError{st, vk_last_error()};
}
void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CliError{VK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

// classify() of the reference CLI (voxelkit_main.cpp:46-66) by status code.
int exit_code(int st) {
  switch (st) {
    case VK_ERR_BAD_MAGIC:
    case VK_ERR_HEADER_MISMATCH:
    case VK_ERR_TRUNCATED: return kIoError;
    case VK_ERR_SHAPE: return kBadStructure;
    case VK_ERR_UNNORMALIZED_PSF:
    case VK_ERR_NEGATIVE:
    case VK_ERR_PLACEMENT:
    case VK_ERR_DEGENERATE_REF:
    case VK_ERR_TOO_SMALL:
    case VK_ERR_ODD_EXTENT:
    case VK_ERR_EVEN_EXTENT: return kBadNumeric;
    case VK_ERR_ARG: return kIoError;  // plain voxelkit::Error (file open / write)
    default: return kBadStructure;
  }
}

struct Args {
  std::string input;
  bool synthetic = false;
  std::vector<uint64_t> shape{32, 128, 128};
  uint64_t objects = 20;
  std::vector<double> radius{6.0, 10.0};
  uint64_t seed = 0;
  double noise = 0.05;
  double anisotropy = 1.0;
  std::string psf_path;
  std::vector<double> gaussian;
  std::string metric = "frc";
  double rel_tol = 1e-3;
  int patience = 3;
  int max_iters = 100;
  bool flat_init = false;
  std::string backend = "reference";
  std::string out_dir = ".";
  int device = 0;
};

void usage(std::ostream& o) {
  o << "usage: voxelkit_b200 deconvolve [--input PATH | --synthetic] [--shape Z Y X] [--objects N]\n"
       "         [--radius MIN [MAX]] [--seed S] [--noise F] [--anisotropy A] [--psf PATH]\n"
       "         [--gaussian S [S S]] [--metric si_psnr|ssim|frc] [--rel-tol T] [--patience P]\n"
       "         [--max-iters N] [--flat-init] [--backend reference|accelerated] [--out DIR]\n"
       "         [--device D]\n";
}

[[noreturn]] void bad_usage(const std::string& m) {
  std::cerr << m << "\n";
  usage(std::cerr);
  std::exit(kUsage);
}

double to_d(const std::string& s, const std::string& opt) {
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  if (s.empty() || *end) bad_usage("invalid value '" + s + "' for " + opt);
  return v;
}
long long to_i(const std::string& s, const std::string& opt) {
  char* end = nullptr;
  const long long v = std::strtoll(s.c_str(), &end, 10);
  if (s.empty() || *end) bad_usage("invalid value '" + s + "' for " + opt);
  return v;
}

Args parse(int argc, char** argv) {
  if (argc < 2) bad_usage("a subcommand is required");
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    usage(std::cout);
    std::exit(kOk);
  }
  if (sub != "deconvolve") bad_usage("unsupported subcommand '" + sub + "' (only deconvolve is on the B200 path)");
  Args a;
  std::vector<std::string> tok;
  for (int i = 2; i < argc; ++i) {
    std::string t = argv[i];
    const size_t eq = t.find('=');
    if (t.rfind("--", 0) == 0 && eq != std::string::npos) {
      tok.push_back(t.substr(0, eq));
      tok.push_back(t.substr(eq + 1));
    } else {
      tok.push_back(t);
    }
  }
  auto values = [&](size_t& i, size_t lo, size_t hi, const std::string& opt) {
    std::vector<std::string> v;
    while (i + 1 < tok.size() && v.size() < hi && !(tok[i + 1].rfind("--", 0) == 0)) v.push_back(tok[++i]);
    if (v.size() < lo) bad_usage(opt + " expects " + std::to_string(lo) + " value(s)");
    return v;
  };
  for (size_t i = 0; i < tok.size(); ++i) {
    const std::string& o = tok[i];
    if (o == "--input") a.input = values(i, 1, 1, o)[0];
    else if (o == "--synthetic") a.synthetic = true;
    else if (o == "--shape") {
      a.shape.clear();
      for (auto& v : values(i, 3, 3, o)) a.shape.push_back((uint64_t)to_i(v, o));
    } else if (o == "--objects") a.objects = (uint64_t)to_i(values(i, 1, 1, o)[0], o);
    else if (o == "--radius") {
      a.radius.clear();
      for (auto& v : values(i, 1, 2, o)) a.radius.push_back(to_d(v, o));
    } else if (o == "--seed") a.seed = (uint64_t)to_i(values(i, 1, 1, o)[0], o);
    else if (o == "--noise") a.noise = to_d(values(i, 1, 1, o)[0], o);
    else if (o == "--anisotropy") a.anisotropy = to_d(values(i, 1, 1, o)[0], o);
    else if (o == "--psf") a.psf_path = values(i, 1, 1, o)[0];
    else if (o == "--gaussian") {
      a.gaussian.clear();
      for (auto& v : values(i, 1, 3, o)) a.gaussian.push_back(to_d(v, o));
    } else if (o == "--metric") a.metric = values(i, 1, 1, o)[0];
    else if (o == "--rel-tol") a.rel_tol = to_d(values(i, 1, 1, o)[0], o);
    else if (o == "--patience") a.patience = (int)to_i(values(i, 1, 1, o)[0], o);
    else if (o == "--max-iters") a.max_iters = (int)to_i(values(i, 1, 1, o)[0], o);
    else if (o == "--flat-init") a.flat_init = true;
    else if (o == "--backend") a.backend = values(i, 1, 1, o)[0];
    else if (o == "--out") a.out_dir = values(i, 1, 1, o)[0];
    else if (o == "--device") a.device = (int)to_i(values(i, 1, 1, o)[0], o);
    else if (o == "-h" || o == "--help") {
      usage(std::cout);
      std::exit(kOk);
    } else bad_usage("unknown option '" + o + "'");
  }
  return a;
}

// json_double of vk_io.cpp's header writer, for summary.json values.
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string out, digits;
  const char* p = buf;
  if (*p == '-') {
    out += '-';
    ++p;
  }
  while (*p && *p != 'e') {
    if (*p != '.') digits += *p;
    ++p;
  }
  const int e10 = std::atoi(p + 1);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = (int)digits.size(), n = e10 + 1;
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int ex = n - 1, ab = ex < 0 ? -ex : ex;
    out += ex < 0 ? "e-" : "e+";
    if (ab < 10) out += '0';
    out += std::to_string(ab);
  }
  return out;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

// metrics::si_psnr (metrics.cpp:67-101) on host copies.
double si_psnr(const std::vector<float>& x, const std::vector<float>& r) {
  const double n = (double)x.size();
  double sx = 0, sr = 0, sxx = 0, sxr = 0, srr = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    const double a = x[i], b = r[i];
    sx += a;
    sr += b;
    sxx += a * a;
    sxr += a * b;
    srr += b * b;
  }
  const double var_r = srr / n - (sr / n) * (sr / n);
  if (var_r <= 0.0) throw CliError{VK_ERR_DEGENERATE_REF, "DegenerateReference: si_psnr needs a non-constant reference"};
  const double var_x = sxx / n - (sx / n) * (sx / n);
  double a = 0.0;
  if (var_x > 0.0) a = (sxr / n - (sx / n) * (sr / n)) / var_x;
  const double b = sr / n - a * (sx / n);
  double err = 0;
  for (size_t i = 0; i < x.size(); ++i) {
    const double d = a * x[i] + b - r[i];
    err += d * d;
  }
  err /= n;
  if (err <= 0.0) return std::numeric_limits<double>::infinity();
  float mn = r[0], mx = r[0];
  for (float v : r) {
    mn = std::min(mn, v);
    mx = std::max(mx, v);
  }
  const double range = (double)mx - mn;
  return 10.0 * std::log10(range * range / err);
}

__global__ void clip_kernel(float* v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    v[i] = v[i] < 0.0f ? 0.0f : v[i];  // std::max(v, 0.f) (core_ops.cpp:42)
}

template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(size_t n) { cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
};

std::vector<float> to_f32(const vk_volume_info& info, const std::vector<char>& raw) {
  size_t n = 1;
  for (int a = 0; a < info.rank; ++a) n *= info.shape[a];
  std::vector<float> v(n);
  for (size_t i = 0; i < n; ++i) {
    switch (info.elem) {
      case VK_ELEM_F32: std::memcpy(&v[i], raw.data() + 4 * i, 4); break;
      case VK_ELEM_U16: {
        uint16_t u;
        std::memcpy(&u, raw.data() + 2 * i, 2);
        v[i] = (float)u;
        break;
      }
      case VK_ELEM_U32: {
        uint32_t u;
        std::memcpy(&u, raw.data() + 4 * i, 4);
        v[i] = (float)u;
        break;
      }
      default: v[i] = raw[i] ? 1.0f : 0.0f;
    }
  }
  return v;
}

// Host read of any element kind as f32 (NdImage::as_f32).
std::vector<float> read_host_f32(const std::string& path, vk_volume_info& info) {
  check(vk_volume_info_read(path.c_str(), &info));
  std::vector<char> raw(info.payload_bytes);
  check(vk_volume_read(path.c_str(), &info, raw.data(), raw.size()));
  return to_f32(info, raw);
}

void mkdirs(const std::string& dir) {
  std::string cur;
  std::stringstream ss(dir);
  std::string part;
  if (!dir.empty() && dir[0] == '/') cur = "/";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    cur += part + "/";
    mkdir(cur.c_str(), 0777);
  }
  struct stat st {};
  if (stat(dir.c_str(), &st) != 0 || !S_ISDIR(st.st_mode))
    throw CliError{VK_ERR_ARG, "cannot create directory '" + dir + "'"};
}

std::ofstream open_out(const std::string& path) {
  std::ofstream out(path);
  if (!out) throw CliError{VK_ERR_ARG, "cannot open '" + path + "' for writing"};
  return out;
}

int run(const Args& args) {
  cuda(cudaSetDevice(args.device), "cudaSetDevice");
  cudaStream_t s;
  cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");

  // PSF: a volume file, or gaussian_psf with 2 ceil(4 sigma) + 1 extents
  std::vector<float> psf;
  std::vector<uint64_t> kshape;
  if (!args.psf_path.empty()) {
    vk_volume_info pi{};
    psf = read_host_f32(args.psf_path, pi);
    kshape.assign(pi.shape, pi.shape + pi.rank);
  } else {
    std::vector<double> sg = args.gaussian.empty() ? std::vector<double>{1.0, 2.0, 2.0} : args.gaussian;
    for (double v : sg) kshape.push_back(2 * (uint64_t)std::ceil(4.0 * v) + 1);
    size_t n = 1;
    for (auto e : kshape) n *= e;
    psf.resize(n);
    check(vk_gaussian_psf((int)kshape.size(), kshape.data(), sg.data(), (int)sg.size(), psf.data()));
  }

  // observed: the input volume, or blobs blurred by the PSF and clipped at 0
  std::vector<uint64_t> shape;
  vk_volume_info obs_info{};
  bool have_truth = false;
  size_t n = 0;
  Dev<float>* d_obs = nullptr;
  Dev<float>* d_truth = nullptr;
  if (!args.input.empty()) {
    check(vk_volume_info_read(args.input.c_str(), &obs_info));
    shape.assign(obs_info.shape, obs_info.shape + obs_info.rank);
    n = 1;
    for (auto e : shape) n *= e;
    d_obs = new Dev<float>(n);
    if (obs_info.elem == VK_ELEM_F32) {
      check(vk_volume_read_device(args.input.c_str(), &obs_info, d_obs->p, n * sizeof(float), s));
    } else {
      std::vector<float> h = read_host_f32(args.input, obs_info);
      cuda(cudaMemcpy(d_obs->p, h.data(), n * sizeof(float), cudaMemcpyHostToDevice), "H2D");
    }
  } else {
    vk_synth_spec sp{};
    std::vector<uint64_t> sh = args.shape;
    if (sh == std::vector<uint64_t>{32, 128, 128}) sh = {24, 96, 96};  // voxelkit_main.cpp:420-421
    for (int a = 0; a < 3; ++a) sp.shape[a] = sh[a];
    sp.n_objects = args.objects;
    sp.radius_min = args.radius.at(0);
    sp.radius_max = args.radius.size() > 1 ? args.radius[1] : args.radius[0];
    sp.seed = args.seed;
    sp.noise_sigma = args.noise;
    sp.anisotropy = args.anisotropy;
    shape = sh;
    n = sh[0] * sh[1] * sh[2];
    d_truth = new Dev<float>(n);
    d_obs = new Dev<float>(n);
    double spacing[3];
    check(vk_generate_blobs(args.device, &sp, d_truth->p, spacing, s));
    obs_info.rank = 3;
    for (int a = 0; a < 3; ++a) {
      obs_info.shape[a] = sh[a];
      obs_info.spacing[a] = spacing[a];
    }
    obs_info.has_spacing = 1;
    vk_rl_plan conv = nullptr;
    check(vk_conv_plan_create(args.device, 3, shape.data(), (int)kshape.size(), kshape.data(), psf.data(), 0,
                              &conv));
    vk_status st = vk_conv_run_device(conv, d_truth->p, d_obs->p, s);
    vk_rl_plan_destroy(conv);
    check(st);
    clip_kernel<<<148 * 4, 256, 0, s>>>(d_obs->p, n);  // vmax(., 0)
    cuda(cudaGetLastError(), "clip");
    cuda(cudaStreamSynchronize(s), "blur");
    have_truth = true;
  }
  obs_info.elem = VK_ELEM_F32;

  const int metric = args.metric == "si_psnr" ? VK_METRIC_SI_PSNR_VS_INPUT
                     : args.metric == "ssim"  ? VK_METRIC_SSIM_VS_PREV
                                              : VK_METRIC_FRC_RESOLUTION;
  static const char* kMetricName[3] = {"si_psnr_vs_input", "ssim_vs_prev", "frc_resolution"};
  vk_stop_rule rule{metric, args.rel_tol, args.patience, args.max_iters,
                    obs_info.has_spacing ? obs_info.spacing[obs_info.rank - 1] : 0.0};
  // the rule is validated before anything else inside richardson_lucy
  const int cap = std::max(args.max_iters, 1);
  std::vector<double> mv(cap), ws(cap), ll(cap);
  vk_trace tr{};
  tr.capacity = cap;
  tr.metric = mv.data();
  tr.wall_s = ws.data();
  tr.log_likelihood = ll.data();
  Dev<float> d_est(n);
  vk_rl_plan plan = nullptr;
  // richardson_lucy validates the rule before the ranks (deconv.cpp:306-311)
  if (args.rel_tol <= 0 && !std::isinf(args.rel_tol)) throw CliError{VK_ERR_ARG, "rel_tol must be positive"};
  if (args.patience < 1) throw CliError{VK_ERR_ARG, "patience must be >= 1"};
  if (args.max_iters < 1) throw CliError{VK_ERR_ARG, "max_iters must be >= 1"};
  check(vk_rl_plan_create(args.device, (int)shape.size(), shape.data(), (int)kshape.size(), kshape.data(),
                          psf.data(), 1, &plan));
  vk_status st = vk_rl_run_device(plan, d_obs->p, d_est.p, &rule, args.flat_init, &tr, s);
  vk_rl_plan_destroy(plan);
  check(st);
  cuda(cudaStreamSynchronize(s), "deconvolve");

  mkdirs(args.out_dir);
  check(vk_volume_write_device((args.out_dir + "/estimate.ndiv").c_str(), &obs_info, d_est.p, s));
  {
    auto out = open_out(args.out_dir + "/trace.csv");
    out << "iter,metric,value,wall_time_s\n";
    for (int i = 0; i < tr.iters_run; ++i) {
      out << (i + 1) << "," << kMetricName[metric] << ",";
      if (std::isinf(mv[i]))
        out << (mv[i] > 0 ? "inf" : "-inf");
      else
        out << mv[i];
      out << "," << ws[i] << "\n";
    }
  }
  {
    // summary.json as nlohmann's dump(2): sorted keys, 2-space indent
    std::vector<std::pair<std::string, std::string>> kv;
    kv.push_back({"backend", jstr(args.backend == "accelerated" ? "accelerated" : "reference")});
    std::string fs = "[";
    for (size_t a = 0; a < shape.size(); ++a) fs += std::string(a ? "," : "") + "\n    " + std::to_string(tr.fft_shape[a]);
    fs += "\n  ]";
    kv.push_back({"fft_shape", fs});
    const double fm = tr.iters_run ? mv[tr.iters_run - 1] : 0.0;
    kv.push_back({"final_metric", std::isinf(fm) ? jstr(fm > 0 ? "inf" : "-inf") : jnum(fm)});
    kv.push_back({"iters_run", std::to_string(tr.iters_run)});
    kv.push_back({"metric", jstr(kMetricName[metric])});
    kv.push_back({"schema", "1"});
    if (have_truth) {
      std::vector<float> h_obs(n), h_truth(n), h_est(n);
      cuda(cudaMemcpy(h_obs.data(), d_obs->p, n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
      cuda(cudaMemcpy(h_truth.data(), d_truth->p, n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
      cuda(cudaMemcpy(h_est.data(), d_est.p, n * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
      kv.push_back({"si_psnr_blurred_vs_truth", jnum(si_psnr(h_obs, h_truth))});
      kv.push_back({"si_psnr_estimate_vs_truth", jnum(si_psnr(h_est, h_truth))});
    }
    kv.push_back({"stop_reason", jstr(tr.stop_reason == 1 ? "converged" : "max_iters")});
    auto out = open_out(args.out_dir + "/summary.json");
    out << "{\n";
    for (size_t i = 0; i < kv.size(); ++i)
      out << "  " << jstr(kv[i].first) << ": " << kv[i].second << (i + 1 < kv.size() ? ",\n" : "\n");
    out << "}\n";
  }
  std::cout << "stopped after " << tr.iters_run << " iterations ("
            << (tr.stop_reason == 1 ? "converged" : "max_iters") << ")\n";
  delete d_obs;
  delete d_truth;
  cudaStreamDestroy(s);
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  const Args args = parse(argc, argv);
  try {
    return run(args);
  } catch (const CliError& e) {
    std::cerr << "error: " << e.msg << "\n";
    return exit_code(e.status);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kBadStructure;
  }
}
