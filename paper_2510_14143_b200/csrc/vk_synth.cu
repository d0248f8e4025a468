// Synthetic inputs of the reference CLI's `deconvolve` (SURVEY.md §8(f) row
// f2) behind include/vk_io.h:
//   generate_blobs  (/root/reference/proj/src/synth.cpp:199-224, placement
//                    :64-123, rasterisation :127-148, soft edge :169-175,
//                    noise :177-180, RNG :33-59)
//   gaussian_psf    (src/synth.cpp:226-258)
//
// The RNG is std::mt19937_64 with hand-rolled draws (uniform01 = top 53
// bits * 2^-53; Box-Muller normals in cos/sin pairs, the sine kept as the
// next draw).  Placement is sequential rejection sampling and stays on the
// host.  The voxel work moves to the GPU: one CTA per object rasterises its
// bounding box with an order-free max (atomicMax on the f32 bits of values
// in [0, 1]), and the noise pass turns host-drawn raw 64-bit pairs into
// normals on the device, chunked through pinned memory so drawing chunk k+1
// overlaps the transfer and transform of chunk k.  Device arithmetic keeps
// the reference's operation order with contraction disabled (__d*_rn);
// CUDA's double log/sin/cos may differ from glibc's in the last ulp, which
// the f32 cast absorbs except at rare rounding ties.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/vk_io.h"

namespace vk {
void set_last_error(const std::string& msg);
}

namespace {

struct SynFail {
  vk_status code;
  std::string msg;
};
[[noreturn]] void syn_fail(vk_status c, std::string m) { throw SynFail{c, std::move(m)}; }

template <class F>
vk_status syn_guard(F&& f) {
  try {
    f();
    return VK_OK;
  } catch (const SynFail& e) {
    vk::set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    vk::set_last_error("host allocation failed");
    return VK_ERR_OOM;
  } catch (const std::exception& e) {
    vk::set_last_error(e.what());
    return VK_ERR_ARG;
  }
}

void cuda_ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  syn_fail(e == cudaErrorMemoryAllocation ? VK_ERR_OOM : VK_ERR_CUDA,
           std::string(what) + ": " + cudaGetErrorString(e));
}

constexpr double kPi = 3.14159265358979323846;

// The reference's draw sequence over mt19937_64 (synth.cpp:33-59).
struct Stream {
  std::mt19937_64 gen;
  explicit Stream(uint64_t seed) : gen(seed) {}
  double uniform01() { return (double)(gen() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform01(); }
};

struct Object {
  double c[3];     // centre z, y, x
  double semi[3];  // semi-axes z, y, x
  double radius;
  int lo[3], hi[3];  // rasterisation box (inclusive)
};

// Rejection placement (synth.cpp:64-123); throws PlacementFailure / Error
// with the reference's messages.
std::vector<Object> place(const vk_synth_spec& sp, Stream& rng) {
  if (!(sp.radius_min > 0) || sp.radius_max < sp.radius_min)
    syn_fail(VK_ERR_ARG, "radius range must be positive and ordered");
  if (!(sp.anisotropy > 0)) syn_fail(VK_ERR_ARG, "anisotropy must be positive");
  std::vector<Object> objs;
  objs.reserve(sp.n_objects);
  for (uint64_t i = 0; i < sp.n_objects; ++i) {
    bool placed = false;
    for (int attempt = 0; attempt < 200 && !placed; ++attempt) {
      Object o{};
      o.radius = rng.uniform(sp.radius_min, sp.radius_max);
      o.semi[0] = o.radius / sp.anisotropy;
      o.semi[1] = o.semi[2] = o.radius;
      for (int a = 0; a < 3; ++a) {
        const double margin = o.semi[a] + 3.0 + (a > 0 ? sp.inplane_margin : 0.0);
        const double top = (double)sp.shape[a] - 1.0 - margin;
        if (top < margin) syn_fail(VK_ERR_PLACEMENT, "PlacementFailure: objects of this size cannot fit the volume");
        o.c[a] = rng.uniform(margin, top);
      }
      const double reach = std::max(o.semi[0], o.radius) + 1.0;
      bool clash = false;
      for (const Object& q : objs) {
        const double min_d = reach + (std::max(q.semi[0], q.radius) + 1.0) + 2.0;
        double d2 = 0;
        for (int a = 0; a < 3; ++a) {
          const double d = o.c[a] - q.c[a];
          d2 += d * d;
        }
        if (d2 < min_d * min_d) {
          clash = true;
          break;
        }
      }
      if (!clash) {
        objs.push_back(o);
        placed = true;
      }
    }
    if (!placed)
      syn_fail(VK_ERR_PLACEMENT,
               "PlacementFailure: could not place object " + std::to_string(i + 1) + " without overlap");
  }
  for (Object& o : objs) {  // rasterize() box with extent 1 + 1/radius (synth.cpp:131-139)
    const double ext = 1.0 + 1.0 / o.radius;
    for (int a = 0; a < 3; ++a) {
      o.lo[a] = (int)std::max<long>(0, (long)std::floor(o.c[a] - o.semi[a] * ext - 1));
      o.hi[a] = (int)std::min<long>((long)sp.shape[a] - 1, (long)std::ceil(o.c[a] + o.semi[a] * ext + 1));
    }
  }
  return objs;
}

// One CTA per object: soft-edged ellipsoid max-combined into img (>= 0).
__global__ void raster_kernel(const Object* __restrict__ objs, int ny, int nx, unsigned* __restrict__ img) {
  const Object o = objs[blockIdx.x];
  const int bz = o.hi[0] - o.lo[0] + 1, by = o.hi[1] - o.lo[1] + 1, bx = o.hi[2] - o.lo[2] + 1;
  if (bz <= 0 || by <= 0 || bx <= 0) return;
  const double ext = __dadd_rn(1.0, __ddiv_rn(1.0, o.radius));
  const double half_band = __ddiv_rn(1.0, o.radius);
  const size_t n = (size_t)bz * by * bx;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int x = o.lo[2] + (int)(i % bx);
    const size_t t = i / bx;
    const int y = o.lo[1] + (int)(t % by), z = o.lo[0] + (int)(t / by);
    const double dz = __ddiv_rn(__dsub_rn((double)z, o.c[0]), o.semi[0]);
    const double dy = __ddiv_rn(__dsub_rn((double)y, o.c[1]), o.semi[1]);
    const double dx = __ddiv_rn(__dsub_rn((double)x, o.c[2]), o.semi[2]);
    const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dz, dz), __dmul_rn(dy, dy)), __dmul_rn(dx, dx)));
    if (r > ext) continue;
    double v;  // soft_profile (synth.cpp:169-175)
    if (r <= __dsub_rn(1.0, half_band)) {
      v = 1.0;
    } else if (r >= __dadd_rn(1.0, half_band)) {
      v = 0.0;
    } else {
      const double arg = __ddiv_rn(__dmul_rn(kPi, __dsub_rn(r, __dsub_rn(1.0, half_band))), __dmul_rn(2.0, half_band));
      v = __dmul_rn(0.5, __dadd_rn(1.0, cos(arg)));
    }
    const float f = (float)v;
    if (f > 0.f) atomicMax(&img[((size_t)z * ny + y) * nx + x], __float_as_uint(f));
  }
}

// img[2j], img[2j+1] += f32(sigma * (mag cos, mag sin)) of raw pair j.
__global__ void noise_kernel(float* __restrict__ img, size_t first, size_t count, const uint64_t* __restrict__ raw,
                             double sigma) {
  const size_t pairs = (count + 1) / 2;
  for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < pairs; j += (size_t)gridDim.x * blockDim.x) {
    const double u1 = __dmul_rn((double)(raw[2 * j] >> 11), 0x1.0p-53);
    const double u2 = __dmul_rn((double)(raw[2 * j + 1] >> 11), 0x1.0p-53);
    const double mag = __dsqrt_rn(__dmul_rn(-2.0, log(u1)));
    const double ang = __dmul_rn(__dmul_rn(2.0, kPi), u2);
    double sn, cs;
    sincos(ang, &sn, &cs);
    const size_t i = first + 2 * j;
    img[i] = __fadd_rn(img[i], (float)__dmul_rn(sigma, __dmul_rn(mag, cs)));
    if (2 * j + 1 < count) img[i + 1] = __fadd_rn(img[i + 1], (float)__dmul_rn(sigma, __dmul_rn(mag, sn)));
  }
}

}  // namespace

extern "C" {

vk_status vk_generate_blobs(int device, const vk_synth_spec* spec, float* d_out, double* spacing3, void* stream) {
  return syn_guard([&] {
    if (!spec || !d_out) syn_fail(VK_ERR_ARG, "NULL argument");
    int prev = 0;
    cudaGetDevice(&prev);
    cuda_ck(cudaSetDevice(device), "cudaSetDevice");
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{prev};
    const vk_synth_spec sp = *spec;
    Stream rng(sp.seed);
    const std::vector<Object> objs = place(sp, rng);
    const size_t n = (size_t)sp.shape[0] * sp.shape[1] * sp.shape[2];
    cudaStream_t s = (cudaStream_t)stream;
    cuda_ck(cudaMemsetAsync(d_out, 0, n * sizeof(float), s), "memset");
    if (!objs.empty()) {
      Object* d_objs = nullptr;
      cuda_ck(cudaMallocAsync((void**)&d_objs, objs.size() * sizeof(Object), s), "objects");
      cuda_ck(cudaMemcpyAsync(d_objs, objs.data(), objs.size() * sizeof(Object), cudaMemcpyHostToDevice, s), "H2D");
      raster_kernel<<<(unsigned)objs.size(), 256, 0, s>>>(d_objs, (int)sp.shape[1], (int)sp.shape[2],
                                                          reinterpret_cast<unsigned*>(d_out));
      cuda_ck(cudaGetLastError(), "raster");
      cuda_ck(cudaFreeAsync(d_objs, s), "free");
    }
    // noise_sigma scales the clean range, 1 with objects and 0 without
    // (synth.cpp:212-215); add_noise returns early for sigma <= 0.
    const double sigma = sp.noise_sigma * (objs.empty() ? 0.0 : 1.0);
    if (sigma > 0 && n > 0) {
      constexpr size_t kChunkVox = size_t(8) << 20;  // voxels per chunk (even)
      uint64_t* host[2] = {nullptr, nullptr};
      uint64_t* dev[2] = {nullptr, nullptr};
      cudaEvent_t done[2] = {nullptr, nullptr};
      struct Free {
        uint64_t** h;
        uint64_t** d;
        cudaEvent_t* e;
        ~Free() {
          for (int i = 0; i < 2; ++i) {
            if (e[i]) cudaEventSynchronize(e[i]), cudaEventDestroy(e[i]);
            if (h[i]) cudaFreeHost(h[i]);
            if (d[i]) cudaFree(d[i]);
          }
        }
      } guard{host, dev, done};
      const size_t chunk = std::min(kChunkVox, n + (n & 1));
      for (int i = 0; i < 2; ++i) {
        cuda_ck(cudaHostAlloc((void**)&host[i], chunk * sizeof(uint64_t), 0), "pinned noise");
        cuda_ck(cudaMalloc((void**)&dev[i], chunk * sizeof(uint64_t)), "noise raw");
        cuda_ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "event");
      }
      bool used[2] = {false, false};
      int k = 0;
      for (size_t first = 0; first < n; first += chunk) {
        const size_t count = std::min(chunk, n - first);
        if (used[k]) cuda_ck(cudaEventSynchronize(done[k]), "noise wait");
        uint64_t* h = host[k];
        for (size_t j = 0; j < (count + 1) / 2; ++j) {  // normal(): redraw u1 while it is 0
          uint64_t a = rng.gen();
          while ((a >> 11) == 0) a = rng.gen();
          h[2 * j] = a;
          h[2 * j + 1] = rng.gen();
        }
        const size_t words = 2 * ((count + 1) / 2);
        cuda_ck(cudaMemcpyAsync(dev[k], h, words * sizeof(uint64_t), cudaMemcpyHostToDevice, s), "H2D");
        noise_kernel<<<148 * 4, 256, 0, s>>>(d_out, first, count, dev[k], sigma);
        cuda_ck(cudaGetLastError(), "noise");
        cuda_ck(cudaEventRecord(done[k], s), "event");
        used[k] = true;
        k ^= 1;
      }
    }
    cuda_ck(cudaStreamSynchronize(s), "generate_blobs");
    if (spacing3) {
      spacing3[0] = sp.anisotropy;
      spacing3[1] = 1.0;
      spacing3[2] = 1.0;
    }
  });
}

vk_status vk_gaussian_psf(int rank, const uint64_t* shape, const double* sigmas, int nsig, float* out) {
  return syn_guard([&] {
    if (!shape || !sigmas || !out || rank < 1 || nsig < 1) syn_fail(VK_ERR_ARG, "NULL argument");
    std::vector<double> sg(sigmas, sigmas + nsig);
    if (sg.size() == 1 && rank > 1) sg.resize(rank, sg[0]);
    if ((int)sg.size() != rank) syn_fail(VK_ERR_SHAPE, "ShapeMismatch: gaussian_psf: one sigma per axis");
    std::string shp = "[";
    for (int a = 0; a < rank; ++a) shp += (a ? "," : "") + std::to_string(shape[a]);
    shp += "]";
    for (int a = 0; a < rank; ++a)
      if (shape[a] % 2 == 0) syn_fail(VK_ERR_EVEN_EXTENT, "EvenExtent: gaussian_psf needs odd extents, got " + shp);
    size_t n = 1;
    for (int a = 0; a < rank; ++a) n *= shape[a];
    std::vector<double> vals(n);
    std::vector<long> coord(rank, 0);
    double sum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      double v = 1.0;
      for (int a = 0; a < rank; ++a) {
        const double d = coord[a] - (double)(shape[a] / 2);
        if (sg[a] <= 0.0)
          v *= d == 0.0 ? 1.0 : 0.0;
        else
          v *= std::exp(-0.5 * (d / sg[a]) * (d / sg[a]));
      }
      vals[i] = v;
      sum += v;
      for (int a = rank - 1; a >= 0; --a) {  // row-major odometer
        if (++coord[a] < (long)shape[a]) break;
        coord[a] = 0;
      }
    }
    for (size_t i = 0; i < n; ++i) out[i] = (float)(vals[i] / sum);
  });
}

}  // extern "C"
