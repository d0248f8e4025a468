// On-device stopping metric: single-image Fourier ring/shell correlation.
//
// The reference's default StoppingRule metric is frc_resolution
// (include/voxelkit/deconv.hpp:36), evaluated every iteration on the f32 crop
// of the estimate as metrics::single_image_frc(even_view(current), spacing)
// (src/deconv.cpp:285-289, src/metrics.cpp:146-264):
//   * even_view trims a trailing odd voxel per axis;
//   * the image splits into two half-size sub-images on the (0,0,0) and
//     (1,1,1) checkerboard diagonals;
//   * both get an r2c FFT; per integer-radius ring j of width 1/n_max
//     (n_max = the largest half extent), num = sum w Re(A conj B),
//     den_a = sum w |A|^2, den_b = sum w |B|^2 with w = 2 for kx planes that
//     stand for a conjugate pair (1 for kx = 0 and the even-length Nyquist);
//   * correlation = num / sqrt(den_a den_b); the first crossing of 1/7 above
//     DC (linear interpolation) gives the resolution spacing*2 / nu.
// Here the split reads the P-domain estimate directly, the two spectra come
// from a sub-plan's r2c passes (the same kernels as the OTF build), and the
// ring sums are block-reduced in shared memory then added with FP64 atomics.
// Only the final curve walk (a few hundred bins) runs on the host.
#pragma once
#include <math_constants.h>
#include "rl_passes.cuh"

namespace vk {

// est: P-domain estimate; the crop starts at (oz, oy, ox).  h*: half extents
// (1 for absent axes), s*: 1 where the axis exists (checkerboard shift).
__global__ void frc_split_kernel(const float* __restrict__ est, Geom g, int hz, int hy, int hx, int sz, int sy,
                                 int sx, float* __restrict__ even, float* __restrict__ odd) {
  const size_t n = (size_t)hz * hy * hx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % hx);
    const size_t t = i / hx;
    const int y = (int)(t % hy), z = (int)(t / hy);
    const int ze = (sz ? 2 * z : 0) + g.oz, ye = (sy ? 2 * y : 0) + g.oy, xe = (sx ? 2 * x : 0) + g.ox;
    even[i] = est[((size_t)ze * g.Py + ye) * g.Px + xe];
    odd[i] = est[((size_t)(ze + sz) * g.Py + (ye + sy)) * g.Px + (xe + sx)];
  }
}

// Ring sums over two half spectra laid out [Hx][Wz][Wy] (OTF layout).
// bins: [3][nbins] = num, den_a, den_b.  Shared scratch: 3*nbins doubles.
// A warp takes 32 consecutive elements (consecutive ky of one (kx, kz) row),
// whose ring indices form runs; a segmented shuffle scan sums each run and
// only its last lane adds to the shared histogram (FP64 shared atomics with
// 32-way contention were the kernel's cost).
// The ring index llround(nu / bin_freq) is first estimated in f32 (error
// < 1e-4 of a ring); only values within 1e-3 of a half-integer are redone in
// double exactly as the reference computes them.  Each block writes its
// histogram to partial[blockIdx.x]; frc_bins_reduce adds the blocks in a
// fixed order (deterministic sums).
// slices: histogram copies in shared memory (warp w uses slice w % slices),
// one per warp when they fit, to keep warps off each other's bins.
__global__ void frc_bins_kernel(const float2* __restrict__ A, const float2* __restrict__ B, int Wz, int Wy, int Wx,
                                int Hx, double bin_freq, int nbins, double* __restrict__ partial, int slices) {
  extern __shared__ double hist[];  // [slices][3][nbins]
  const int nw = slices;
  for (int i = threadIdx.x; i < 3 * nbins * nw; i += blockDim.x) hist[i] = 0.0;
  __syncthreads();
  double* wh = hist + (size_t)((threadIdx.x >> 5) % slices) * 3 * nbins;
  // work item = 32 consecutive ky of one (kx, kz) row: one division per item
  const int cpr = (Wy + 31) / 32;
  const int nitems = Hx * Wz * cpr;  // < 2^31 (checked by the host)
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
  const unsigned full = 0xffffffffu;
  const float rz = 1.0f / Wz, ry = 1.0f / Wy, rx = 1.0f / Wx, rb = (float)(1.0 / bin_freq);
  for (int item = warp; item < nitems; item += nwarps) {
    const int row = item / cpr, ky = (item - row * cpr) * 32 + lane;
    const int kx = row / Wz, kz = row - kx * Wz;
    const size_t i = (size_t)row * Wy + ky;
    int bin = -1;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    if (ky < Wy) {
      const int mz = min(kz, Wz - kz), my = min(ky, Wy - ky), mx = min(kx, Wx - kx);
      const float gz = mz * rz, gy = my * ry, gx = mx * rx;
      const float xf = sqrtf(gz * gz + gy * gy + gx * gx) * rb;
      long long b = (long long)(xf + 0.5f);
      if (fabsf(xf - floorf(xf) - 0.5f) < 1e-3f) {  // near a tie: the reference's double path
        const double fz = (double)mz / Wz, fy = (double)my / Wy, fx = (double)mx / Wx;
        b = llround(sqrt(fz * fz + fy * fy + fx * fx) / bin_freq);  // metrics.cpp:186-187
      }
      if (b < nbins) {
        bin = (int)b;
        const bool selfc = kx == 0 || ((Wx % 2 == 0) && 2 * kx == Wx);
        const double w = selfc ? 1.0 : 2.0;
        const float2 a = A[i], c = B[i];
        v0 = w * ((double)a.x * c.x + (double)a.y * c.y);
        v1 = w * ((double)a.x * a.x + (double)a.y * a.y);
        v2 = w * ((double)c.x * c.x + (double)c.y * c.y);
      }
    }
    // runs of equal ring index -> segment ids
    const int prevb = __shfl_up_sync(full, bin, 1);
    const unsigned heads = __ballot_sync(full, lane == 0 || prevb != bin);
    const int seg = __popc(heads & (lane == 31 ? full : ((2u << lane) - 1u)));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double u0 = __shfl_up_sync(full, v0, o), u1 = __shfl_up_sync(full, v1, o),
                   u2 = __shfl_up_sync(full, v2, o);
      const int s = __shfl_up_sync(full, seg, o);
      if (lane >= o && s == seg) {
        v0 += u0;
        v1 += u1;
        v2 += u2;
      }
    }
    const int nextseg = __shfl_down_sync(full, seg, 1);
    if (bin >= 0 && (lane == 31 || nextseg != seg)) {  // run tails: distinct bins except across the ky fold
      atomicAdd(&wh[bin], v0);
      atomicAdd(&wh[nbins + bin], v1);
      atomicAdd(&wh[2 * nbins + bin], v2);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * nbins; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += hist[(size_t)w * 3 * nbins + i];
    partial[(size_t)blockIdx.x * 3 * nbins + i] = s;
  }
}

// One CTA per value: strided per-thread sums then a fixed-shape tree.
__global__ void frc_bins_reduce(const double* __restrict__ partial, int nblocks, int nvals, double* __restrict__ bins) {
  __shared__ double red[256];
  const int i = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[(size_t)b * nvals + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) bins[i] = red[0];
}

// Direct DFT along one axis, for FRC half extents that are not 5-smooth (the
// reference's FFTW plans any length; the line FFTs here are radix 2/3/5).
// Logical output coordinates (c0, c1, c2) over extents (e0, e1, e2); axis
// `ax` sums n input samples with the exact twiddle tw[(j k) mod n] =
// exp(-2 pi i (j k mod n) / n).  Strides in elements; REAL_IN reads floats.
// Cost n per output: a fallback, used only where the FFT path cannot run.
template <bool REAL_IN>
__global__ void dft_axis_kernel(const void* __restrict__ in, float2* __restrict__ out, int e0, int e1, int e2,
                                int ax, int n, long long is0, long long is1, long long is2, long long os0,
                                long long os1, long long os2, const float2* __restrict__ tw) {
  const size_t total = (size_t)e0 * e1 * e2;
  const long long isa = ax == 0 ? is0 : ax == 1 ? is1 : is2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    int c[3];
    c[2] = (int)(i % e2);
    const size_t t = i / e2;
    c[1] = (int)(t % e1);
    c[0] = (int)(t / e1);
    const int k = c[ax];
    c[ax] = 0;
    const long long base = c[0] * is0 + c[1] * is1 + c[2] * is2;
    c[ax] = k;
    float re = 0.f, im = 0.f;
    int m = 0;
    for (int j = 0; j < n; ++j) {
      const float2 w = tw[m];
      if (REAL_IN) {
        const float v = static_cast<const float*>(in)[base + j * isa];
        re = fmaf(v, w.x, re);
        im = fmaf(v, w.y, im);
      } else {
        const float2 v = static_cast<const float2*>(in)[base + j * isa];
        re = fmaf(v.x, w.x, fmaf(-v.y, w.y, re));
        im = fmaf(v.x, w.y, fmaf(v.y, w.x, im));
      }
      m += k;
      if (m >= n) m -= n;
    }
    out[c[0] * os0 + c[1] * os1 + c[2] * os2] = make_float2(re, im);
  }
}

// ---------------------------------------------------------------------------
// ssim_vs_prev: metrics::ssim(current, previous) (src/metrics.cpp:103-144)
// with filters::gaussian(sigma 1.5, truncate 3.5) (src/filters.cpp:78-140).
// Five moments (x, r, x^2, r^2, x r; the squares and product in f32 as
// metrics.cpp:121-125 forms them) are smoothed by one separable 13-tap pass
// per image axis with mirror boundary (nd_utils.hpp:31-38).  Like the
// reference the passes accumulate in double, in tap order, with every product
// and sum rounded separately (no FMA contraction), and keep double between
// passes; the last pass rounds the five moments to f32 (filters.cpp:135-138)
// and folds the SSIM map and its sum into the same kernel.  The moments stay
// in HBM between passes: 40 B per voxel and field pair per pass.
// ---------------------------------------------------------------------------

constexpr int kSsimHalf = 6;  // ceil(3.5 * 1.5)
struct SsimTaps {
  double w[2 * kSsimHalf + 1];
};

// Crop the P-domain estimate into `cur` and record its [min, max] as f32 bits
// (values are >= 0; -0 is ordered as +0) for the next iteration's range.
__global__ void crop_range_kernel(const float* __restrict__ est, float* __restrict__ out, Geom g,
                                  unsigned int* __restrict__ range) {
  const size_t n = (size_t)g.Iz * g.Iy * g.Ix;
  unsigned int mn = 0x7f800000u, mx = 0u;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.Ix);
    const size_t t = i / g.Ix;
    const int y = (int)(t % g.Iy), z = (int)(t / g.Iy);
    const float v = est[((size_t)(z + g.oz) * g.Py + (y + g.oy)) * g.Px + (x + g.ox)];
    out[i] = v;
    const unsigned int b = v == 0.f ? 0u : __float_as_uint(v);
    mn = min(mn, b);
    mx = max(mx, b);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&range[0], mn);
    atomicMax(&range[1], mx);
  }
}

__device__ __forceinline__ int ssim_mirror(int i, int n) {  // |offset| <= 6 < n
  if (i < 0) return -i;
  if (i >= n) return 2 * (n - 1) - i;
  return i;
}

// One smoothing pass along an axis of extent `ext` and element stride
// `stride`.  FIRST: the moments come from (xc, rp); otherwise from `in`
// (5 fields of n doubles).  LAST: no store; the SSIM map is summed into *sum
// with c1, c2 from the previous image's range (range[0..1] = f32 bits).
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(256) ssim_axis_kernel(const float* __restrict__ xc, const float* __restrict__ rp,
                                                        const double* __restrict__ in, double* __restrict__ out,
                                                        size_t n, int ext, size_t stride, SsimTaps t,
                                                        const unsigned int* __restrict__ range,
                                                        double* __restrict__ sum) {
  double c1 = 0, c2 = 0;
  if (LAST) {
    const double r = (double)__uint_as_float(range[1]) - (double)__uint_as_float(range[0]);
    c1 = __dmul_rn(__dmul_rn(0.01, r), __dmul_rn(0.01, r));
    c2 = __dmul_rn(__dmul_rn(0.03, r), __dmul_rn(0.03, r));
  }
  double part = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int c = (int)((i / stride) % (size_t)ext);
    const size_t base = i - (size_t)c * stride;
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = -kSsimHalf; k <= kSsimHalf; ++k) {
      const size_t j = base + (size_t)ssim_mirror(c + k, ext) * stride;
      const double w = t.w[k + kSsimHalf];
      double v[5];
      if (FIRST) {
        const float a = xc[j], b = rp[j];
        v[0] = a;
        v[1] = b;
        v[2] = __fmul_rn(a, a);
        v[3] = __fmul_rn(b, b);
        v[4] = __fmul_rn(a, b);
      } else {
#pragma unroll
        for (int f = 0; f < 5; ++f) v[f] = in[f * n + j];
      }
#pragma unroll
      for (int f = 0; f < 5; ++f) acc[f] = __dadd_rn(acc[f], __dmul_rn(w, v[f]));
    }
    if (!LAST) {
#pragma unroll
      for (int f = 0; f < 5; ++f) out[f * n + i] = acc[f];
    } else {
      // metrics.cpp:133-142 on the f32-rounded moments
      const double mx = (float)acc[0], mr = (float)acc[1];
      const double mxx = (float)acc[2], mrr = (float)acc[3], mxr = (float)acc[4];
      const double var_x = __dsub_rn(mxx, __dmul_rn(mx, mx));
      const double var_r = __dsub_rn(mrr, __dmul_rn(mr, mr));
      const double cov = __dsub_rn(mxr, __dmul_rn(mx, mr));
      const double num = __dmul_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mx), mr), c1),
                                   __dadd_rn(__dmul_rn(2.0, cov), c2));
      const double den = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(mx, mx), __dmul_rn(mr, mr)), c1),
                                   __dadd_rn(__dadd_rn(var_x, var_r), c2));
      part += __ddiv_rn(num, den);
    }
  }
  if (LAST) {  // block partials [gridDim.x] in `sum`, reduced in a fixed order by the caller
    double v1[1] = {part};
    block_partial<1>(v1, sum + blockIdx.x);
  }
}

}  // namespace vk

namespace vk {

// ---- device-side stopping rule (CUDA-graph while loop, vk_rl.cu run_graph) ----
// The iteration body is one graph; this kernel, its last node, evaluates the
// stopping rule of deconv.cpp:401-423 on the device and sets the while
// node's condition, so a run that may stop early never syncs the host per
// iteration.
struct StopState {
  int it;       // iterations completed
  int fails;    // consecutive changes below rel_tol
  int stopped;  // the rule fired ("converged")
  int pad;
  double prev;  // metric of the previous iteration
};

struct RuleArgs {
  StopState* st;
  double* values;         // [iters] metric per iteration
  unsigned long long* ts; // [iters + 1] %globaltimer at iteration ends (ts[0] = start)
  const double* xpart;    // x-pass block partials of this iteration [nblocks][4] (si_psnr)
  int nblocks;
  double* acc;            // [iters][4]: LL, sum x, sum x^2, sum x r
  const ObsStats* obs;    // reference statistics of the observed image
  double n_img;
  const double* metric_in;  // ssim: SSIM-map sum (divided by n_img); frc: the resolution
  int metric;             // vk_stop_metric
  double rel_tol;
  int patience, iters;
  cudaGraphConditionalHandle handle;
};

__device__ __forceinline__ double rel_change_dev(double prev, double cur) {  // deconv.cpp:296-300
  if (isinf(prev) && isinf(cur) && prev == cur) return 0.0;
  if (isinf(prev) || isinf(cur)) return CUDART_INF;
  return fabs(cur - prev) / fmax(fabs(prev), 1e-30);
}

// si_psnr from the fused sums (metrics.cpp:67-101; host twin si_psnr_from_sums)
__device__ __forceinline__ double si_psnr_dev(const ObsStats& o, double n, double sx, double sxx, double sxr) {
  const double var_r = o.srr / n - (o.sr / n) * (o.sr / n);
  const double var_x = sxx / n - (sx / n) * (sx / n);
  const double cov = sxr / n - (sx / n) * (o.sr / n);
  const double a = var_x > 0.0 ? cov / var_x : 0.0;
  const double err = var_r - a * cov;
  if (err <= 0.0) return CUDART_INF;
  const double range = (double)__uint_as_float(o.maxbits) - (double)__uint_as_float(o.minbits);
  return 10.0 * log10(range * range / err);
}

__global__ void __launch_bounds__(256) rule_step_kernel(RuleArgs a) {
  const int k = a.st->it;  // 0-based index of the iteration just completed
  for (int v = 0; v < 4; ++v) {  // this iteration's x-pass sums (LL; si_psnr sums), fixed order
    const double s = block_sum_fixed(a.nblocks, [&](int b) { return a.xpart[(size_t)b * 4 + v]; });
    if (threadIdx.x == 0) a.acc[(size_t)k * 4 + v] = s;
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  double value;
  if (a.metric == 0) {
    const double* s = a.acc + (size_t)k * 4;
    value = si_psnr_dev(*a.obs, a.n_img, s[1], s[2], s[3]);
  } else if (a.metric == 1) {  // VK_METRIC_SSIM_VS_PREV
    value = a.metric_in[0] / a.n_img;
  } else {  // VK_METRIC_FRC_RESOLUTION
    value = a.metric_in[0];
  }
  a.values[k] = value;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  a.ts[k + 1] = t;
  StopState st = *a.st;
  if (k > 0) {
    st.fails = rel_change_dev(st.prev, value) < a.rel_tol ? st.fails + 1 : 0;
    if (st.fails >= a.patience) st.stopped = 1;
  }
  st.prev = value;
  st.it = k + 1;
  *a.st = st;
  cudaGraphSetConditional(a.handle, (!st.stopped && st.it < a.iters) ? 1u : 0u);
}

__global__ void timestamp_kernel(unsigned long long* ts) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *ts = t;
}

// frc_resolution of the ring sums (metrics.cpp:146-239; host twin frc_eval):
// first ring below 1/7 (DC excluded), linear interpolation, 2*spacing / nu.
__global__ void frc_value_kernel(const double* __restrict__ bins, int nb, double binf, double spacing,
                                 double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* num = bins;
  const double* da = bins + nb;
  const double* db = bins + 2 * nb;
  auto corr = [&](int j) {
    const double den = sqrt(da[j] * db[j]);
    return den > 0 ? num[j] / den : 0.0;
  };
  const double threshold = 1.0 / 7.0, sp = spacing * 2.0;
  double res = CUDART_INF;  // kUnresolved
  for (int j = 1; j < nb; ++j) {
    if (corr(j) < threshold) {
      double nu;
      if (j == 1 || corr(j - 1) < threshold) {
        nu = j * binf;
      } else {
        const double c0 = corr(j - 1), c1 = corr(j);
        const double f0 = (j - 1) * binf, f1 = j * binf;
        nu = f0 + (f1 - f0) * (c0 - threshold) / (c0 - c1);
      }
      res = nu <= 0 ? CUDART_INF : sp / nu;
      break;
    }
  }
  *out = res;
}

}  // namespace vk
