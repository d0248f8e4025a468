// Richardson-Lucy pass kernels for sm_100a.
//
// The reference iteration (proj/src/deconv.cpp:359-399) performs, per
// iteration, two 'same' linear convolutions on the padded domain P through a
// zero-padded FFT grid W (deconv.cpp:135-147), a ratio, and a clipped
// multiplicative update, with ~12 full host sweeps in double.  Here the
// iteration is a chain of device passes over a PRUNED complex64 spectrum:
//
//   S_A [Hx][Pz][Py]   x-transformed rows, transposed so every (kx) plane is
//                      contiguous (Hx = Wx/2+1).  Only the Pz*Py rows that carry
//                      data exist: rows outside P are zero before the forward
//                      transform and cropped away after the inverse.
//   S_B [Hx][Pz][Wy]   after the y transform (3D only).
//   OTF [Hx][Wz][Wy]   PSF spectrum, 1/prod(W) folded in (fft_plan.cpp:95-96).
//
// Passes (3D):  X-pass (C2R -> pointwise epilogue -> R2C)  ->  Y fwd  ->
//               Z (fwd * OTF * inv, crop)  ->  Y inv (crop)  -> next X-pass.
// 2D/1D problems are the 3D code with unit leading extents; there the Y pass
// carries the OTF multiply (Y fwd * OTF * Y inv) and the Z pass vanishes.
//
// X-pass epilogues (fused, so no intermediate real field ever hits HBM):
//   RATIO : model -> ratio = obs_p / max(model, 1e-12) over all of P
//           (deconv.cpp:382-390), Poisson log-likelihood over the interior in
//           FP64 (deconv.cpp:364-379), R2C of the ratio.
//   UPDATE: corr -> est = max(est*corr, 0) (deconv.cpp:393-398), si_psnr
//           partial sums of the f32 crop (metrics.cpp:67-101), R2C of est, or
//           on the last iteration the cropped f32 output (deconv.cpp:239-252).
// Observed values are read clamp-indexed from the UNPADDED image, which is the
// reference's edge-replicate padding (deconv.cpp:221-237) without storing it.
#pragma once
#include "fft_core.cuh"

namespace vk {

constexpr float kEps = 1e-12f;  // kDivEpsilon, include/voxelkit/core_ops.hpp:26

// XM_CONV_OUT (generic kernel only): C2R and store of the cropped result,
// for filters::fft_convolve plans.
enum XMode : int { XM_FWD = 0, XM_RATIO = 1, XM_UPDATE = 2, XM_UPDATE_LAST = 3, XM_CONV_OUT = 4 };
enum YMode : int { YM_FWD = 0, YM_INV = 1, YM_CONV = 2 };
enum ZMode : int { ZM_CONV = 0, ZM_FWD_OUT = 1 };

struct Geom {
  int Iz, Iy, Ix;  // image
  int Pz, Py, Px;  // iteration domain
  int oz, oy, ox;  // image offset inside P (floor(K/2) or 0)
  int Wz, Wy, Wx, Hx;
  int cz, cy, cx;  // crop offset (K-1)/2
};

struct XArgs {
  LinePlan plan;
  Geom g;
  int mode;
  int L;
  int rows_y;           // rows per z plane in this pass (Py, or Ky for the PSF)
  int rows_z;
  int len;              // valid samples per row before the transform (Px or Kx)
  float2* S;            // [Hx][rows_z][rows_y]
  const float* src;     // FWD: real rows [rows_z][rows_y][len]
  float scale;          // FWD: input scale
  int xoff;             // FWD: slot of sample 0 in the line (fast path: cx, PSF: 0)
  float* est;           // UPDATE: [Pz][Py][Px]
  const float* obs;     // [Iz][Iy][Ix]
  double* acc;          // this iteration's partials [blocks][4]: RATIO [0] = LL, UPDATE [1..3] = sx, sxx, sxr
  float* out;           // UPDATE_LAST: cropped f32 estimate [Iz][Iy][Ix]
  int zoff;             // first z row of this launch (z-chunked iterations)
  int pf;               // fast path: L2 prefetch of the CTA's inputs at entry (1 spectrum, 2 rows)
  int tbk, tnb;         // xpass_tma: kx per TMA box, boxes per CTA
};

struct YArgs {
  LinePlan plan;
  int mode;
  int L;
  int nlines;
  int n_in, in_pitch;
  int n_out, out_pitch, out_off;
  const float2* in;
  float2* out;
  const float2* otf;    // CONV: otf[line * N + k]
  // z-chunked passes (zcn > 0): the nlines = Hx * zcn lines are (kx, z) with
  // z in [zc0, zc0 + zcn) of zrows rows per kx plane
  int zc0, zcn, zrows;
  int bst;  // ypass_tma FWD: bulk-store each output line (16-byte aligned lines only)
  // ypass_tma CONV (2D) with a separable OTF: fx[Hx], fy[Wy], fz[1] back to
  // back (factor_otfs), O(kx, ky) = (fx[kx] * fy[ky]) * fz[0]; nullptr: read otf
  const float2* ofac;
  int ohx;
};

// Global line of a pass-local line index (identity unless z-chunked).
__device__ __forceinline__ int y_line(const YArgs& a, int local) {
  if (a.zcn == 0) return local;
  const int kx = local / a.zcn;
  return kx * a.zrows + a.zc0 + (local - kx * a.zcn);
}

struct ZArgs {
  LinePlan plan;
  int mode;
  int L;
  int Wy;               // row length (ky extent)
  int zrows;            // stored z rows per kx plane in S
  int n_in;             // valid z rows
  int n_out, out_off;   // CONV: rows written back
  float2* S;            // [Hx][zrows][Wy]
  const float2* otf;    // [Hx][Wz][Wy]
  float2* otf_out;      // FWD_OUT: [Hx][Wz][Wy]
  int hx;               // number of kx planes (persistent kernels)
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Interleaved line pitch of the generic kernels: L + 1 (conflict-free
// transposed staging), except one line per CTA (long lines), which needs no
// pad -- that halves the shared memory of the longest lines, so the generic
// path plans axes up to ~14k points (the paper's own volume, W = 90 x 6480 x
// 7680 with a PSF as large as the image).
__host__ __device__ __forceinline__ int line_pitch(int L) { return L == 1 ? 1 : L + 1; }

// Deterministic sums.  Every block writes its N partial sums (a fixed
// shuffle tree, then warp 0 over the warps in order) to dst[0..N) -- no
// atomics -- and reduce_partials_kernel / reduce_iter_partials_kernel add the
// partials of all blocks in a fixed order.  Trace values, the flat_init mean
// and the stopping decisions are then bitwise reproducible run to run (the
// reference's sums are serial, deconv.cpp:364-379, metrics.cpp:67-101).
template <int N>
__device__ __forceinline__ void block_partial(double (&v)[N], double* dst) {
  __shared__ double red[32][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) red[w][i] = v[i];
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = lane < nw ? red[lane][i] : 0.0;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) dst[i] = s;
    }
  }
}

// Sum of n values in a fixed order by one 256-thread block: strided serial
// sums per thread, then a fixed tree.  get(i) returns value i.
template <class F>
__device__ __forceinline__ double block_sum_fixed(int n, F&& get) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += get(i);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  return red[0];
}

#ifndef VK_NO_GENERIC_KERNELS  // generic (runtime-length) kernels: defined once, in vk_rl.cu

// out[k] = sum over blocks b of part[b * stride + k], k = blockIdx.x.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ part, int nblocks, int stride,
                                                             double* __restrict__ out) {
  const int k = blockIdx.x;
  const double s = block_sum_fixed(nblocks, [&](int b) { return part[(size_t)b * stride + k]; });
  if (threadIdx.x == 0) out[k] = s;
}

// Per-iteration x-pass sums: iterations it0 .. it0 + gridDim.x/4 - 1
// (0-based) live in ring slot it % ring as [nblocks][4]; acc[it][k] = sum.
__global__ void __launch_bounds__(256) reduce_iter_partials_kernel(const double* __restrict__ part, int nblocks,
                                                                  int ring, int it0, double* __restrict__ acc) {
  const int it = it0 + (int)blockIdx.x / 4, k = blockIdx.x % 4;
  const double* base = part + (size_t)(it % ring) * nblocks * 4;
  const double s = block_sum_fixed(nblocks, [&](int b) { return base[(size_t)b * 4 + k]; });
  if (threadIdx.x == 0) acc[(size_t)it * 4 + k] = s;
}


// Forward R2C of the 2L real rows packed in `in` (line l = rows l and L+l) and
// store of both Hermitian halves into S.
__device__ __forceinline__ void x_forward_store(float2* in, float2* tmp, const XArgs& a, int LP, int z,
                                                int y0) {
  const int L = a.L, Wx = a.g.Wx, Hx = a.g.Hx;
  float2* R = fft_lines<false>(in, tmp, L, LP, a.plan);
  for (int idx = threadIdx.x; idx < Hx * L; idx += blockDim.x) {
    const int kx = idx / L, l = idx - kx * L;
    const float2 zk = R[kx * LP + l];
    const float2 zn = R[(kx == 0 ? 0 : Wx - kx) * LP + l];
    const float2 xa = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
    const float2 xb = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
    const size_t row = ((size_t)kx * a.rows_z + z) * a.rows_y;
    if (y0 + l < a.rows_y) a.S[row + y0 + l] = xa;
    if (y0 + L + l < a.rows_y) a.S[row + y0 + L + l] = xb;
  }
}

__global__ void __launch_bounds__(256) xpass_kernel(const XArgs a) {
  extern __shared__ float2 smem[];
  const int L = a.L, LP = line_pitch(L), Wx = a.g.Wx, Hx = a.g.Hx;
  float2* A = smem;
  float2* B = smem + Wx * LP;  // B also stages Hx*2L (host sizes it as max of both)
  const int z = blockIdx.y + a.zoff;
  const int y0 = blockIdx.x * 2 * L;

  if (a.mode == XM_FWD) {
    for (int idx = threadIdx.x; idx < 2 * L * Wx; idx += blockDim.x) {
      const int r = idx / Wx, x = idx - r * Wx;
      const int y = y0 + r;
      float v = 0.f;
      if (x < a.len && y < a.rows_y) v = a.src[((size_t)z * a.rows_y + y) * a.len + x] * a.scale;
      float* p = reinterpret_cast<float*>(&A[x * LP + (r % L)]);
      p[r / L] = v;
    }
    __syncthreads();
    x_forward_store(A, B, a, LP, z, y0);
    return;
  }

  const Geom& g = a.g;
  // 1. stage the two Hermitian half-spectra of each line: B[kx*2L + r]
  for (int idx = threadIdx.x; idx < Hx * 2 * L; idx += blockDim.x) {
    const int kx = idx / (2 * L), r = idx - kx * 2 * L;
    const int y = y0 + r;
    B[idx] = y < g.Py ? a.S[((size_t)kx * g.Pz + z) * g.Py + y] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  // 2. pack Z[k] = Xa[k] + i Xb[k] over the full length (Hermitian extension);
  //    imaginary parts of DC / Nyquist are dropped as FFTW's c2r does.
  for (int idx = threadIdx.x; idx < Wx * L; idx += blockDim.x) {
    const int k = idx / L, l = idx - k * L;
    float2 xa, xb;
    if (k < Hx) {
      xa = B[k * 2 * L + l];
      xb = B[k * 2 * L + L + l];
      if (k == 0 || 2 * k == Wx) {
        xa.y = 0.f;
        xb.y = 0.f;
      }
    } else {
      xa = cconj(B[(Wx - k) * 2 * L + l]);
      xb = cconj(B[(Wx - k) * 2 * L + L + l]);
    }
    A[k * LP + l] = make_float2(xa.x - xb.y, xa.y + xb.x);
  }
  __syncthreads();
  float2* R = fft_lines<true>(A, B, L, LP, a.plan);
  float2* O = (R == A) ? B : A;

  if (a.mode == XM_CONV_OUT) {  // P == I: every row is inside
    for (int idx = threadIdx.x; idx < g.Px * 2 * L; idx += blockDim.x) {
      const int x = idx / (2 * L), r = idx - x * 2 * L;
      const int y = y0 + r;
      if (y < g.Py) {
        const float2 c = R[(x + g.cx) * LP + r % L];
        a.out[((size_t)z * g.Py + y) * g.Px + x] = r / L ? c.y : c.x;
      }
    }
    return;
  }

  // 3. pointwise epilogue over the P-domain rows of this CTA
  double accv[3] = {0.0, 0.0, 0.0};
  const bool last = a.mode == XM_UPDATE_LAST;
  for (int idx = threadIdx.x; idx < g.Px * 2 * L; idx += blockDim.x) {
    const int x = idx / (2 * L), r = idx - x * 2 * L;
    const int l = r % L, hi = r / L;
    const int y = y0 + r;
    float val = 0.f;
    if (y < g.Py) {
      const float2 c = R[(x + g.cx) * LP + l];
      const float m = hi ? c.y : c.x;
      const int iz = z - g.oz, iy = y - g.oy, ix = x - g.ox;
      const bool inside = iz >= 0 && iz < g.Iz && iy >= 0 && iy < g.Iy && ix >= 0 && ix < g.Ix;
      const size_t oidx = ((size_t)clampi(iz, 0, g.Iz - 1) * g.Iy + clampi(iy, 0, g.Iy - 1)) * g.Ix +
                          clampi(ix, 0, g.Ix - 1);
      const float o = __ldg(&a.obs[oidx]);
      if (a.mode == XM_RATIO) {
        const float mm = fmaxf(m, kEps);
        val = o / mm;
        if (inside) accv[0] += (double)o * log((double)mm) - (double)mm;
      } else {
        const size_t eidx = ((size_t)z * g.Py + y) * g.Px + x;
        val = fmaxf(a.est[eidx] * m, 0.f);
        if (!last) a.est[eidx] = val;
        if (inside) {
          accv[0] += val;
          accv[1] += (double)val * val;
          accv[2] += (double)val * o;
          if (last) a.out[oidx] = val;
        }
      }
    }
    reinterpret_cast<float*>(&O[x * LP + l])[hi] = val;
  }
  {  // this block's partials in the iteration's slot (reduce_iter_partials_kernel)
    double* dst = a.acc + ((size_t)(blockIdx.y + a.zoff) * gridDim.x + blockIdx.x) * 4;
    if (a.mode == XM_RATIO) {
      double v1[1] = {accv[0]};
      block_partial<1>(v1, dst);
    } else {
      block_partial<3>(accv, dst + 1);
    }
  }
  if (last) return;
  for (int idx = threadIdx.x; idx < (Wx - g.Px) * L; idx += blockDim.x) {
    const int x = g.Px + idx / L, l = idx % L;
    O[x * LP + l] = make_float2(0.f, 0.f);
  }
  __syncthreads();
  x_forward_store(O, R, a, LP, z, y0);
}

__global__ void __launch_bounds__(256) ypass_kernel(const YArgs a) {
  extern __shared__ float2 smem[];
  const int L = a.L, LP = line_pitch(L), N = a.plan.n;
  float2* A = smem;
  float2* B = smem + N * LP;
  const int line0 = blockIdx.x * L;
  for (int idx = threadIdx.x; idx < L * N; idx += blockDim.x) {
    const int l = idx / N, i = idx - l * N;
    const int line = line0 + l;
    float2 v = make_float2(0.f, 0.f);
    if (line < a.nlines && i < a.n_in) v = a.in[(size_t)y_line(a, line) * a.in_pitch + i];
    A[i * LP + l] = v;
  }
  __syncthreads();
  float2* R;
  if (a.mode == YM_INV) {
    R = fft_lines<true>(A, B, L, LP, a.plan);
  } else {
    R = fft_lines<false>(A, B, L, LP, a.plan);
    if (a.mode == YM_CONV) {
      for (int idx = threadIdx.x; idx < L * N; idx += blockDim.x) {
        const int l = idx / N, k = idx - l * N;
        const int line = line0 + l;
        if (line < a.nlines) R[k * LP + l] = cmul(R[k * LP + l], __ldg(&a.otf[(size_t)line * N + k]));
      }
      __syncthreads();
      R = fft_lines<true>(R, R == A ? B : A, L, LP, a.plan);
    }
  }
  for (int idx = threadIdx.x; idx < L * a.n_out; idx += blockDim.x) {
    const int l = idx / a.n_out, j = idx - l * a.n_out;
    const int line = line0 + l;
    if (line < a.nlines) a.out[(size_t)y_line(a, line) * a.out_pitch + j] = R[(j + a.out_off) * LP + l];
  }
}

__global__ void __launch_bounds__(256) zpass_kernel(const ZArgs a) {
  extern __shared__ float2 smem[];
  const int L = a.L, LP = line_pitch(L), N = a.plan.n;
  float2* A = smem;
  float2* B = smem + N * LP;
  const int kx = blockIdx.y;
  const int ky0 = blockIdx.x * L;
  const size_t plane = (size_t)kx * a.zrows * a.Wy;
  for (int idx = threadIdx.x; idx < N * L; idx += blockDim.x) {
    const int z = idx / L, l = idx - z * L;
    const int ky = ky0 + l;
    float2 v = make_float2(0.f, 0.f);
    if (z < a.n_in && ky < a.Wy) v = a.S[plane + (size_t)z * a.Wy + ky];
    A[z * LP + l] = v;
  }
  __syncthreads();
  float2* R = fft_lines<false>(A, B, L, LP, a.plan);
  const size_t oplane = (size_t)kx * N * a.Wy;
  if (a.mode == ZM_FWD_OUT) {
    for (int idx = threadIdx.x; idx < N * L; idx += blockDim.x) {
      const int kz = idx / L, l = idx - kz * L;
      const int ky = ky0 + l;
      if (ky < a.Wy) a.otf_out[oplane + (size_t)kz * a.Wy + ky] = R[kz * LP + l];
    }
    return;
  }
  for (int idx = threadIdx.x; idx < N * L; idx += blockDim.x) {
    const int kz = idx / L, l = idx - kz * L;
    const int ky = ky0 + l;
    if (ky < a.Wy) R[kz * LP + l] = cmul(R[kz * LP + l], __ldg(&a.otf[oplane + (size_t)kz * a.Wy + ky]));
  }
  __syncthreads();
  R = fft_lines<true>(R, R == A ? B : A, L, LP, a.plan);
  for (int idx = threadIdx.x; idx < a.n_out * L; idx += blockDim.x) {
    const int z = idx / L, l = idx - z * L;
    const int ky = ky0 + l;
    if (ky < a.Wy) a.S[plane + (size_t)z * a.Wy + ky] = R[(z + a.out_off) * LP + l];
  }
}

// ---- setup / bookkeeping kernels ----------------------------------------

// Statistics of the observed image: [0] negative flag (v < 0; NaN passes as
// in deconv.cpp:316-318), sums for si_psnr (sr, srr) and min/max for
// metrics.cpp:36-43 range_of.
struct ObsStats {
  double sr, srr;
  unsigned int neg;
  unsigned int minbits, maxbits;
  unsigned int pad;
  double sump;  // sum over the padded domain (flat_init mean, deconv.cpp:337-341)
};

// part: [gridDim.x][2] block partials of (sum r, sum r^2), reduced into
// st->sr, st->srr by reduce_partials_kernel.
__global__ void obs_stats_kernel(const float* __restrict__ obs, size_t n, ObsStats* st, double* part) {
  double v[2] = {0.0, 0.0};
  unsigned int neg = 0;
  unsigned int mn = 0x7f800000u, mx = 0u;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float o = obs[i];
    neg |= (o < 0.f) ? 1u : 0u;
    v[0] += o;
    v[1] += (double)o * o;
    const unsigned int b = o == 0.f ? 0u : __float_as_uint(o);  // -0 orders as +0
    if (!(o < 0.f)) {
      mn = min(mn, b);
      mx = max(mx, b);
    }
  }
  block_partial<2>(v, part + (size_t)blockIdx.x * 2);
  for (int o = 16; o > 0; o >>= 1) {
    neg |= __shfl_xor_sync(0xffffffffu, neg, o);
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (neg) atomicOr(&st->neg, 1u);
    atomicMin(&st->minbits, mn);
    atomicMax(&st->maxbits, mx);
  }
}

// est = edge-replicate pad of obs (deconv.cpp:221-237, 335-344); also the
// padded-domain sum for flat_init.
// sum_z0/sum_z1: P rows whose values enter sump (a slab sums its own rows).
// part: [gridDim.x] block partials of the padded-domain sum (-> st->sump).
__global__ void pad_kernel(const float* __restrict__ obs, float* __restrict__ est, Geom g, double* part,
                           int sum_z0, int sum_z1) {
  const size_t n = (size_t)g.Pz * g.Py * g.Px;
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.Px);
    const size_t t = i / g.Px;
    const int y = (int)(t % g.Py), z = (int)(t / g.Py);
    const size_t o = ((size_t)clampi(z - g.oz, 0, g.Iz - 1) * g.Iy + clampi(y - g.oy, 0, g.Iy - 1)) * g.Ix +
                     clampi(x - g.ox, 0, g.Ix - 1);
    const float val = obs[o];
    est[i] = val;
    if (z >= sum_z0 && z < sum_z1) v[0] += val;
  }
  block_partial<1>(v, part + blockIdx.x);
}

// Constant fill (a slab's flat_init with the mean of the whole volume).
__global__ void fill_value_kernel(float* __restrict__ est, size_t n, float value) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    est[i] = value;
}

// flat_init: est = mean(obs_p) evaluated in double then stored in f32.
__global__ void fill_mean_kernel(float* __restrict__ est, size_t n, const ObsStats* st) {
  const float mean = (float)(st->sump / (double)n);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    est[i] = mean;
}

// Circular-mode kernel of filters::fft_convolve (filters.cpp:215-233): the
// kernel centre (K-1)/2 wrapped to index 0 of the W grid (dst pre-zeroed).
__global__ void wrap_kernel_kernel(const float* __restrict__ k, int Kz, int Ky, int Kx, int Wz, int Wy, int Wx,
                                   float* __restrict__ dst) {
  const size_t n = (size_t)Kz * Ky * Kx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % Kx);
    const size_t t = i / Kx;
    const int y = (int)(t % Ky), z = (int)(t / Ky);
    const int wz = ((z - (Kz - 1) / 2) % Wz + Wz) % Wz;
    const int wy = ((y - (Ky - 1) / 2) % Wy + Wy) % Wy;
    const int wx = ((x - (Kx - 1) / 2) % Wx + Wx) % Wx;
    dst[((size_t)wz * Wy + wy) * Wx + wx] = k[i];
  }
}

// Periodic extension for circular fft_convolve on extents the device FFT
// does not plan (not 5-smooth): dst [Ez][Ey][Ex] = src[(i - h) mod A] per axis.
__global__ void wrap_extend_kernel(const float* __restrict__ src, int Az, int Ay, int Ax, float* __restrict__ dst,
                                   int Ez, int Ey, int Ex, int hz, int hy, int hx) {
  const size_t n = (size_t)Ez * Ey * Ex;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % Ex);
    const size_t t = i / Ex;
    const int y = (int)(t % Ey), z = (int)(t / Ey);
    const int sz = ((z - hz) % Az + Az) % Az, sy = ((y - hy) % Ay + Ay) % Ay, sx = ((x - hx) % Ax + Ax) % Ax;
    dst[i] = src[((size_t)sz * Ay + sy) * Ax + sx];
  }
}

// dst [Az][Ay][Ax] = src [Ez][Ey][Ex] at offset (hz, hy, hx).
__global__ void crop_block_kernel(const float* __restrict__ src, int Ey, int Ex, float* __restrict__ dst, int Az,
                                  int Ay, int Ax, int hz, int hy, int hx) {
  const size_t n = (size_t)Az * Ay * Ax;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % Ax);
    const size_t t = i / Ax;
    const int y = (int)(t % Ay), z = (int)(t / Ay);
    dst[i] = src[((size_t)(z + hz) * Ey + (y + hy)) * Ex + (x + hx)];
  }
}

// P -> I crop (deconv.cpp:239-252) for runs that stop early.
__global__ void crop_kernel(const float* __restrict__ est, float* __restrict__ out, Geom g) {
  const size_t n = (size_t)g.Iz * g.Iy * g.Ix;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.Ix);
    const size_t t = i / g.Ix;
    const int y = (int)(t % g.Iy), z = (int)(t / g.Iy);
    out[i] = est[((size_t)(z + g.oz) * g.Py + (y + g.oy)) * g.Px + (x + g.ox)];
  }
}

#endif  // VK_NO_GENERIC_KERNELS

}  // namespace vk
