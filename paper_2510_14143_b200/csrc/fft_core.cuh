// Shared-memory mixed-radix Stockham FFT for sm_100a.
//
// Replaces the reference's FFTW double r2c/c2r layer (reference
// proj/src/fft_plan.cpp:84-97) on the device, in float32 with twiddles
// computed in double and rounded once (no recurrences).
//
// Layout convention used by every pass kernel: a CTA transforms L lines of
// length n that live INTERLEAVED in shared memory, element i of line l at
// buf[i*LP + l] with LP = L + 1.  Consecutive threads take consecutive lines,
// so every Stockham read and write of a warp touches consecutive float2 words;
// the +1 pitch keeps the transposed global<->smem staging (consecutive i,
// fixed l) free of bank conflicts as well.
//
// Stockham step for radix R (Ns = product of the radices already applied,
// m = n/R):
//   for j < m:  k = j mod Ns
//     v_r = src[j + r m] * w_{Ns R}^{r k}           r = 0..R-1
//     V   = DFT_R(v)
//     dst[(j/Ns) Ns R + k + q Ns] = V_q             q = 0..R-1
// which is self-sorting for any mixed-radix factorisation (checked against
// numpy in tests/test_fft_host.py through the host twin in fft_plan.hpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace vk {

constexpr int kMaxStages = 20;

// Per-length plan: radix schedule plus a pointer to the length-n twiddle table
// tw[m] = exp(-2 pi i m / n) (double-evaluated, rounded to float).
struct LinePlan {
  int n;
  int nst;
  int rad[kMaxStages];
  int ns[kMaxStages];
  const float2* tw;
  const float2* tw2;  // fast path: pass-2 twiddles, butterfly-major (reg::load_twiddles2 layout), global
};

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// Multiply by -i (forward) or +i (inverse).
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(float2* v) {
  float2 a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <bool INV>
__device__ __forceinline__ void dft3(float2* v) {
  const float c = -0.5f, s = 0.86602540378443864676f;
  float2 a = cadd(v[1], v[2]), b = csub(v[1], v[2]);
  float2 y0 = cadd(v[0], a);
  float2 t = make_float2(fmaf(c, a.x, v[0].x), fmaf(c, a.y, v[0].y));
  float2 u = mul_mi<INV>(cscale(b, s));
  v[0] = y0;
  v[1] = cadd(t, u);
  v[2] = csub(t, u);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2* v) {
  float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  float2 a2 = cadd(v[1], v[3]), a3 = mul_mi<INV>(csub(v[1], v[3]));
  v[0] = cadd(a0, a2);
  v[2] = csub(a0, a2);
  v[1] = cadd(a1, a3);
  v[3] = csub(a1, a3);
}

template <bool INV>
__device__ __forceinline__ void dft5(float2* v) {
  const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
  const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
  float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  float2 y0 = cadd(v[0], cadd(a1, a2));
  float2 t1 = make_float2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
  float2 t2 = make_float2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
  float2 u1 = mul_mi<INV>(make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
  float2 u2 = mul_mi<INV>(make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
  v[0] = y0;
  v[1] = cadd(t1, u1);
  v[4] = csub(t1, u1);
  v[2] = cadd(t2, u2);
  v[3] = csub(t2, u2);
}

template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
  const float h = 0.70710678118654752440f;
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft4<INV>(e);
  dft4<INV>(o);
  // o_q *= w8^q  (w8 = exp(-+ i pi/4))
  o[1] = INV ? make_float2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
             : make_float2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
  o[2] = mul_mi<INV>(o[2]);
  o[3] = INV ? make_float2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
             : make_float2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = cadd(e[q], o[q]);
    v[q + 4] = csub(e[q], o[q]);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2* v) {
  if constexpr (R == 2) dft2<INV>(v);
  else if constexpr (R == 3) dft3<INV>(v);
  else if constexpr (R == 4) dft4<INV>(v);
  else if constexpr (R == 5) dft5<INV>(v);
  else if constexpr (R == 8) dft8<INV>(v);
}

// One Stockham stage over L interleaved lines, work split over the CTA.
template <int R, bool INV>
__device__ __forceinline__ void stockham_stage(const float2* __restrict__ src, float2* __restrict__ dst,
                                               int L, int LP, int n, int Ns,
                                               const float2* __restrict__ tw) {
  const int m = n / R;
  const int tstride = n / (Ns * R);
  const int total = L * m;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int l = t % L;
    const int j = t / L;
    const int k = j % Ns;
    float2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[(j + r * m) * LP + l];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const float2 w = __ldg(&tw[r * k * tstride]);
        v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
      }
    }
    dft<R, INV>(v);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int q = 0; q < R; ++q) dst[(base + q * Ns) * LP + l] = v[q];
  }
}

// Transforms L interleaved lines held in `a` using `b` as ping-pong scratch.
// Returns the buffer holding the result.  Caller must __syncthreads() before
// (data in a complete) — this function syncs after every stage.
template <bool INV>
__device__ float2* fft_lines(float2* a, float2* b, int L, int LP, const LinePlan& p) {
  float2* src = a;
  float2* dst = b;
  for (int s = 0; s < p.nst; ++s) {
    switch (p.rad[s]) {
      case 2: stockham_stage<2, INV>(src, dst, L, LP, p.n, p.ns[s], p.tw); break;
      case 3: stockham_stage<3, INV>(src, dst, L, LP, p.n, p.ns[s], p.tw); break;
      case 4: stockham_stage<4, INV>(src, dst, L, LP, p.n, p.ns[s], p.tw); break;
      case 5: stockham_stage<5, INV>(src, dst, L, LP, p.n, p.ns[s], p.tw); break;
      default: stockham_stage<8, INV>(src, dst, L, LP, p.n, p.ns[s], p.tw); break;
    }
    __syncthreads();
    float2* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

}  // namespace vk
