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

// ---- complex arithmetic ----------------------------------------------------
// On sm_100a the FP32 pipe has packed two-lane forms (FADD2 / FMUL2 / FFMA2,
// PTX add/sub/mul/fma.rn.f32x2) whose operands can broadcast one lane
// (.F32) or swap the lanes (.LO_HI) for free.  A float2 complex value is one
// such register pair, so a complex add is ONE instruction, a +/- i*b ONE fused
// multiply-add with a (+-1, -+1) constant pair, and a complex product TWO
// (instead of 2, 2 and 4 scalar ones).  The transforms are issue-bound
// (ncu: ~590 M warp instructions per C2 iteration, issue active 51-64%),
// so this is a straight cut of their instruction count.  Products round
// like fmaf pairs (one rounding per fma), as before.
// VK_SCALAR_CPLX=1 builds the scalar forms (A/B measurements).
#if !defined(VK_SCALAR_CPLX) || !VK_SCALAR_CPLX
namespace pk {
__device__ __forceinline__ unsigned long long u(float2 v) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 f(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ float2 add(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u(a)), "l"(u(b)));
  return f(r);
}
__device__ __forceinline__ float2 sub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u(a)), "l"(u(b)));
  return f(r);
}
__device__ __forceinline__ float2 mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u(a)), "l"(u(b)));
  return f(r);
}
__device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) {  // a*b + c
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(u(a)), "l"(u(b)), "l"(u(c)));
  return f(r);
}
__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 sw(float2 a) { return make_float2(a.y, a.x); }
}  // namespace pk

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return pk::add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return pk::sub(a, b); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {  // (a.x b - a.y (b.y, -b.x))
  return pk::fma(pk::bc(a.y), make_float2(-b.y, b.x), pk::mul(pk::bc(a.x), b));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return pk::fma(pk::bc(a.y), pk::sw(b), pk::mul(pk::bc(a.x), make_float2(b.x, -b.y)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return pk::mul(a, pk::bc(s)); }
// a + s*b, real s
__device__ __forceinline__ float2 caxpy(float s, float2 b, float2 a) { return pk::fma(pk::bc(s), b, a); }
// Multiply by -i (forward) or +i (inverse).
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return pk::mul(pk::sw(a), INV ? make_float2(-1.f, 1.f) : make_float2(1.f, -1.f));
}
// t + s*(-+i)*u and t - s*(-+i)*u in one packed fma each (s real)
template <bool INV>
__device__ __forceinline__ float2 add_mi(float2 t, float2 u, float s = 1.f) {
  return pk::fma(pk::sw(u), INV ? make_float2(-s, s) : make_float2(s, -s), t);
}
template <bool INV>
__device__ __forceinline__ float2 sub_mi(float2 t, float2 u, float s = 1.f) {
  return pk::fma(pk::sw(u), INV ? make_float2(s, -s) : make_float2(-s, s), t);
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 caxpy(float s, float2 b, float2 a) { return make_float2(fmaf(s, b.x, a.x), fmaf(s, b.y, a.y)); }
template <bool INV>
__device__ __forceinline__ float2 mul_mi(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
template <bool INV>
__device__ __forceinline__ float2 add_mi(float2 t, float2 u, float s = 1.f) {
  return cadd(t, mul_mi<INV>(cscale(u, s)));
}
template <bool INV>
__device__ __forceinline__ float2 sub_mi(float2 t, float2 u, float s = 1.f) {
  return csub(t, mul_mi<INV>(cscale(u, s)));
}
#endif
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

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
  float2 t = caxpy(c, a, v[0]);
  v[0] = y0;
  v[1] = add_mi<INV>(t, b, s);
  v[2] = sub_mi<INV>(t, b, s);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2* v) {
  float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
  float2 a2 = cadd(v[1], v[3]), d = csub(v[1], v[3]);
  v[0] = cadd(a0, a2);
  v[2] = csub(a0, a2);
  v[1] = add_mi<INV>(a1, d);
  v[3] = sub_mi<INV>(a1, d);
}

template <bool INV>
__device__ __forceinline__ void dft5(float2* v) {
  const float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
  const float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
  float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  float2 y0 = cadd(v[0], cadd(a1, a2));
  float2 t1 = caxpy(c2, a2, caxpy(c1, a1, v[0]));
  float2 t2 = caxpy(c1, a2, caxpy(c2, a1, v[0]));
  float2 w1 = caxpy(s2, b2, cscale(b1, s1));
  float2 w2 = caxpy(-s1, b2, cscale(b1, s2));
  v[0] = y0;
  v[1] = add_mi<INV>(t1, w1);
  v[4] = sub_mi<INV>(t1, w1);
  v[2] = add_mi<INV>(t2, w2);
  v[3] = sub_mi<INV>(t2, w2);
}

template <bool INV>
__device__ __forceinline__ void dft8(float2* v) {
  const float h = 0.70710678118654752440f;
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft4<INV>(e);
  dft4<INV>(o);
  // o_q *= w8^q  (w8 = exp(-+ i pi/4)): o1 = h (o1 -+ i o1), o3 = h (-o3 -+ i o3)
  o[1] = add_mi<INV>(cscale(o[1], h), o[1], h);
  o[3] = add_mi<INV>(cscale(o[3], -h), o[3], h);
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o[1]);
  v[5] = csub(e[1], o[1]);
  v[2] = add_mi<INV>(e[2], o[2]);  // o2 *= -+i
  v[6] = sub_mi<INV>(e[2], o[2]);
  v[3] = cadd(e[3], o[3]);
  v[7] = csub(e[3], o[3]);
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
