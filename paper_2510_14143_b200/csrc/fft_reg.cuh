// Register-resident mixed-radix FFT building blocks (compile-time lengths).
//
// The generic Stockham engine (fft_core.cuh) walks one radix-2..8 stage per
// shared-memory round trip with runtime index math.  For the FFT lengths the
// benchmark grids use, this header builds each line transform as TWO passes
// of large register radices, N = R1 * R2 (e.g. 576 = 24*24, 1080 = 30*36):
//
//   pass 1 (no twiddles):   y[j*R1 + q] = DFT_R1( x[j + r*R2] )_q          j < R2
//   pass 2 (in place):      z[j + q*R1] = DFT_R2( y[j + r*R1] * w_N^{r j} )_q  j < R1
//
// i.e. the Stockham recurrence with Ns = 1 then Ns = R1, so the output is in
// natural order.  Each radix-R DFT runs entirely in registers as a nested
// Cooley-Tukey over R = A*B with compile-time twiddles (constexpr sin/cos in
// double, rounded once to float).  Lines are interleaved in shared memory with
// a one-element pad: element i of line l lives at
//     sw<L>(i, l) = i*(L+1) + l
// A row (fixed i, L lines) is L consecutive float2 (Stockham passes, kx-row
// staging) and a column (fixed l, consecutive i: the transposed
// global<->shared staging) strides 2L+2 words, which covers all 32 banks per
// half-warp for 8-byte accesses.  Unlike an XOR swizzle, every address in an
// unrolled pass is a per-thread base plus a compile-time immediate, which
// removes most integer address arithmetic from the transforms (measured:
// ~45% of zpass instructions were LEA/IADD3/LOP3 with the swizzle).  Pass-2
// twiddles come from a per-CTA shared table tw[m] = w_N^m (double-evaluated).
#pragma once
#include <cuda_runtime.h>

#include <utility>

#include "fft_core.cuh"

namespace vk {
namespace reg {

// ---- constexpr trigonometry (double) ---------------------------------------
constexpr double kPi = 3.14159265358979323846264338327950288;

__host__ __device__ constexpr double ce_sin_series(double x) {
  double term = x, sum = x;
  for (int n = 1; n < 30; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double ce_cos_series(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 30; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}
// exp(-2 pi i k / n) evaluated exactly on the octant grid, series elsewhere.
__host__ __device__ constexpr double ce_cos2pi(long k, long n) {
  k %= n;
  if (k < 0) k += n;
  // reduce to [0, n/4] using symmetries via exact integer arithmetic on 8k vs n
  if (8 * k <= n) return ce_cos_series(2.0 * kPi * (double)k / (double)n);
  if (4 * k <= n) return ce_sin_series(2.0 * kPi * (double)(n - 4 * k) / (4.0 * (double)n));
  if (2 * k <= n) return -ce_cos2pi(n - 2 * k, 2 * n);  // cos(pi - a) = -cos(a), a = 2 pi (n/2 - k)/n
  return ce_cos2pi(n - k, n);
}
__host__ __device__ constexpr double ce_sin2pi(long k, long n) {
  k %= n;
  if (k < 0) k += n;
  if (2 * k > n) return -ce_sin2pi(n - k, n);
  if (4 * k > n) return ce_sin2pi(n - 2 * k, 2 * n);  // sin(pi - a) = sin(a)
  if (8 * k > n) return ce_cos_series(2.0 * kPi * (double)(n - 4 * k) / (4.0 * (double)n));
  return ce_sin_series(2.0 * kPi * (double)k / (double)n);
}

template <int N, int K>
struct Tw {
  // forward twiddle exp(-2 pi i K / N)
  static constexpr float c = (float)ce_cos2pi(K, N);
  static constexpr float s = (float)(-ce_sin2pi(K, N));
};

// ---- static_for -------------------------------------------------------------
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// v * w_N^K (conjugated twiddle for the inverse), with exact special cases.
template <int N, int K, bool INV>
__device__ __forceinline__ float2 twiddle(float2 v) {
  constexpr int k = ((K % N) + N) % N;
  if constexpr (k == 0) {
    return v;
  } else if constexpr (4 * k == N) {
    return mul_mi<INV>(v);
  } else if constexpr (2 * k == N) {
    return cscale(v, -1.f);
  } else if constexpr (4 * k == 3 * N) {
    return mul_mi<!INV>(v);
  } else {
    constexpr float c = Tw<N, k>::c;
    constexpr float s = INV ? -Tw<N, k>::s : Tw<N, k>::s;
    return cmul(v, make_float2(c, s));
  }
}

// Smallest leaf factor used to split a composite radix.
template <int R>
__host__ __device__ constexpr int split_factor() {
  if (R % 8 == 0 && R != 8) return 8;
  if (R % 4 == 0 && R != 4) return 4;
  if (R % 5 == 0 && R != 5) return 5;
  if (R % 3 == 0 && R != 3) return 3;
  if (R % 2 == 0 && R != 2) return 2;
  return R;
}

// In-register DFT of compile-time size R, natural order in and out.
template <int R, bool INV>
__device__ __forceinline__ void rdft(float2 (&v)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2 || R == 3 || R == 4 || R == 5 || R == 8) {
    dft<R, INV>(v);
  } else {
    constexpr int A = split_factor<R>();
    constexpr int B = R / A;
    static_assert(A * B == R && A > 1 && B > 1, "radix must be 2^a 3^b 5^c");
    // n = B*n1 + n2 ; k = k1 + A*k2
    static_for<0, B>([&](auto n2c) {
      constexpr int n2 = decltype(n2c)::value;
      float2 u[A];
      static_for<0, A>([&](auto n1c) { u[decltype(n1c)::value] = v[B * decltype(n1c)::value + n2]; });
      rdft<A, INV>(u);
      static_for<0, A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        v[B * k1 + n2] = twiddle<R, n2 * k1, INV>(u[k1]);
      });
    });
    float2 out[R];
    static_for<0, A>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      float2 u[B];
      static_for<0, B>([&](auto n2c) { u[decltype(n2c)::value] = v[B * k1 + decltype(n2c)::value]; });
      rdft<B, INV>(u);
      static_for<0, B>([&](auto k2c) { out[k1 + A * decltype(k2c)::value] = u[decltype(k2c)::value]; });
    });
    static_for<0, R>([&](auto i) { v[decltype(i)::value] = out[decltype(i)::value]; });
  }
}

// Length-N twiddle table into shared memory (N <= blockDim multiple loops).
__device__ __forceinline__ void load_twiddles(float2* tw_s, const float2* __restrict__ tw_g, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) tw_s[i] = tw_g[i];
}

// Pass-2 twiddles of fft2<R1, R2> laid out by butterfly: tw_s[j*R2 + r] =
// w_N^{r j} (j < R1, r < R2) gathered from the natural table tw_g[m] = w_N^m
// (r j < N, no reduction needed).  A pass-2 butterfly then reads its R2-1
// twiddles at one base address plus compile-time offsets instead of holding
// R2-1 separate address registers.
template <int R1, int R2>
__device__ __forceinline__ void load_twiddles2(float2* tw_s, const float2* __restrict__ tw_g) {
  for (int i = threadIdx.x; i < R1 * R2; i += blockDim.x) {
    const int j = i / R2, r = i - j * R2;
    tw_s[i] = tw_g[r * j];
  }
}

// threadIdx.x through a volatile asm: index math derived from it cannot be
// hoisted out of a persistent task loop (which otherwise keeps every unrolled
// shared-memory address of the transform live in registers across tasks).
__device__ __forceinline__ int fresh_tid() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

template <int L>
__device__ __forceinline__ int sw(int i, int l) {
  return i * (L + 1) + l;
}

// In-place two-pass transform of L interleaved (swizzled) lines of
// length N = R1*R2 held in `buf` (natural order in and out).  NT = blockDim.x
// must cover every pass-1 butterfly with one thread (NT >= L*R2) so pass 1 can
// stage its inputs in registers, sync, and overwrite in place; pass 2 reads
// and writes the same index set per thread.  Caller syncs before.
// TWG: `tw` is the butterfly-major table in global memory (read through L1)
// instead of shared memory.
// Element (i, l) lives at buf[i * LP + l * LS]: LS = 1 is the interleaved
// layout (LP = L+1 pad, or LP = L for 16-lane rows); LP = 1 with LS = row
// pitch is the line-major layout bulk copies land in.
// C2R input of line l, sample i, read from the x pass's TMA-staged spectrum
// tile st = [k][2L] (k = kx <= N/2, rows 2l / 2l+1 = the line's real and
// imaginary halves, one 16-byte pair): Z[i] = Xa[i] + i Xb[i] for i <= N/2,
// conj(Xa[N-i]) + i conj(Xb[N-i]) above; DC / Nyquist imaginary parts
// dropped as FFTW's c2r does.
template <int N, int L>
__device__ __forceinline__ float2 c2r_staged(const float2* st, int i, int l) {
  const bool hi = 2 * i > N;
  const int k = hi ? N - i : i;
  const float4 p = reinterpret_cast<const float4*>(st)[k * L + l];
  if (k == 0 || 2 * k == N) return make_float2(p.x, p.z);
  return hi ? make_float2(p.x + p.w, p.z - p.y) : make_float2(p.x - p.w, p.y + p.z);
}

// STG: pass 1 gathers its inputs with c2r_staged from the staged tile that
// occupies the front of `buf` (all reads complete before the barrier that
// precedes the first store, so the tile may alias the transform buffer).
template <int R1, int R2, int L, int NT, bool INV, int LP = L + 1, bool TWG = false, int LS = 1, bool STG = false>
__device__ __forceinline__ void fft2(float2* buf, const float2* tw) {
  static_assert(NT >= L * R2, "pass 1 needs one butterfly per thread");
#ifdef VK_DEBUG_NOFFT  // experiment builds only: isolate the memory cost of a pass
  __syncthreads();
  return;
#endif
  {
    const int t = fresh_tid();
    const int l = t % L, j = t / L;
    const bool act = t < L * R2;
    float2 v[R1];
    if (act) {
      if constexpr (STG)
        static_for<0, R1>([&](auto r) { v[decltype(r)::value] = c2r_staged<R1 * R2, L>(buf, j + decltype(r)::value * R2, l); });
      else
        static_for<0, R1>([&](auto r) { v[decltype(r)::value] = buf[(j + decltype(r)::value * R2) * LP + l * LS]; });
    }
    __syncthreads();
    if (act) {
      rdft<R1, INV>(v);
      static_for<0, R1>([&](auto q) { buf[(j * R1 + decltype(q)::value) * LP + l * LS] = v[decltype(q)::value]; });
    }
    __syncthreads();
  }
#pragma unroll 1
  for (int t = fresh_tid(); t < L * R1; t += NT) {
    // With 8 lines per block a half-warp spans two butterflies j; rows j and
    // j+1 share a bank pair under the (L+1) pad, rows j and j+8 do not, so
    // pair groups (2m, 2m+1) map to j = m and m+8 within each 16 butterflies.
    const int l = t % L, g = t / L;
    constexpr int G16 = (R1 / 16) * 16;
    const int j = (L == 8 && LP == 9 && LS == 1 && g < G16) ? ((g & ~15) | ((g >> 1) & 7) | ((g & 1) << 3)) : g;
    float2 v[R2];
    v[0] = buf[j * LP + l * LS];
    static_for<1, R2>([&](auto r) {
      constexpr int rr = decltype(r)::value;
      const float2 w = TWG ? __ldg(tw + j * R2 + rr) : tw[j * R2 + rr];  // load_twiddles2 layout
      const float2 x = buf[(j + rr * R1) * LP + l * LS];
      v[rr] = INV ? cmulc(x, w) : cmul(x, w);
    });
    rdft<R2, INV>(v);
    static_for<0, R2>([&](auto q) { buf[(j + decltype(q)::value * R1) * LP + l * LS] = v[decltype(q)::value]; });
  }
  __syncthreads();
}

}  // namespace reg
}  // namespace vk
