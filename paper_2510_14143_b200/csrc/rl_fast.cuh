// Compile-time-length pass kernels (the fast path for the FFT lengths the
// configs use).  Same contracts as the generic kernels in rl_passes.cuh, with
// these differences:
//
//  * the line transform is fft_reg.cuh's two-pass register FFT, in place in
//    ONE shared buffer with the XOR-swizzled line layout sw<L>(i, l);
//  * the x crop offset cx (deconv.cpp:59-72) is realised as a phase ramp
//    exp(+2 pi i cx kx / Wx) folded into both OTFs at plan creation, so a
//    P-domain row lives at slots [cx, cx+Px) of its length-Wx line before the
//    forward transform AND after the inverse one.  The pointwise epilogue then
//    reads the model and writes the ratio / update into the same slot.
//    (Circular shift by cx, then by -cx: exact; the linear-convolution
//    support [0, P+K-1) still fits inside Wx.)
//  * the x-pass epilogue works on whole row PAIRS (the re/im halves of one
//    packed line) so every shared access is 8 bytes and conflict-free;
//  * memory-level parallelism: pure copies global->shared use cp.async
//    (LDGSTS) issued all at once; loads that feed arithmetic are batched
//    U-deep per thread before use; OTF tiles are prefetched with cp.async
//    while the forward transform runs.
#pragma once
#include "fft_reg.cuh"
#include "rl_passes.cuh"

namespace vk {

using reg::sw;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <int R1, int R2, int L, bool OTF_PREFETCH = false>
struct FastCfg {
  static_assert((L & (L - 1)) == 0, "L must be a power of two (swizzle)");
  static constexpr int N = R1 * R2;
  static constexpr int NT = ((L * (R1 > R2 ? R1 : R2)) + 31) / 32 * 32;
  static constexpr size_t smem = (size_t)(N * L + N + (OTF_PREFETCH ? N * L : 0)) * sizeof(float2);
};

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT)
    xpass_fast(const XArgs a) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, NT = C::NT;
  constexpr int Hx = N / 2 + 1;
  constexpr int NW = NT / 32;
  constexpr int U = 4;
  constexpr int CH = 32 * U;  // samples per work item
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  reg::load_twiddles(tw, a.plan.tw, N);
  const int z = blockIdx.y;
  const int y0 = blockIdx.x * 2 * L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Geom& g = a.g;

  if (a.mode == XM_FWD) {
    // real rows (l, L+l) -> line l, samples at slots [xoff, xoff+len)
    const int nch = (N + CH - 1) / CH;
    for (int item = warp; item < L * nch; item += NW) {
      const int l = item / nch, x0 = (item % nch) * CH;
      const int ya = y0 + l, yb = y0 + L + l;
      const bool va = ya < a.rows_y, vb = yb < a.rows_y;
      const float* ra = a.src + ((size_t)z * a.rows_y + (va ? ya : 0)) * a.len;
      const float* rb = a.src + ((size_t)z * a.rows_y + (vb ? yb : 0)) * a.len;
      float pa[U], pb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int xs = x0 + u * 32 + lane - a.xoff;
        const bool in = xs >= 0 && xs < a.len;
        pa[u] = (va && in) ? __ldg(&ra[xs]) * a.scale : 0.f;
        pb[u] = (vb && in) ? __ldg(&rb[xs]) * a.scale : 0.f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = x0 + u * 32 + lane;
        if (x < N) A[sw<L>(x, l)] = make_float2(pa[u], pb[u]);
      }
    }
  } else {
    // Hermitian halves of row pair (l, L+l) -> Z[k] = Xa[k] + i Xb[k], k < N
    const float2 zero = make_float2(0.f, 0.f);
    for (int base = threadIdx.x; base < Hx * L; base += NT * U) {
      float2 xa[U], xb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * NT;
        const int kx = idx / L, l = idx % L;
        const size_t row = ((size_t)kx * g.Pz + z) * g.Py;
        const int ya = y0 + l, yb = y0 + L + l;
        const bool ok = idx < Hx * L;
        xa[u] = (ok && ya < g.Py) ? a.S[row + ya] : zero;
        xb[u] = (ok && yb < g.Py) ? a.S[row + yb] : zero;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = base + u * NT;
        if (idx >= Hx * L) break;
        const int kx = idx / L, l = idx % L;
        if (kx == 0 || 2 * kx == N) {
          A[sw<L>(kx, l)] = make_float2(xa[u].x, xb[u].x);  // imaginary parts of DC/Nyquist dropped (c2r)
        } else {
          A[sw<L>(kx, l)] = make_float2(xa[u].x - xb[u].y, xa[u].y + xb[u].x);
          A[sw<L>(N - kx, l)] = make_float2(xa[u].x + xb[u].y, xb[u].x - xa[u].y);
        }
      }
    }
    __syncthreads();
    reg::fft2<R1, R2, L, NT, true>(A, tw);

    const bool last = a.mode == XM_UPDATE_LAST;
    const bool ratio = a.mode == XM_RATIO;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    // work item = (line l, chunk of CH samples); one warp per item, U samples
    // of both rows of the line per lane
    const int nch = (g.Px + CH - 1) / CH;
    for (int item = warp; item < L * nch; item += NW) {
      const int l = item / nch, x0 = (item % nch) * CH;
      const int ya = y0 + l, yb = y0 + L + l;
      const bool va = ya < g.Py, vb = yb < g.Py;
      const int iz = z - g.oz, iya = ya - g.oy, iyb = yb - g.oy;
      const bool zin = iz >= 0 && iz < g.Iz;
      const bool ina = va && zin && iya >= 0 && iya < g.Iy, inb = vb && zin && iyb >= 0 && iyb < g.Iy;
      const size_t zoff = (size_t)clampi(iz, 0, g.Iz - 1) * g.Iy;
      const size_t oa_off = (zoff + clampi(iya, 0, g.Iy - 1)) * g.Ix;
      const size_t ob_off = (zoff + clampi(iyb, 0, g.Iy - 1)) * g.Ix;
      const float* oa = a.obs + oa_off;
      const float* ob = a.obs + ob_off;
      float* ea = a.est + ((size_t)z * g.Py + (va ? ya : 0)) * g.Px;
      float* eb = a.est + ((size_t)z * g.Py + (vb ? yb : 0)) * g.Px;
      float2 m[U];
      float o_a[U], o_b[U], e_a[U], e_b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = x0 + u * 32 + lane;
        const bool ok = x < g.Px;
        const int xo = clampi(x - g.ox, 0, g.Ix - 1);
        m[u] = ok ? A[sw<L>(x + g.cx, l)] : make_float2(0.f, 0.f);
        o_a[u] = (ok && va) ? __ldg(&oa[xo]) : 0.f;
        o_b[u] = (ok && vb) ? __ldg(&ob[xo]) : 0.f;
        e_a[u] = (!ratio && ok && va) ? ea[x] : 0.f;
        e_b[u] = (!ratio && ok && vb) ? eb[x] : 0.f;
      }
      float f0 = 0.f, f1 = 0.f, f2 = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int x = x0 + u * 32 + lane;
        if (x >= g.Px) break;
        const int ix = x - g.ox;
        const bool xin = ix >= 0 && ix < g.Ix;
        float2 val;
        if (ratio) {
          const float ma = fmaxf(m[u].x, kEps), mb = fmaxf(m[u].y, kEps);
          val = make_float2(va ? o_a[u] / ma : 0.f, vb ? o_b[u] / mb : 0.f);
          if (xin && ina) f0 += fmaf(o_a[u], logf(ma), -ma);
          if (xin && inb) f0 += fmaf(o_b[u], logf(mb), -mb);
        } else {
          val = make_float2(va ? fmaxf(e_a[u] * m[u].x, 0.f) : 0.f, vb ? fmaxf(e_b[u] * m[u].y, 0.f) : 0.f);
          if (!last) {
            if (va) ea[x] = val.x;
            if (vb) eb[x] = val.y;
          }
          if (xin && ina) {
            f0 += val.x;
            f1 = fmaf(val.x, val.x, f1);
            f2 = fmaf(val.x, o_a[u], f2);
            if (last) a.out[oa_off + ix] = val.x;
          }
          if (xin && inb) {
            f0 += val.y;
            f1 = fmaf(val.y, val.y, f1);
            f2 = fmaf(val.y, o_b[u], f2);
            if (last) a.out[ob_off + ix] = val.y;
          }
        }
        A[sw<L>(x + g.cx, l)] = val;
      }
      acc0 += f0;
      acc1 += f1;
      acc2 += f2;
    }
    if (ratio) {
      double v1[1] = {acc0};
      block_accumulate<1>(v1, a.acc);
    } else {
      double v3[3] = {acc0, acc1, acc2};
      block_accumulate<3>(v3, a.acc + 1);
    }
    if (last) return;
    // zero the slots outside [cx, cx+Px) before the forward transform
    for (int idx = threadIdx.x; idx < (N - g.Px) * L; idx += NT) {
      const int s = idx / L, l = idx % L;
      const int x = s < g.cx ? s : s + g.Px;
      A[sw<L>(x, l)] = make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  for (int idx = threadIdx.x; idx < Hx * L; idx += NT) {
    const int kx = idx / L, l = idx % L;
    const float2 zk = A[sw<L>(kx, l)];
    const float2 zn = A[sw<L>(kx == 0 ? 0 : N - kx, l)];
    const float2 xa = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
    const float2 xb = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
    const size_t row = ((size_t)kx * a.rows_z + z) * a.rows_y;
    if (y0 + l < a.rows_y) a.S[row + y0 + l] = xa;
    if (y0 + L + l < a.rows_y) a.S[row + y0 + L + l] = xb;
  }
}

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT)
    ypass_fast(const YArgs a) {
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  float2* O = A + N * L;  // OTF tile [l][k] (CONV only)
  const int line0 = blockIdx.x * L;
  // async copies: the L input rows (zero padding written directly)
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    const bool ok = line < a.nlines;
    const float2* in = a.in + (size_t)(ok ? line : 0) * a.in_pitch;
    for (int i = threadIdx.x; i < N; i += NT) {
      if (ok && i < a.n_in)
        cp_async8(&A[sw<L>(i, l)], &in[i]);
      else
        A[sw<L>(i, l)] = make_float2(0.f, 0.f);
    }
  }
  cp_async_commit();
  if (a.mode == YM_CONV) {
    for (int l = 0; l < L; ++l) {
      const int line = line0 + l;
      if (line >= a.nlines) break;
      const float2* o = a.otf + (size_t)line * N;
      for (int k = threadIdx.x; k < N; k += NT) cp_async8(&O[l * N + k], &o[k]);
    }
    cp_async_commit();
  }
  reg::load_twiddles(tw, a.plan.tw, N);
  if (a.mode == YM_CONV)
    cp_async_wait_1();  // input rows landed, OTF may still fly
  else
    cp_async_wait_all();
  __syncthreads();
  if (a.mode == YM_INV) {
    reg::fft2<R1, R2, L, NT, true>(A, tw);
  } else {
    reg::fft2<R1, R2, L, NT, false>(A, tw);
    if (a.mode == YM_CONV) {
      cp_async_wait_all();
      __syncthreads();
      for (int idx = threadIdx.x; idx < N * L; idx += NT) {
        const int k = idx / L, l = idx % L;
        A[sw<L>(k, l)] = cmul(A[sw<L>(k, l)], O[l * N + k]);
      }
      __syncthreads();
      reg::fft2<R1, R2, L, NT, true>(A, tw);
    }
  }
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    if (line >= a.nlines) break;
    float2* out = a.out + (size_t)line * a.out_pitch;
    for (int j = threadIdx.x; j < a.n_out; j += NT) out[j] = A[sw<L>(j + a.out_off, l)];
  }
}

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT)
    zpass_fast(const ZArgs a) {
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  float2* O = A + N * L;  // OTF tile, [kz][l] row-major (pitch L)
  const int kx = blockIdx.y;
  const int ky0 = blockIdx.x * L;
  const size_t plane = (size_t)kx * a.zrows * a.Wy;
  const size_t oplane = (size_t)kx * N * a.Wy;
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (z < a.n_in && ky < a.Wy)
      cp_async8(&A[sw<L>(z, l)], &a.S[plane + (size_t)z * a.Wy + ky]);
    else
      A[sw<L>(z, l)] = make_float2(0.f, 0.f);
  }
  cp_async_commit();
  const bool conv = a.mode == ZM_CONV;
  if (conv) {
    for (int idx = threadIdx.x; idx < N * L; idx += NT) {
      const int kz = idx / L, l = idx % L;
      const int ky = ky0 + l;
      if (ky < a.Wy) cp_async8(&O[idx], &a.otf[oplane + (size_t)kz * a.Wy + ky]);
    }
    cp_async_commit();
  }
  reg::load_twiddles(tw, a.plan.tw, N);
  if (conv)
    cp_async_wait_1();
  else
    cp_async_wait_all();
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  if (!conv) {
    for (int idx = threadIdx.x; idx < N * L; idx += NT) {
      const int kz = idx / L, l = idx % L;
      const int ky = ky0 + l;
      if (ky < a.Wy) a.otf_out[oplane + (size_t)kz * a.Wy + ky] = A[sw<L>(kz, l)];
    }
    return;
  }
  cp_async_wait_all();
  __syncthreads();
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int kz = idx / L, l = idx % L;
    A[sw<L>(kz, l)] = cmul(A[sw<L>(kz, l)], O[idx]);
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, true>(A, tw);
  for (int idx = threadIdx.x; idx < a.n_out * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (ky < a.Wy) a.S[plane + (size_t)z * a.Wy + ky] = A[sw<L>(z + a.out_off, l)];
  }
}

// Phase ramp exp(+2 pi i cx kx / Wx) over an OTF laid out [Hx][Wz][Wy].
__global__ void otf_ramp_kernel(float2* __restrict__ otf, int Hx, size_t plane, int Wx, int cx) {
  const size_t n = (size_t)Hx * plane;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i / plane);
    const long long m = ((long long)cx * kx) % Wx;
    double s, c;
    sincospi(2.0 * (double)m / (double)Wx, &s, &c);
    otf[i] = cmul(otf[i], make_float2((float)c, (float)s));
  }
}

}  // namespace vk
