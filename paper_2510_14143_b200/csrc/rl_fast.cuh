// Compile-time-length pass kernels (the fast path for the FFT lengths the
// configs use).  Same contracts as the generic kernels in rl_passes.cuh, with
// these differences:
//
//  * the line transform is fft_reg.cuh's two-pass register FFT, in place in
//    ONE shared buffer;
//  * the x crop offset cx (deconv.cpp:59-72) is realised as a phase ramp
//    exp(+2 pi i cx kx / Wx) folded into both OTFs at plan creation, so a
//    P-domain row lives at slots [cx, cx+Px) of its length-Wx line before the
//    forward transform AND after the inverse one.  The pointwise epilogue then
//    reads the model and writes the ratio / update into the same slot.
//    (Circular shift by cx, then by -cx: exact; the linear-convolution
//    support [0, P+K-1) still fits inside Wx.)
//  * memory-level parallelism: pure copies global->shared use cp.async
//    (LDGSTS) issued all at once; loads that feed arithmetic are batched
//    U-deep per thread before use; the z-pass OTF tile is prefetched with
//    cp.async while the forward transform runs.
#pragma once
#include "fft_reg.cuh"
#include "rl_passes.cuh"

namespace vk {

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int R1, int R2, int L, bool OTF_PREFETCH = false>
struct FastCfg {
  static constexpr int N = R1 * R2;
  static constexpr int LP = L + 1;
  static constexpr int NT = ((L * (R1 > R2 ? R1 : R2)) + 31) / 32 * 32;
  static constexpr size_t smem = (size_t)(N * LP + N + (OTF_PREFETCH ? N * L : 0)) * sizeof(float2);
};

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT)
    xpass_fast(const XArgs a) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  constexpr int Hx = N / 2 + 1;
  constexpr int NW = NT / 32;
  constexpr int U = 4;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  reg::load_twiddles(tw, a.plan.tw, N);
  const int z = blockIdx.y;
  const int y0 = blockIdx.x * 2 * L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Geom& g = a.g;

  if (a.mode == XM_FWD) {
    // real rows [xoff, xoff+len) of each line, zero elsewhere; one warp per row
    for (int r = warp; r < 2 * L; r += NW) {
      const int y = y0 + r;
      const bool yok = y < a.rows_y;
      const float* row = a.src + ((size_t)z * a.rows_y + (yok ? y : 0)) * a.len;
      float* dst = reinterpret_cast<float*>(A) + 2 * (r % L) + (r / L);
      for (int x0 = 0; x0 < N; x0 += 32 * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int x = x0 + u * 32 + lane;
          const int xs = x - a.xoff;
          v[u] = (yok && x < N && xs >= 0 && xs < a.len) ? __ldg(&row[xs]) * a.scale : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int x = x0 + u * 32 + lane;
          if (x < N) dst[2 * x * LP] = v[u];
        }
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
          A[kx * LP + l] = make_float2(xa[u].x, xb[u].x);  // imaginary parts of DC/Nyquist dropped (c2r)
        } else {
          A[kx * LP + l] = make_float2(xa[u].x - xb[u].y, xa[u].y + xb[u].x);
          A[(N - kx) * LP + l] = make_float2(xa[u].x + xb[u].y, xb[u].x - xa[u].y);
        }
      }
    }
    __syncthreads();
    reg::fft2<R1, R2, L, NT, true>(A, tw);

    double accv[3] = {0.0, 0.0, 0.0};
    const bool last = a.mode == XM_UPDATE_LAST;
    const bool ratio = a.mode == XM_RATIO;
    // one warp per row, U x 32 samples in flight per lane
    for (int r = warp; r < 2 * L; r += NW) {
      const int y = y0 + r;
      const int l = r % L, hi = r / L;
      float* slots = reinterpret_cast<float*>(A) + 2 * l + hi;  // slot(x) = slots[2 * (x + cx) * LP]
      if (y >= g.Py) {
        for (int x = lane; x < g.Px; x += 32) slots[2 * (x + g.cx) * LP] = 0.f;
        continue;
      }
      const int iz = z - g.oz, iy = y - g.oy;
      const bool zyin = iz >= 0 && iz < g.Iz && iy >= 0 && iy < g.Iy;
      const size_t orow_off = ((size_t)clampi(iz, 0, g.Iz - 1) * g.Iy + clampi(iy, 0, g.Iy - 1)) * g.Ix;
      const float* orow = a.obs + orow_off;
      float* erow = a.est + ((size_t)z * g.Py + y) * g.Px;
      for (int x0 = 0; x0 < g.Px; x0 += 32 * U) {
        float m[U], o[U], e[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int x = x0 + u * 32 + lane;
          const bool ok = x < g.Px;
          m[u] = ok ? slots[2 * (x + g.cx) * LP] : 0.f;
          o[u] = ok ? __ldg(&orow[clampi(x - g.ox, 0, g.Ix - 1)]) : 0.f;
          e[u] = (!ratio && ok) ? erow[x] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int x = x0 + u * 32 + lane;
          if (x >= g.Px) break;
          const int ix = x - g.ox;
          const bool inside = zyin && ix >= 0 && ix < g.Ix;
          float val;
          if (ratio) {
            const float mm = fmaxf(m[u], kEps);
            val = o[u] / mm;
            if (inside) accv[0] += (double)o[u] * (double)logf(mm) - (double)mm;
          } else {
            val = fmaxf(e[u] * m[u], 0.f);
            if (!last) erow[x] = val;
            if (inside) {
              accv[0] += val;
              accv[1] += (double)val * val;
              accv[2] += (double)val * o[u];
              if (last) a.out[orow_off + ix] = val;
            }
          }
          slots[2 * (x + g.cx) * LP] = val;
        }
      }
    }
    if (ratio) {
      double v1[1] = {accv[0]};
      block_accumulate<1>(v1, a.acc);
    } else {
      block_accumulate<3>(accv, a.acc + 1);
    }
    if (last) return;
    // zero the slots outside [cx, cx+Px) before the forward transform
    for (int idx = threadIdx.x; idx < (N - g.Px) * L; idx += NT) {
      const int s = idx / L, l = idx % L;
      const int x = s < g.cx ? s : s + g.Px;
      A[x * LP + l] = make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  for (int idx = threadIdx.x; idx < Hx * L; idx += NT) {
    const int kx = idx / L, l = idx % L;
    const float2 zk = A[kx * LP + l];
    const float2 zn = A[(kx == 0 ? 0 : N - kx) * LP + l];
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
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  float2* O = A + N * LP;  // OTF tile [l][k] (CONV only)
  const int line0 = blockIdx.x * L;
  // async copies: the L input rows (zero padding written directly)
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    const bool ok = line < a.nlines;
    const float2* in = a.in + (size_t)(ok ? line : 0) * a.in_pitch;
    for (int i = threadIdx.x; i < N; i += NT) {
      if (ok && i < a.n_in)
        cp_async8(&A[i * LP + l], &in[i]);
      else
        A[i * LP + l] = make_float2(0.f, 0.f);
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
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // input rows landed, OTF may still fly
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
        A[k * LP + l] = cmul(A[k * LP + l], O[l * N + k]);
      }
      __syncthreads();
      reg::fft2<R1, R2, L, NT, true>(A, tw);
    }
  }
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    if (line >= a.nlines) break;
    float2* out = a.out + (size_t)line * a.out_pitch;
    for (int j = threadIdx.x; j < a.n_out; j += NT) out[j] = A[(j + a.out_off) * LP + l];
  }
}

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT)
    zpass_fast(const ZArgs a) {
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  float2* O = A + N * LP;  // OTF tile, same [kz][l] layout as A (pitch L)
  const int kx = blockIdx.y;
  const int ky0 = blockIdx.x * L;
  const size_t plane = (size_t)kx * a.zrows * a.Wy;
  const size_t oplane = (size_t)kx * N * a.Wy;
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (z < a.n_in && ky < a.Wy)
      cp_async8(&A[z * LP + l], &a.S[plane + (size_t)z * a.Wy + ky]);
    else
      A[z * LP + l] = make_float2(0.f, 0.f);
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
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  else
    cp_async_wait_all();
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  if (!conv) {
    for (int idx = threadIdx.x; idx < N * L; idx += NT) {
      const int kz = idx / L, l = idx % L;
      const int ky = ky0 + l;
      if (ky < a.Wy) a.otf_out[oplane + (size_t)kz * a.Wy + ky] = A[kz * LP + l];
    }
    return;
  }
  cp_async_wait_all();
  __syncthreads();
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int kz = idx / L, l = idx % L;
    A[kz * LP + l] = cmul(A[kz * LP + l], O[idx]);
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, true>(A, tw);
  for (int idx = threadIdx.x; idx < a.n_out * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (ky < a.Wy) a.S[plane + (size_t)z * a.Wy + ky] = A[(z + a.out_off) * LP + l];
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
