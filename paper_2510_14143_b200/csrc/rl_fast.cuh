// Compile-time-length pass kernels (the fast path for the FFT lengths the
// configs use).  Same contracts as the generic kernels in rl_passes.cuh, with
// two differences that make every transform in-place in ONE shared buffer:
//
//  * the line transform is fft_reg.cuh's two-pass register FFT;
//  * the x crop offset cx (deconv.cpp:59-72) is realised as a phase ramp
//    exp(+2 pi i cx kx / Wx) folded into both OTFs at plan creation, so a
//    P-domain row lives at slots [cx, cx+Px) of its length-Wx line before the
//    forward transform AND after the inverse one.  The pointwise epilogue then
//    reads the model and writes the ratio / update into the same slot.
//    (Circular shift by cx, then by -cx: exact; the linear-convolution
//    support [0, P+K-1) still fits inside Wx.)
#pragma once
#include "fft_reg.cuh"
#include "rl_passes.cuh"

namespace vk {

template <int R1, int R2, int L>
struct FastCfg {
  static constexpr int N = R1 * R2;
  static constexpr int LP = L + 1;
  static constexpr int NT = ((L * (R1 > R2 ? R1 : R2)) + 31) / 32 * 32;
  static constexpr size_t smem = (size_t)(N * LP + N) * sizeof(float2);
};

template <int R1, int R2, int L>
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT)
    xpass_fast(const XArgs a) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  constexpr int Hx = N / 2 + 1;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  reg::load_twiddles(tw, a.plan.tw, N);
  const int z = blockIdx.y;
  const int y0 = blockIdx.x * 2 * L;
  const Geom& g = a.g;

  if (a.mode == XM_FWD) {
    // real rows [off, off+len) of each line, zero elsewhere
    for (int r = 0; r < 2 * L; ++r) {
      const int y = y0 + r;
      const bool yok = y < a.rows_y;
      const float* row = a.src + ((size_t)z * a.rows_y + (yok ? y : 0)) * a.len;
      for (int x = threadIdx.x; x < N; x += NT) {
        const int xs = x - a.xoff;
        float v = 0.f;
        if (yok && xs >= 0 && xs < a.len) v = row[xs] * a.scale;
        reinterpret_cast<float*>(&A[x * LP + (r % L)])[r / L] = v;
      }
    }
  } else {
    // Hermitian halves of row pair (l, L+l) -> Z[k] = Xa[k] + i Xb[k], k < N
    for (int idx = threadIdx.x; idx < Hx * L; idx += NT) {
      const int kx = idx / L, l = idx % L;
      const size_t row = ((size_t)kx * g.Pz + z) * g.Py;
      const int ya = y0 + l, yb = y0 + L + l;
      const float2 xa = ya < g.Py ? a.S[row + ya] : make_float2(0.f, 0.f);
      const float2 xb = yb < g.Py ? a.S[row + yb] : make_float2(0.f, 0.f);
      if (kx == 0 || 2 * kx == N) {
        A[kx * LP + l] = make_float2(xa.x, xb.x);  // imaginary parts of DC/Nyquist dropped (c2r)
      } else {
        A[kx * LP + l] = make_float2(xa.x - xb.y, xa.y + xb.x);
        A[(N - kx) * LP + l] = make_float2(xa.x + xb.y, xb.x - xa.y);
      }
    }
    __syncthreads();
    reg::fft2<R1, R2, L, NT, true>(A, tw);

    double accv[3] = {0.0, 0.0, 0.0};
    const bool last = a.mode == XM_UPDATE_LAST;
    const bool ratio = a.mode == XM_RATIO;
    for (int r = 0; r < 2 * L; ++r) {
      const int y = y0 + r;
      const int l = r % L, hi = r / L;
      if (y >= g.Py) {
        for (int x = threadIdx.x; x < g.Px; x += NT) reinterpret_cast<float*>(&A[(x + g.cx) * LP + l])[hi] = 0.f;
        continue;
      }
      const int iz = z - g.oz, iy = y - g.oy;
      const bool zyin = iz >= 0 && iz < g.Iz && iy >= 0 && iy < g.Iy;
      const float* orow = a.obs + ((size_t)clampi(iz, 0, g.Iz - 1) * g.Iy + clampi(iy, 0, g.Iy - 1)) * g.Ix;
      float* erow = a.est + ((size_t)z * g.Py + y) * g.Px;
      float* outrow = last ? a.out + ((size_t)clampi(iz, 0, g.Iz - 1) * g.Iy + clampi(iy, 0, g.Iy - 1)) * g.Ix
                           : nullptr;
      for (int x = threadIdx.x; x < g.Px; x += NT) {
        float* slot = reinterpret_cast<float*>(&A[(x + g.cx) * LP + l]) + hi;
        const float m = *slot;
        const int ix = x - g.ox;
        const bool inside = zyin && ix >= 0 && ix < g.Ix;
        const float o = __ldg(&orow[clampi(ix, 0, g.Ix - 1)]);
        float val;
        if (ratio) {
          const float mm = fmaxf(m, kEps);
          val = o / mm;
          if (inside) accv[0] += (double)o * (double)logf(mm) - (double)mm;
        } else {
          val = fmaxf(erow[x] * m, 0.f);
          if (!last) erow[x] = val;
          if (inside) {
            accv[0] += val;
            accv[1] += (double)val * val;
            accv[2] += (double)val * o;
            if (last) outrow[ix] = val;
          }
        }
        *slot = val;
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
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT)
    ypass_fast(const YArgs a) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  reg::load_twiddles(tw, a.plan.tw, N);
  const int line0 = blockIdx.x * L;
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    const bool ok = line < a.nlines;
    const float2* in = a.in + (size_t)(ok ? line : 0) * a.in_pitch;
    for (int i = threadIdx.x; i < N; i += NT)
      A[i * LP + l] = (ok && i < a.n_in) ? in[i] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  if (a.mode == YM_INV) {
    reg::fft2<R1, R2, L, NT, true>(A, tw);
  } else {
    reg::fft2<R1, R2, L, NT, false>(A, tw);
    if (a.mode == YM_CONV) {
      for (int l = 0; l < L; ++l) {
        const int line = line0 + l;
        if (line >= a.nlines) break;
        const float2* o = a.otf + (size_t)line * N;
        for (int k = threadIdx.x; k < N; k += NT) A[k * LP + l] = cmul(A[k * LP + l], __ldg(&o[k]));
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
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT)
    zpass_fast(const ZArgs a) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, LP = C::LP, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;
  float2* A = smem + N;
  reg::load_twiddles(tw, a.plan.tw, N);
  const int kx = blockIdx.y;
  const int ky0 = blockIdx.x * L;
  const size_t plane = (size_t)kx * a.zrows * a.Wy;
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    A[z * LP + l] = (z < a.n_in && ky < a.Wy) ? a.S[plane + (size_t)z * a.Wy + ky] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  const size_t oplane = (size_t)kx * N * a.Wy;
  if (a.mode == ZM_FWD_OUT) {
    for (int idx = threadIdx.x; idx < N * L; idx += NT) {
      const int kz = idx / L, l = idx % L;
      const int ky = ky0 + l;
      if (ky < a.Wy) a.otf_out[oplane + (size_t)kz * a.Wy + ky] = A[kz * LP + l];
    }
    return;
  }
  for (int idx = threadIdx.x; idx < N * L; idx += NT) {
    const int kz = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (ky < a.Wy) A[kz * LP + l] = cmul(A[kz * LP + l], __ldg(&a.otf[oplane + (size_t)kz * a.Wy + ky]));
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
