// One-launch y/z convolution for 3D plans: a persistent dataflow kernel.
//
// The 3-launch convolution (y fwd -> z * OTF * z -> y inv, rl_fast.cuh) moves
// the y-transformed spectrum S_B through HBM twice (write + read per launch
// boundary, 4 x 210 MB per convolution at C2).  A kx plane (Pz x Wy complex,
// 728 KB at C2) does not fit one SM, so the three stages cannot simply be one
// CTA's work.  Here they are TASKS of one persistent, cooperatively launched
// kernel:
//
//   Yf(p, c)  y-forward of rows [c*LY, ...) of plane p: S_A -> ring[p % R]
//   Z (p, c)  z-forward * OTF * z-inverse of ky columns [c*LZ, ...): in ring
//   Yi(p, c)  y-inverse of rows [c*LY, ...): ring -> S_A (cropped)
//
// with per-plane completion counters: Z(p,*) waits for all Yf(p,*), Yi(p,*)
// for all Z(p,*), and Yf(p,*) for Yi(p-R,*) (ring slot reuse).  One CTA per
// task; each CTA takes a ticket from one atomic counter when it starts and
// runs task[ticket].  The host orders the task list by "step"
// s = {Yf(s), Z(s-D), Yi(s-2D)} with R > 2D, so every task only waits on
// tasks with smaller tickets, i.e. on CTAs that started before it: no
// deadlock whatever the hardware's CTA dispatch order (the decoupled
// look-back argument), and no co-residency requirement.
//
// The ring (R planes, ~17-23 MB) is the only intermediate and is marked
// L2-persisting by the host, so S_B traffic stays on chip: HBM sees S_A read +
// S_A write + OTF once per convolution.
//
// Visibility: producers store with st.global, __syncthreads, then one thread
// fences (gpu scope) and bumps the counter; a consumer's thread 0 acquires the
// counter with ld.acquire.gpu and then executes a gpu-scope fence, which also
// invalidates the SM's L1 (CCTL.IVALL) so ring slots reused across planes are
// never read from stale L1 lines by the cp.async.ca copies that follow.
#pragma once
#include "rl_fast.cuh"

namespace vk {

template <int YR1, int YR2, int YL, int ZR1, int ZR2, int ZL>
struct DfCfg {
  static constexpr int NY = YR1 * YR2, NZ = ZR1 * ZR2;
  static constexpr int NT = FastCfg<YR1, YR2, YL>::NT > FastCfg<ZR1, ZR2, ZL>::NT ? FastCfg<YR1, YR2, YL>::NT
                                                                                  : FastCfg<ZR1, ZR2, ZL>::NT;
  static constexpr int WORK_Y = NY * (YL + 1), WORK_Z = NZ * (ZL + 1) + NZ * ZL;  // padded blocks (+ OTF tile)
  static constexpr int WORK = WORK_Y > WORK_Z ? WORK_Y : WORK_Z;
  static constexpr size_t smem = (size_t)((NY > NZ ? NY : NZ) + WORK) * sizeof(float2);
  // resident CTAs per SM the register budget is sized for (smem-limited)
  static constexpr int MINB_SMEM = (int)((227u * 1024u) / (smem + 1024u));
  static constexpr int MINB = MINB_SMEM < 1 ? 1 : (MINB_SMEM > 4 ? 4 : MINB_SMEM);
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// y transform of `nv` (<= L) rows: in rows of n_in samples (zero padded to
// N), out rows of n_out samples starting at transform index out_off.
template <int R1, int R2, int L, int NT, bool INV>
__device__ __forceinline__ void df_y_task(float2* A, const float2* tw, const float2* in, size_t in_pitch, int n_in,
                                          int nv, float2* out, size_t out_pitch, int n_out, int out_off) {
  constexpr int N = R1 * R2;
  for (int l = 0; l < L; ++l) {
    const float2* row = in + (size_t)(l < nv ? l : 0) * in_pitch;
    for (int i = reg::fresh_tid(); i < N; i += NT) {
      if (l < nv && i < n_in)
        cp_async8(&A[sw<L>(i, l)], &row[i]);
      else
        A[sw<L>(i, l)] = make_float2(0.f, 0.f);
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  reg::fft2<R1, R2, L, NT, INV>(A, tw);
  for (int l = 0; l < nv; ++l) {
    float2* o = out + (size_t)l * out_pitch;
    for (int j = reg::fresh_tid(); j < n_out; j += NT) o[j] = A[sw<L>(j + out_off, l)];
  }
}

// z forward * OTF * z inverse of L ky columns of one plane (rows pitch Wy).
template <int R1, int R2, int L, int NT>
__device__ __forceinline__ void df_z_task(float2* A, float2* O, const float2* tw, float2* plane, int Wy, int n_in,
                                          int n_out, int out_off, const float2* otf_plane, int ky0) {
  constexpr int N = R1 * R2;
  for (int idx = reg::fresh_tid(); idx < N * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (z < n_in && ky < Wy)
      cp_async8(&A[sw<L>(z, l)], &plane[(size_t)z * Wy + ky]);
    else
      A[sw<L>(z, l)] = make_float2(0.f, 0.f);
  }
  cp_async_commit();
  for (int idx = reg::fresh_tid(); idx < N * L; idx += NT) {
    const int kz = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (ky < Wy) cp_async8(&O[idx], &otf_plane[(size_t)kz * Wy + ky]);
  }
  cp_async_commit();
  cp_async_wait_1();
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false>(A, tw);
  cp_async_wait_all();
  __syncthreads();
  for (int idx = reg::fresh_tid(); idx < N * L; idx += NT) {
    const int kz = idx / L, l = idx % L;
    A[sw<L>(kz, l)] = cmul(A[sw<L>(kz, l)], O[idx]);
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, true>(A, tw);
  for (int idx = reg::fresh_tid(); idx < n_out * L; idx += NT) {
    const int z = idx / L, l = idx % L;
    const int ky = ky0 + l;
    if (ky < Wy) plane[(size_t)z * Wy + ky] = A[sw<L>(z + out_off, l)];
  }
}

template <int YR1, int YR2, int YL, int ZR1, int ZR2, int ZL>
__global__ void __launch_bounds__(DfCfg<YR1, YR2, YL, ZR1, ZR2, ZL>::NT, DfCfg<YR1, YR2, YL, ZR1, ZR2, ZL>::MINB)
    yzconv_dataflow(const DfArgs a) {
  using C = DfCfg<YR1, YR2, YL, ZR1, ZR2, ZL>;
  constexpr int NY = C::NY, NZ = C::NZ, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = smem;              // the twiddle table of the task's transform
  float2* W = smem + (NY > NZ ? NY : NZ);
  __shared__ int s_task;
  const Geom& g = a.g;
  int* const done0 = a.ctr + 1;  // done counters of task type t live at done0 + t*Hx
  // one task per CTA; the ticket is taken when the CTA starts, so every
  // dependency belongs to a CTA that started earlier (no deadlock, no
  // co-residency requirement).
  if (threadIdx.x == 0) s_task = atomicAdd(a.ctr, 1);
  __syncthreads();
  const int t = s_task;
  if (t >= a.ntasks) return;
  const unsigned code = a.tasks[t];
  const unsigned type = code >> 30, p = (code >> 14) & 0xffffu, c = code & 0x3fffu;
  if (type == DF_Z)
    reg::load_twiddles2<ZR1, ZR2>(tw, a.twz);
  else
    reg::load_twiddles2<YR1, YR2>(tw, a.twy);
  if (threadIdx.x == 0) {
    const int* dep = nullptr;
    int need = 0;
    if (type == DF_YF) {
      if ((int)p >= a.R) {
        dep = done0 + DF_YI * g.Hx + (p - a.R);
        need = a.nYi;
      }
    } else if (type == DF_Z) {
      dep = done0 + DF_YF * g.Hx + p;
      need = a.nYf;
    } else {
      dep = done0 + DF_Z * g.Hx + p;
      need = a.nZ;
    }
    if (dep) {
      unsigned ns = 32;
      while (ld_acquire(dep) < need) {
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : ns;
      }
    }
    __threadfence();  // acquire side; also drops stale L1 lines of reused ring slots
  }
  __syncthreads();
  float2* slot = a.ring + (size_t)(p % a.R) * g.Pz * g.Wy;
  if (type == DF_YF) {
    const int z0 = c * YL, nv = min(YL, g.Pz - z0);
    df_y_task<YR1, YR2, YL, NT, false>(W, tw, a.SA + ((size_t)p * g.Pz + z0) * g.Py, g.Py, g.Py, nv,
                                       slot + (size_t)z0 * g.Wy, g.Wy, g.Wy, 0);
  } else if (type == DF_Z) {
    df_z_task<ZR1, ZR2, ZL, NT>(W, W + NZ * (ZL + 1), tw, slot, g.Wy, g.Pz, g.Pz, g.cz,
                                a.otf + (size_t)p * NZ * g.Wy, c * ZL);
  } else {
    const int z0 = c * YL, nv = min(YL, g.Pz - z0);
    df_y_task<YR1, YR2, YL, NT, true>(W, tw, slot + (size_t)z0 * g.Wy, g.Wy, g.Wy, nv,
                                      a.SA + ((size_t)p * g.Pz + z0) * g.Py, g.Py, g.Py, g.cy);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(done0 + type * g.Hx + p, 1);
  }
}

}  // namespace vk
