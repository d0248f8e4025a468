// Compile-time-length pass kernels (the fast path for the FFT lengths the
// configs use).  Same contracts as the generic kernels in rl_passes.cuh, with
// these differences:
//
//  * the line transform is fft_reg.cuh's two-pass register FFT, in place in
//    ONE shared buffer with the padded line layout sw<L>(i, l) = i*(L+1) + l;
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

// Reciprocal / natural log of a NORMAL float (the ratio's max(model, 1e-12)):
// the .ftz approximations, without the denormal-range fix-ups __fdividef /
// __logf carry (same values for normal inputs; 2 ulp / 2^-21 abs as before).
__device__ __forceinline__ float rcp_n(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float log_n(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r * 0.693147180559945309f;
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// mbarrier / TMA helpers (tx-count completion, bulk and tensor copies)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"((unsigned)__cvta_generic_to_shared(smem_src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"((unsigned)__cvta_generic_to_shared(smem_src)), "r"(bytes)
               : "memory");
}
// generic-proxy shared-memory writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// End-of-kernel bulk / TMA stores: wait only until the shared source has
// been read (the writes complete with the grid), so the CTA's slot frees
// without waiting out the store's global write latency (y passes -4 to -6%,
// C2 +1.1%: profiles/r02/bulk_wait_read_ab.txt).
__device__ __forceinline__ void bulk_commit_and_release() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          (unsigned)__cvta_generic_to_shared(smem_dst)),
      "l"(map), "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Programmatic dependent launch: the host launches the fast pass kernels
// with cudaLaunchAttributeProgrammaticStreamSerialization.  Each grid lets
// the next one launch as soon as all of its CTAs are resident (the next
// grid's CTAs then fill the SMs our tail wave frees), and waits for the
// previous grid to complete and flush before touching its results.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Group index of thread groups of L lanes, permuted so that the two groups
// of a half-warp (2m, 2m+1) address rows m and m+8 (within each 16 groups)
// when L = 8: rows one apart share a bank pair under the (L+1) pad, rows
// eight apart do not (see reg::fft2 pass 2).  Bijective on [0, ngroups).
template <int L>
__device__ __forceinline__ int group_remap(int g, int ngroups) {
  if (L == 8 && g < (ngroups / 16) * 16) return (g & ~15) | ((g >> 1) & 7) | ((g & 1) << 3);
  return g;
}

template <int R1, int R2, int L, bool OTF_PREFETCH = false>
struct FastCfg {
  static_assert((L & (L - 1)) == 0, "L must be a power of two (cheap line/index split)");
  static constexpr int N = R1 * R2;
  static constexpr int NT = ((L * (R1 > R2 ? R1 : R2)) + 31) / 32 * 32;
  static constexpr int DATA = N * (L + 1);  // padded line block, see reg::sw
  static constexpr size_t smem = (size_t)(DATA + N + (OTF_PREFETCH ? N * L : 0)) * sizeof(float2);
  static constexpr size_t smem_x = (size_t)DATA * sizeof(float2);  // x pass: twiddles from global
};

// TWG: pass-2 twiddles read from global memory (L1) instead of a shared
// table, when dropping the table buys one more resident CTA per SM.
// MINB: resident CTAs per SM the register allocation must allow.  PB: the
// partial-chunk epilogue batches its loads like the full one (worth its
// registers only where partial chunks are common, e.g. Ix = 1000).
//
// Row pairing: the CTA's 2L rows y0 .. y0+2L-1 are packed as line l = rows
// (y0+2l, y0+2l+1), so both halves of a line are adjacent in S_A (one
// 16-byte access) and in the TMA-staged tile.
// STAGED (xpass_tma, RATIO/UPDATE): the CTA's spectrum rows arrive as TMA
// boxes {2L rows, 1, BK kx} of the tensor S_A {Py, Pz, Hx} -- a dense [kx][2L]
// tile in the same shared buffer -- and the C2R transform's first pass reads
// the Hermitian pairs straight from it (reg::fft2 STG), so there is no pack
// phase and no per-thread global load of the spectrum.
template <int R1, int R2, int L, bool TWG, bool PB, bool STAGED>
__device__ __forceinline__ void xpass_body(const XArgs& a, const CUtensorMap* xmap) {
  using C = FastCfg<R1, R2, L>;
  constexpr int N = C::N, NT = C::NT;
  constexpr int Hx = N / 2 + 1;
  constexpr int NW = NT / 32;
  constexpr int U = 4;
  constexpr int CH = 32 * U;  // samples per work item
  extern __shared__ __align__(128) float2 smem[];
  const float2* tw = TWG ? a.plan.tw2 : smem;
  float2* A = TWG ? smem : smem + (N + 15) / 16 * 16;  // 128-byte aligned (TMA boxes land here)
  pdl_trigger();
  if (!TWG) reg::load_twiddles2<R1, R2>(smem, a.plan.tw);  // constant table: before the wait
  const int z = blockIdx.y + a.zoff;
  const int y0 = blockIdx.x * 2 * L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Geom& g = a.g;

  if (a.mode == XM_FWD) {
    pdl_wait();
    // real rows (2l, 2l+1) -> line l, samples at slots [xoff, xoff+len)
    const int nch = (N + CH - 1) / CH;
    for (int item = warp; item < L * nch; item += NW) {
      const int l = item / nch, x0 = (item % nch) * CH;
      const int ya = y0 + 2 * l, yb = ya + 1;
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
    // Hermitian halves of row pair (2l, 2l+1) -> Z[k] = Xa[k] + i Xb[k], k < N.
    // NT is a multiple of L, so a thread keeps one line l and strides kx by
    // NT/L; spectrum offsets are 32-bit and incremental.
    constexpr int KS = NT / L;  // kx stride per thread
    const float2 zero = make_float2(0.f, 0.f);
    __shared__ uint64_t xbar;
    if (STAGED) {
      if (threadIdx.x == 0) {
        mbar_init(&xbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
    }
    // L2 prefetch at entry: every load round of this CTA after the first, and
    // the epilogue's observed / estimate rows, then hit L2 instead of HBM (the
    // epilogue walks its rows in ~12 dependent load rounds per warp).
    auto prefetch_tile = [&](const int zz, const int yy0, const int mask) {
      if (mask & 1) {  // (also ahead of the TMA boxes: issued before the PDL wait)
        const unsigned plane = (unsigned)g.Pz * g.Py;
        const float2* base = a.S + (unsigned)zz * g.Py + yy0;
        for (int i = threadIdx.x; i < 2 * Hx; i += NT)
          if (yy0 + (i & 1) * L < g.Py) prefetch_l2(base + (unsigned)(i >> 1) * plane + (i & 1) * L);
      }
      if (mask & 2) {
        const int iz = clampi(zz - g.oz, 0, g.Iz - 1);
        const int nlo = (g.Ix + 31) / 32 + 1, nle = (g.Px + 31) / 32 + 1;
        const bool upd = a.mode != XM_RATIO;
        const int per = nlo + (upd ? nle : 0);
        for (int i = threadIdx.x; i < 2 * L * per; i += NT) {
          const int r = i / per, k = i - r * per;
          const int y = min(yy0 + r, g.Py - 1);
          if (k < nlo) {
            const int iy = clampi(y - g.oy, 0, g.Iy - 1);
            const float* row = a.obs + ((size_t)iz * g.Iy + iy) * g.Ix;
            prefetch_l2(row + min(k * 32, g.Ix - 1));
          } else {
            const float* row = a.est + ((size_t)zz * g.Py + y) * g.Px;
            prefetch_l2(row + min((k - nlo) * 32, g.Px - 1));
          }
        }
      }
    };
    prefetch_tile(z, y0, a.pf & 3);
    // the prefetches are hints (L2 is coherent): issued before the wait, they
    // overlap the previous pass's tail
    pdl_wait();
    if (STAGED) {
      // rows [y0, y0+2L) of kx in [b*BK, b*BK+BK): box b lands at A + b*BK*2L;
      // rows >= Py and kx >= Hx arrive as zeros (TMA out-of-bounds fill)
      if (threadIdx.x == 0) {
        mbar_expect_tx(&xbar, (unsigned)(a.tnb * a.tbk * 2 * L * sizeof(float2)));
        for (int b = 0; b < a.tnb; ++b) tma_load_3d(A + b * a.tbk * 2 * L, xmap, &xbar, y0, z, b * a.tbk);
      }
    } else {
      const int l = threadIdx.x & (L - 1);
      const int ya = y0 + 2 * l, yb = ya + 1;
      const bool va = ya < g.Py, vb = yb < g.Py;
      const float2* Sa = a.S + ((unsigned)z * g.Py + (va ? ya : 0));
      const float2* Sb = a.S + ((unsigned)z * g.Py + (vb ? yb : 0));
      const unsigned plane = (unsigned)g.Pz * g.Py;
      const bool vec = (g.Py & 1) == 0;  // then vb == va (ya even)
#ifndef VK_XLOAD_U
#define VK_XLOAD_U 6  // C2 x passes -1.8% vs 4 (and no spill at 576); 8 / 12: -2.0% / +-0
#endif
      constexpr int UL = VK_XLOAD_U;  // spectrum loads in flight per thread (profiles/r02/xload_u_ab.txt)
      for (int kx0 = group_remap<L>(threadIdx.x / L, KS); kx0 < Hx; kx0 += KS * UL) {
        float2 xa[UL], xb[UL];
#pragma unroll
        for (int u = 0; u < UL; ++u) {
          const int kx = kx0 + u * KS;
          const bool ok = kx < Hx;
          if (vec) {  // rows 2l, 2l+1 adjacent and 16-byte aligned: one load
            const float4 v = (ok && va) ? *reinterpret_cast<const float4*>(Sa + (unsigned)kx * plane)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
            xa[u] = make_float2(v.x, v.y);
            xb[u] = make_float2(v.z, v.w);
          } else {
            xa[u] = (ok && va) ? Sa[(unsigned)kx * plane] : zero;
            xb[u] = (ok && vb) ? Sb[(unsigned)kx * plane] : zero;
          }
        }
#pragma unroll
        for (int u = 0; u < UL; ++u) {
          const int kx = kx0 + u * KS;
          if (kx >= Hx) break;
          if (kx == 0 || 2 * kx == N) {
            A[sw<L>(kx, l)] = make_float2(xa[u].x, xb[u].x);  // imaginary parts of DC/Nyquist dropped (c2r)
          } else {
            A[sw<L>(kx, l)] = make_float2(xa[u].x - xb[u].y, xa[u].y + xb[u].x);
            A[sw<L>(N - kx, l)] = make_float2(xa[u].x + xb[u].y, xb[u].x - xa[u].y);
          }
        }
      }
    }
    // per-row offsets / flags of the epilogue, once per CTA (visible after
    // the transform's barriers): observed row (clamped = edge replicate),
    // estimate row, bit 0 row exists (y < Py), bit 1 row inside the image
    __shared__ unsigned s_oo[2 * L], s_eo[2 * L];
    __shared__ unsigned char s_fl[2 * L];
    if (threadIdx.x < 2 * L) {
      const int r = threadIdx.x, y = y0 + r;
      const bool v = y < g.Py;
      const int iy = y - g.oy, iz = z - g.oz;
      const bool in = v && iz >= 0 && iz < g.Iz && iy >= 0 && iy < g.Iy;
      s_oo[r] = ((unsigned)clampi(iz, 0, g.Iz - 1) * g.Iy + clampi(iy, 0, g.Iy - 1)) * (unsigned)g.Ix;
      s_eo[r] = ((unsigned)z * g.Py + (v ? y : 0)) * (unsigned)g.Px;
      s_fl[r] = (v ? 1 : 0) | (in ? 2 : 0);
    }
    if (STAGED) mbar_wait(&xbar, 0);
    __syncthreads();
    reg::fft2<R1, R2, L, NT, true, L + 1, TWG, 1, STAGED>(A, tw);

    const bool last = a.mode == XM_UPDATE_LAST;
    const bool ratio = a.mode == XM_RATIO;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    // Work items (line l, chunk c), one warp each.  Chunks c < nci cover the
    // interior columns [ox, ox+Ix) in CH-sample pieces aligned at ox (U
    // samples of both rows of the line per lane, no x clamp); the remaining
    // chunks cover the 2*ox pad columns, one sample per lane, whose observed
    // value is the replicated edge (deconv.cpp:221-237) and which never enter
    // the sums.
    const int nci = (g.Ix + CH - 1) / CH;
    const int npad = g.Px - g.Ix;
    const int nch = nci + (npad + 31) / 32;
    // items (l, ch) walked with incremental carries instead of div/mod
    int l = 0, ch = warp;
    while (ch >= nch) {
      ch -= nch;
      ++l;
    }
    for (; l < L; ch += NW) {
      while (ch >= nch) {
        ch -= nch;
        ++l;
      }
      if (l >= L) break;
      const int fa = s_fl[2 * l], fb = s_fl[2 * l + 1];
      const bool va = fa & 1, vb = fb & 1, ina = fa & 2, inb = fb & 2;
      const unsigned oa_off = s_oo[2 * l], ob_off = s_oo[2 * l + 1];
      float* ea = a.est + s_eo[2 * l];
      float* eb = a.est + s_eo[2 * l + 1];
      if (ch >= nci) {
        // pad columns: x in [0, ox) and [ox+Ix, Px)
        const int p = (ch - nci) * 32 + lane;
        if (p < npad) {
          const bool left = p < g.ox;
          const int x = left ? p : p + g.Ix;
          const int xo = left ? 0 : g.Ix - 1;
          const int sidx = sw<L>(x + g.cx, l);
          const float2 m = A[sidx];
          float2 val;
          if (ratio) {
            val = make_float2(va ? __ldg(a.obs + oa_off + xo) * rcp_n(fmaxf(m.x, kEps)) : 0.f,
                              vb ? __ldg(a.obs + ob_off + xo) * rcp_n(fmaxf(m.y, kEps)) : 0.f);
          } else {
            val = make_float2(va ? fmaxf(ea[x] * m.x, 0.f) : 0.f, vb ? fmaxf(eb[x] * m.y, 0.f) : 0.f);
            if (!last) {
              if (va) ea[x] = val.x;
              if (vb) eb[x] = val.y;
            }
          }
          A[sidx] = val;
        }
        continue;
      }
      const int c0 = ch * CH;  // interior column of this chunk's first sample
      const int x0 = g.ox + c0;
      const int s0 = sw<L>(x0 + lane + g.cx, l);
      const float* oa2 = a.obs + oa_off + c0 + lane;
      const float* ob2 = a.obs + ob_off + c0 + lane;
      float* ea2 = ea + x0 + lane;
      float* eb2 = eb + x0 + lane;
      if (va && vb && c0 + CH <= g.Ix) {
        // full chunk of two existing rows (the common case): no predicates
        float2 m[U];
        float o_a[U], o_b[U], e_a[U], e_b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          m[u] = A[s0 + u * 32 * (L + 1)];
          o_a[u] = __ldg(oa2 + u * 32);
          o_b[u] = __ldg(ob2 + u * 32);
          if (!ratio) {
            e_a[u] = ea2[u * 32];
            e_b[u] = eb2[u * 32];
          }
        }
        float fa0 = 0.f, fa1 = 0.f, fa2 = 0.f, fb0 = 0.f, fb1 = 0.f, fb2 = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float2 val;
          if (ratio) {
            // fast reciprocal/log (<= 2 ulp / 2^-21 abs): the f32 path's own
            // rounding (~1e-7 rel) dominates either way
            const float ma = fmaxf(m[u].x, kEps), mb = fmaxf(m[u].y, kEps);
            val = make_float2(o_a[u] * rcp_n(ma), o_b[u] * rcp_n(mb));
            fa0 += fmaf(o_a[u], log_n(ma), -ma);
            fb0 += fmaf(o_b[u], log_n(mb), -mb);
          } else {
            val = make_float2(fmaxf(e_a[u] * m[u].x, 0.f), fmaxf(e_b[u] * m[u].y, 0.f));
            if (!last) {
              ea2[u * 32] = val.x;
              eb2[u * 32] = val.y;
            } else {
              if (ina) a.out[oa_off + c0 + lane + u * 32] = val.x;
              if (inb) a.out[ob_off + c0 + lane + u * 32] = val.y;
            }
            fa0 += val.x;
            fa1 = fmaf(val.x, val.x, fa1);
            fa2 = fmaf(val.x, o_a[u], fa2);
            fb0 += val.y;
            fb1 = fmaf(val.y, val.y, fb1);
            fb2 = fmaf(val.y, o_b[u], fb2);
          }
          A[s0 + u * 32 * (L + 1)] = val;
        }
        if (ina) {
          acc0 += fa0;
          acc1 += fa1;
          acc2 += fa2;
        }
        if (inb) {
          acc0 += fb0;
          acc1 += fb1;
          acc2 += fb2;
        }
        continue;
      }
      // partial chunk (last interior piece or a missing second row): the
      // same batched loads, predicated per lane
      if (PB) {
        float fa0 = 0.f, fa1 = 0.f, fa2 = 0.f, fb0 = 0.f, fb1 = 0.f, fb2 = 0.f;
        float2 m[U];
        float o_a[U], o_b[U], e_a[U], e_b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const bool ok = c0 + u * 32 + lane < g.Ix;
          m[u] = ok ? A[s0 + u * 32 * (L + 1)] : make_float2(0.f, 0.f);
          o_a[u] = ok ? __ldg(oa2 + u * 32) : 0.f;
          o_b[u] = ok ? __ldg(ob2 + u * 32) : 0.f;
          if (!ratio) {
            e_a[u] = (ok && va) ? ea2[u * 32] : 0.f;
            e_b[u] = (ok && vb) ? eb2[u * 32] : 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c >= g.Ix) break;
          float2 val;
          if (ratio) {
            const float ma = fmaxf(m[u].x, kEps), mb = fmaxf(m[u].y, kEps);
            val = make_float2(va ? o_a[u] * rcp_n(ma) : 0.f, vb ? o_b[u] * rcp_n(mb) : 0.f);
            fa0 += fmaf(o_a[u], log_n(ma), -ma);
            fb0 += fmaf(o_b[u], log_n(mb), -mb);
          } else {
            val = make_float2(fmaxf(e_a[u] * m[u].x, 0.f), fmaxf(e_b[u] * m[u].y, 0.f));
            if (!last) {
              if (va) ea2[u * 32] = val.x;
              if (vb) eb2[u * 32] = val.y;
            } else {
              if (ina) a.out[oa_off + c] = val.x;
              if (inb) a.out[ob_off + c] = val.y;
            }
            fa0 += val.x;
            fa1 = fmaf(val.x, val.x, fa1);
            fa2 = fmaf(val.x, o_a[u], fa2);
            fb0 += val.y;
            fb1 = fmaf(val.y, val.y, fb1);
            fb2 = fmaf(val.y, o_b[u], fb2);
          }
          A[s0 + u * 32 * (L + 1)] = val;
        }
        if (ina) {
          acc0 += fa0;
          acc1 += fa1;
          acc2 += fa2;
        }
        if (inb) {
          acc0 += fb0;
          acc1 += fb1;
          acc2 += fb2;
        }
      } else {  // sample by sample (fewest registers)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + u * 32 + lane;
          if (c >= g.Ix) break;
          const int sidx = s0 + u * 32 * (L + 1);
          const float2 m = A[sidx];
          const float o_a = __ldg(oa2 + u * 32), o_b = __ldg(ob2 + u * 32);
          float2 val;
          if (ratio) {
            const float ma = fmaxf(m.x, kEps), mb = fmaxf(m.y, kEps);
            val = make_float2(va ? o_a * rcp_n(ma) : 0.f, vb ? o_b * rcp_n(mb) : 0.f);
            if (ina) acc0 += fmaf(o_a, log_n(ma), -ma);
            if (inb) acc0 += fmaf(o_b, log_n(mb), -mb);
          } else {
            val = make_float2(va ? fmaxf(ea2[u * 32] * m.x, 0.f) : 0.f, vb ? fmaxf(eb2[u * 32] * m.y, 0.f) : 0.f);
            if (!last) {
              if (va) ea2[u * 32] = val.x;
              if (vb) eb2[u * 32] = val.y;
            }
            if (ina) {
              acc0 += val.x;
              acc1 += (double)val.x * val.x;
              acc2 += (double)val.x * o_a;
              if (last) a.out[oa_off + c] = val.x;
            }
            if (inb) {
              acc0 += val.y;
              acc1 += (double)val.y * val.y;
              acc2 += (double)val.y * o_b;
              if (last) a.out[ob_off + c] = val.y;
            }
          }
          A[sidx] = val;
        }
      }
    }
    {  // this block's partials in the iteration's slot (reduce_iter_partials_kernel)
      double* dst = a.acc + ((size_t)(blockIdx.y + a.zoff) * gridDim.x + blockIdx.x) * 4;
      if (ratio) {
        double v1[1] = {acc0};
        block_partial<1>(v1, dst);
      } else {
        double v3[3] = {acc0, acc1, acc2};
        block_partial<3>(v3, dst + 1);
      }
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
  reg::fft2<R1, R2, L, NT, false, L + 1, TWG>(A, tw);
  {
    constexpr int KS = NT / L;
    const int l = threadIdx.x & (L - 1);
    const int ya = y0 + 2 * l;
    const bool va = ya < a.rows_y, vb = ya + 1 < a.rows_y;
    // rows (2l, 2l+1) adjacent: one 16-byte store when rows_y is even
    const bool vec = vb && (a.rows_y & 1) == 0;
    float2* Sa = a.S + ((unsigned)z * a.rows_y + ya);
    const unsigned plane = (unsigned)a.rows_z * a.rows_y;
    for (int kx = group_remap<L>(threadIdx.x / L, KS); kx < Hx; kx += KS) {
      const float2 zk = A[sw<L>(kx, l)];
      const float2 zn = A[sw<L>(kx == 0 ? 0 : N - kx, l)];
      const float2 xa = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
      const float2 xb = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
      float2* d = Sa + (unsigned)kx * plane;
      if (vec) {
        *reinterpret_cast<float4*>(d) = make_float4(xa.x, xa.y, xb.x, xb.y);
      } else {
        if (va) d[0] = xa;
        if (vb) d[1] = xb;
      }
    }
  }
}

template <int R1, int R2, int L, bool TWG, int MINB, bool PB>
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT, MINB == 1 ? 0 : MINB)  // 1: leave the heuristic alone
    xpass_fast(const __grid_constant__ XArgs a) {
  xpass_body<R1, R2, L, TWG, PB, false>(a, nullptr);
}

template <int R1, int R2, int L, bool TWG, int MINB, bool PB>
__global__ void __launch_bounds__(FastCfg<R1, R2, L>::NT, MINB == 1 ? 0 : MINB)
    xpass_tma(const __grid_constant__ XTmaArgs t) {
  xpass_body<R1, R2, L, TWG, PB, true>(t.x, &t.map);
}

// PREF: the CONV mode stages the OTF tile in shared memory with cp.async
// while the forward transform runs; without it (long lines, where the tile
// would cost a resident CTA) the multiply reads the OTF from global directly.
template <int R1, int R2, int L, bool TWG, bool PREF>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT)
    ypass_fast(const YArgs a) {
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = TWG ? nullptr : smem;  // TWG: pass-2 twiddles from global (a.plan.tw2)
  float2* A = TWG ? smem : smem + N;
  float2* O = A + C::DATA;  // OTF tile [l][k] (CONV only)
  const int line0 = blockIdx.x * L;
  pdl_trigger();
  pdl_wait();
  // async copies: the L input rows (zero padding written directly)
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    const bool ok = line < a.nlines;
    const float2* in = a.in + (size_t)(ok ? y_line(a, line) : 0) * a.in_pitch;
    for (int i = threadIdx.x; i < N; i += NT) {
      if (ok && i < a.n_in)
        cp_async8(&A[sw<L>(i, l)], &in[i]);
      else
        A[sw<L>(i, l)] = make_float2(0.f, 0.f);
    }
  }
  cp_async_commit();
  if (PREF && a.mode == YM_CONV) {
    for (int l = 0; l < L; ++l) {
      const int line = line0 + l;
      if (line >= a.nlines) break;
      const float2* o = a.otf + (size_t)line * N;
      for (int k = threadIdx.x; k < N; k += NT) cp_async8(&O[l * N + k], &o[k]);
    }
    cp_async_commit();
  }
  if (!TWG) reg::load_twiddles2<R1, R2>(tw, a.plan.tw);
  const float2* twp = TWG ? a.plan.tw2 : tw;
  if (PREF && a.mode == YM_CONV)
    cp_async_wait_1();  // input rows landed, OTF may still fly
  else
    cp_async_wait_all();
  __syncthreads();
  if (a.mode == YM_INV) {
    reg::fft2<R1, R2, L, NT, true, L + 1, TWG>(A, twp);
  } else {
    reg::fft2<R1, R2, L, NT, false, L + 1, TWG>(A, twp);
    if (a.mode == YM_CONV) {
      if (PREF) {
        cp_async_wait_all();
        __syncthreads();
        for (int idx = threadIdx.x; idx < N * L; idx += NT) {
          const int k = idx / L, l = idx % L;
          A[sw<L>(k, l)] = cmul(A[sw<L>(k, l)], O[l * N + k]);
        }
      } else {
        // line-major walk: coalesced OTF reads, stride L+1 (odd) in smem
        for (int l = 0; l < L; ++l) {
          const int line = line0 + l;
          if (line >= a.nlines) break;
          const float2* o = a.otf + (size_t)line * N;
          for (int k = threadIdx.x; k < N; k += NT) A[sw<L>(k, l)] = cmul(A[sw<L>(k, l)], __ldg(o + k));
        }
      }
      __syncthreads();
      reg::fft2<R1, R2, L, NT, true, L + 1, TWG>(A, twp);
    }
  }
  for (int l = 0; l < L; ++l) {
    const int line = line0 + l;
    if (line >= a.nlines) break;
    float2* out = a.out + (size_t)y_line(a, line) * a.out_pitch;
    for (int j = threadIdx.x; j < a.n_out; j += NT) out[j] = A[sw<L>(j + a.out_off, l)];
  }
}

// TWG / PREF / MINB as for the x and y passes: pass-2 twiddles from global,
// OTF tile staged in shared memory during the forward transform (else read
// from global in the multiply), and the resident CTAs per SM to allow for.
template <int R1, int R2, int L, bool TWG, bool PREF, int MINB>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT, MINB == 1 ? 0 : MINB)
    zpass_fast(const ZArgs a) {
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, NT = C::NT;
  extern __shared__ float2 smem[];
  float2* tw = TWG ? nullptr : smem;
  float2* A = TWG ? smem : smem + N;
  float2* O = A + C::DATA;  // OTF tile, [kz][l] row-major (pitch L)
  // NT is a multiple of L: a thread owns one column l (ky = ky0 + l) and
  // strides z by ZS = NT/L; offsets are 32-bit and compile-time unrolled.
  constexpr int ZS = NT / L;
  constexpr int IT = (N + ZS - 1) / ZS;
  const int kx = blockIdx.y;
  const int l = threadIdx.x & (L - 1), z0 = threadIdx.x / L;
  const int ky = blockIdx.x * L + l;
  const bool kok = ky < a.Wy;
  float2* col = a.S + ((unsigned)kx * a.zrows * a.Wy + (kok ? ky : 0));
  const unsigned oplane = (unsigned)kx * N * a.Wy + (kok ? ky : 0);
  const unsigned Wy = a.Wy;
  pdl_trigger();
  pdl_wait();
#pragma unroll
  for (int k = 0; k < IT; ++k) {
    const int z = z0 + k * ZS;
    if (z < N) {
      if (kok && z < a.n_in)
        cp_async8(&A[sw<L>(z, l)], &col[(unsigned)z * Wy]);
      else
        A[sw<L>(z, l)] = make_float2(0.f, 0.f);
    }
  }
  cp_async_commit();
  const bool conv = a.mode == ZM_CONV;
  if (PREF && conv) {
    const float2* o = a.otf + oplane;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int z = z0 + k * ZS;
      if (z < N && kok) cp_async8(&O[z * L + l], &o[(unsigned)z * Wy]);
    }
    cp_async_commit();
  }
  if (!TWG) reg::load_twiddles2<R1, R2>(tw, a.plan.tw);
  const float2* twp = TWG ? a.plan.tw2 : tw;
  if (PREF && conv)
    cp_async_wait_1();
  else
    cp_async_wait_all();
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false, L + 1, TWG>(A, twp);
  if (!conv) {
    float2* o = a.otf_out + oplane;
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int z = z0 + k * ZS;
      if (z < N && kok) o[(unsigned)z * Wy] = A[sw<L>(z, l)];
    }
    return;
  }
  if (PREF) {
    cp_async_wait_all();
    __syncthreads();
  }
  const float2* og = a.otf + oplane;
#pragma unroll
  for (int k = 0; k < IT; ++k) {
    const int z = z0 + k * ZS;
    if (z < N) A[sw<L>(z, l)] = cmul(A[sw<L>(z, l)], PREF ? O[z * L + l] : (kok ? __ldg(&og[(unsigned)z * Wy]) : make_float2(0.f, 0.f)));
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, true, L + 1, TWG>(A, twp);
  if (kok) {
    for (int z = z0; z < a.n_out; z += ZS) col[(unsigned)z * Wy] = A[sw<L>(z + a.out_off, l)];
  }
}

// ---- z convolution with a TMA-staged column tile --------------------------
// The (ky block of 16) x (Pz rows) column tile of kx plane `kx` is one
// cp.async.bulk.tensor.3d load (box {16, Pz, 1} of the tensor
// [Hx][zrows][Wy] complex64, 8-byte elements) into a dense [z][16] shared
// tile, completion tracked by an mbarrier; the transform then runs on the
// unpadded layout (16-lane rows cover all 32 banks, so the (L+1) pad is not
// needed at L = 16).  Rows Pz..N-1 are zeroed by the other threads while the
// copy flies.  The OTF is read from global in the multiply.
// (ZTmaArgs: fast_table.h)

// First stored column of the half-OTF box serving tile [ky0, ky0+16): the
// smallest min(ky, Wy - ky) of its columns (they span <= 16 columns), rounded
// down to even -- a TMA box must start 16-byte aligned in its inner
// dimension -- so the half box is kHalfBox = 18 columns wide.  A negative
// start reads zeros out of bounds (lanes with ky >= Wy).
constexpr int kHalfBox = 18;
__device__ __forceinline__ int half_box_start(int ky0, int Wy) {
  const int s = ky0 + 15 <= Wy / 2 ? ky0 : min(ky0, Wy - ky0 - 15);
  return s & ~1;
}

template <int R1, int R2, bool TWG, int MINB>
__global__ void __launch_bounds__(FastCfg<R1, R2, 16, true>::NT, MINB == 1 ? 0 : MINB)
    zpass_tma(const __grid_constant__ ZTmaArgs ta) {
  constexpr int L = 16;
  using C = FastCfg<R1, R2, L, true>;
  constexpr int N = C::N, NT = C::NT;
  constexpr int ZS = NT / L;
  constexpr int IT = (N + ZS - 1) / ZS;
  // scalar fields straight from param space (a reference to the struct would
  // force a local copy)
  const int n_in = ta.z.n_in, n_out = ta.z.n_out, out_off = ta.z.out_off, zrows = ta.z.zrows;
  float2* const S = ta.z.S;
  const float2* const otf = ta.z.otf;
  extern __shared__ __align__(128) float2 smem[];
  float2* tw = TWG ? nullptr : smem;
  float2* A = TWG ? smem : smem + (N + 15) / 16 * 16;  // dense [z][16], 128-B aligned (TMA destination)
  float2* O = A + N * L;              // OTF tile [kz][16] (half OTF: [kz][kHalfBox]) when ta.otf_tma
  __shared__ uint64_t bar, obar;
  const bool otma = ta.otf_tma != 0;
  const int kx = blockIdx.y, ky0 = blockIdx.x * L;
  const int kxo = kx + ta.kx0;  // absolute kx plane (OTF, factors)
  const int l = threadIdx.x & (L - 1), z0 = threadIdx.x / L;
  const int ky = ky0 + l;
  const unsigned Wy = ta.z.Wy;
  const bool kok = ky < (int)Wy;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&obar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!TWG) reg::load_twiddles2<R1, R2>(tw, ta.z.plan.tw);
  const float2* twp = TWG ? ta.z.plan.tw2 : tw;
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (unsigned)(n_in * L * sizeof(float2)));
    tma_load_3d(A, &ta.map, &bar, ky0, 0, kx);
    if (otma) {  // the OTF tile lands while the forward transform runs
      mbar_expect_tx(&obar, (unsigned)(N * (ta.otf_half ? kHalfBox : L) * sizeof(float2)));
      tma_load_3d(O, &ta.omap, &obar, ta.otf_half ? half_box_start(ky0, (int)Wy) : ky0, 0, kxo);
    }
  }
  // zero padding rows [n_in, N), disjoint from the copy: this thread's rows z0 + k*ZS from the first >= n_in
  for (int z = z0 >= n_in ? z0 : z0 + (n_in - z0 + ZS - 1) / ZS * ZS; z < N; z += ZS) A[z * L + l] = make_float2(0.f, 0.f);
  mbar_wait(&bar, 0);
  __syncthreads();
  reg::fft2<R1, R2, L, NT, false, L, TWG>(A, twp);
  const float2* og = otf + ((unsigned)kxo * N * Wy + (kok ? ky : 0));
  if (ta.ofac) {  // separable PSF: rebuild the OTF column from its 1D factors
    const float2* fz = ta.ofac + ta.z.hx + Wy;
    const float2 c = kok ? cmul(__ldg(ta.ofac + kxo), __ldg(ta.ofac + ta.z.hx + ky)) : make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int z = z0 + k * ZS;
      if (z < N) A[z * L + l] = cmul(A[z * L + l], cmul(c, __ldg(fz + z)));
    }
  } else if (otma) {
    mbar_wait(&obar, 0);
    // half OTF: column ky lives at m = min(ky, Wy - ky), box slot m - start
    const int ol = ta.otf_half ? (ky <= (int)Wy / 2 ? ky : (int)Wy - ky) - half_box_start(ky0, (int)Wy) : l;
    const int op = ta.otf_half ? kHalfBox : L;  // OTF tile pitch
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int z = z0 + k * ZS;
      if (z < N) A[z * L + l] = cmul(A[z * L + l], O[z * op + ol]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int z = z0 + k * ZS;
      if (z < N) A[z * L + l] = cmul(A[z * L + l], kok ? __ldg(&og[(unsigned)z * Wy]) : make_float2(0.f, 0.f));
    }
  }
  __syncthreads();
  reg::fft2<R1, R2, L, NT, true, L, TWG>(A, twp);
  if (ta.tma_store) {  // rows [out_off, out_off+n_out) of the tile ARE the box (n_out = Pz): one TMA store
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_3d(&ta.map, A + out_off * L, ky0, 0, kx);  // columns ky >= Wy are clipped
      bulk_commit_and_release();
    }
    return;
  }
  if (kok) {
    float2* col = S + ((unsigned)kx * zrows * Wy + ky);
    for (int z = z0; z < n_out; z += ZS) col[(unsigned)z * Wy] = A[(z + out_off) * L + l];
  }
}

// ---- y forward / inverse with bulk-copied lines ---------------------------
// Each of the L input lines (n_in contiguous complex) is one
// cp.async.bulk global->shared copy into a line-major tile of pitch YNP
// (YNP = 2 mod 16: the pass-1 loads and pass 2 of the FFT are then free of
// bank conflicts with lanes along l), completion on one mbarrier; the zero
// padding [n_in, N) is written by the other threads meanwhile.  Requires an
// even n_in and in_pitch (16-byte sizes and addresses).
// Row pitch: the smallest NP >= N with NP = 16/L (mod 16) (L <= 8: the L
// lines of a half-warp land on disjoint bank pairs next to consecutive
// butterflies, and NP stays even so every row is 16-byte aligned).
template <int N, int L>
struct YTma {
  static constexpr int RES = L >= 16 ? 1 : 16 / L;
  static constexpr int NP = N + ((RES - N % 16) % 16 + 16) % 16;
};

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem_dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int R1, int R2, int L, bool TWG>
__global__ void __launch_bounds__(FastCfg<R1, R2, L, true>::NT) ypass_tma(const YArgs a) {
  static_assert(L <= 8, "16-byte aligned rows need an even pitch: L <= 8");
  constexpr int N = R1 * R2, NT = FastCfg<R1, R2, L, true>::NT, NP = YTma<N, L>::NP;
  extern __shared__ __align__(128) float2 smem[];
  float2* tw = TWG ? nullptr : smem;
  float2* A = TWG ? smem : smem + ((N + 1) / 2) * 2;  // keep 16-byte alignment
  __shared__ uint64_t bar;
  const int line0 = blockIdx.x * L;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!TWG) reg::load_twiddles2<R1, R2>(tw, a.plan.tw);
  const float2* twp = TWG ? a.plan.tw2 : tw;
  __syncthreads();
  pdl_trigger();
  pdl_wait();
  const int nvalid = min(L, a.nlines - line0);
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (unsigned)(nvalid * a.n_in * sizeof(float2)));
    for (int l = 0; l < nvalid; ++l)
      bulk_load(A + l * NP, a.in + (size_t)y_line(a, line0 + l) * a.in_pitch, (unsigned)(a.n_in * sizeof(float2)),
                &bar);
  }
  {  // zero padding [n_in, N) of the copied lines, and whole missing lines (last CTA only):
     // only the slots that need it (a loop over all L*N slots cost ~17% of the pass's instructions)
    const int padn = N - a.n_in;
    for (int idx = threadIdx.x; idx < nvalid * padn; idx += NT) {
      const int l = idx / padn;
      A[l * NP + a.n_in + (idx - l * padn)] = make_float2(0.f, 0.f);
    }
    for (int idx = nvalid * N + threadIdx.x; idx < L * N; idx += NT) {
      const int l = idx / N;
      A[l * NP + (idx - l * N)] = make_float2(0.f, 0.f);
    }
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  if (a.mode == YM_INV) {
    reg::fft2<R1, R2, L, NT, true, 1, TWG, NP>(A, twp);
  } else {
    reg::fft2<R1, R2, L, NT, false, 1, TWG, NP>(A, twp);
    if (a.mode == YM_CONV && a.ofac) {  // 2D, separable OTF: rebuilt from its 1D factors
      const float2* fy = a.ofac + a.ohx;
      const float2 fz0 = __ldg(fy + N);
      for (int l = 0; l < nvalid; ++l) {
        const float2 c = __ldg(a.ofac + line0 + l);
        for (int k = threadIdx.x; k < N; k += NT) A[l * NP + k] = cmul(A[l * NP + k], cmul(cmul(c, __ldg(fy + k)), fz0));
      }
      __syncthreads();
      reg::fft2<R1, R2, L, NT, true, 1, TWG, NP>(A, twp);
    } else if (a.mode == YM_CONV) {  // 2D: x OTF (line-major reads, coalesced) then inverse
      for (int l = 0; l < nvalid; ++l) {
        const float2* o = a.otf + (size_t)(line0 + l) * N;
        for (int k = threadIdx.x; k < N; k += NT) A[l * NP + k] = cmul(A[l * NP + k], __ldg(o + k));
      }
      __syncthreads();
      reg::fft2<R1, R2, L, NT, true, 1, TWG, NP>(A, twp);
    }
  }
  if (a.bst) {  // 16-byte aligned output lines: one bulk store per line
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int l = 0; l < nvalid; ++l)
        bulk_store(a.out + (size_t)y_line(a, line0 + l) * a.out_pitch, A + l * NP + a.out_off,
                   (unsigned)(a.n_out * sizeof(float2)));
      bulk_commit_and_release();
    }
    return;
  }
  for (int l = 0; l < nvalid; ++l) {
    float2* out = a.out + (size_t)y_line(a, line0 + l) * a.out_pitch;
    for (int j = threadIdx.x; j < a.n_out; j += NT) out[j] = A[l * NP + j + a.out_off];
  }
}

#ifdef VK_FAST_TABLE_MAIN  // defined once, in rl_fast_table.cu
// Phase ramp exp(+2 pi i (cx kx / Wx + cy ky / Wy)) over an OTF laid out
// [Hx][Wz][Wy]: the x crop offset (fast x pass) and, where the y inverse
// bulk-stores its lines, the y crop offset (the cropped y output then starts
// at slot 0, a 16-byte aligned shared address).
__global__ void otf_ramp_kernel(float2* __restrict__ otf, int Hx, size_t plane, int Wx, int cx, int Wy, int cy) {
  const size_t n = (size_t)Hx * plane;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i / plane), ky = (int)(i % Wy);
    const long long m = ((long long)cx * kx) % Wx, my = ((long long)cy * ky) % Wy;
    double s, c;
    sincospi(2.0 * ((double)m / (double)Wx + (double)my / (double)Wy), &s, &c);
    otf[i] = cmul(otf[i], make_float2((float)c, (float)s));
  }
}
#endif

}  // namespace vk
