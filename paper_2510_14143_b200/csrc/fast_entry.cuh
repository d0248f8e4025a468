// make_entry: the FastEntry of one compile-time FFT length (kernel
// pointers, launch shapes, shared-memory sizes).  Included by rl_fast_len.cu,
// which is compiled once per length (-DVK_LEN=N) so the lengths' kernels
// build in parallel.
#pragma once
#ifndef VK_NO_GENERIC_KERNELS
#define VK_NO_GENERIC_KERNELS
#endif
#include "fast_table.h"
#include "rl_fast.cuh"

namespace vk {

// TWG / YPREF / XMINB / XPB: x and y pass variants (rl_fast.cuh); ZTWG /
// ZPREF / ZMINB: the z pass's.  Chosen per length from B200 measurements.
template <int R1, int R2, int LX, int LZ, bool TWG = false, bool YPREF = true, int XMINB = 1, bool XPB = false,
          bool ZTWG = false, bool ZPREF = true, int ZMINB = 1, bool PDL = true, int /*retired: pipelined-z floor*/ = 2, int LY0 = 0,
          int ZTMA = 0,  // ZTMA: resident-CTA floor of the TMA z kernel (0 = no TMA variant)
          bool YTMA = false,
          bool XTMA = false>  // XTMA: TMA-staged RATIO/UPDATE x pass (xpass_tma)
FastEntry make_entry() {
  constexpr int LY = LY0 ? LY0 : LX;  // y-pass lines per CTA (default: the x pass's)
  FastEntry e{};
  e.N = R1 * R2;
  e.pdl = PDL;
  e.R1 = R1;
  // x pass: the transform tile, after the shared twiddle table rounded up to
  // 128 bytes when there is one (TMA destinations)
  e.smem_xp = FastCfg<R1, R2, LX>::smem_x + (TWG ? 0 : (size_t)((R1 * R2 + 15) / 16 * 16) * sizeof(float2));
  e.Lx = LX;
  e.NTx = FastCfg<R1, R2, LX>::NT;
  e.smem_x = FastCfg<R1, R2, LX>::smem;
  e.Ly = LY;
  e.NTy = FastCfg<R1, R2, LY, true>::NT;
  e.smem_yp = (size_t)(FastCfg<R1, R2, LY, true>::DATA + (TWG ? 0 : R1 * R2)) * sizeof(float2);
  e.smem_yconv = (size_t)(FastCfg<R1, R2, LY, true>::DATA + (TWG ? 0 : R1 * R2) + (YPREF ? R1 * R2 * LY : 0)) *
                 sizeof(float2);
  e.xk = (const void*)xpass_fast<R1, R2, LX, TWG, XMINB, XPB>;
  if constexpr (XTMA) e.xtk = (const void*)xpass_tma<R1, R2, LX, TWG, XMINB, XPB>;
  e.yk = (const void*)ypass_fast<R1, R2, LY, TWG, YPREF>;
  e.Lz = LZ;
  e.NTz = FastCfg<R1, R2, LZ, true>::NT;
  e.smem_z = (size_t)(FastCfg<R1, R2, LZ, true>::DATA + (ZTWG ? 0 : R1 * R2) + (ZPREF ? R1 * R2 * LZ : 0)) *
             sizeof(float2);
  e.zk = (const void*)zpass_fast<R1, R2, LZ, ZTWG, ZPREF, ZMINB>;
  if constexpr (YTMA) {
    e.ytk = (const void*)ypass_tma<R1, R2, LY, TWG>;
    e.smem_yt = (size_t)(LY * YTma<R1 * R2, LY>::NP + (TWG ? 0 : ((R1 * R2 + 1) / 2) * 2)) * sizeof(float2);
  }
  if constexpr (ZTMA > 0 && LZ == 16) {
    e.ztk = (const void*)zpass_tma<R1, R2, ZTWG, ZTMA>;
    e.smem_zt = (size_t)(2 * R1 * R2 * 16 + (ZTWG ? 0 : (R1 * R2 + 15) / 16 * 16)) * sizeof(float2);  // twiddles + tile + OTF tile
    e.smem_zt_half = e.smem_zt + (size_t)R1 * R2 * (kHalfBox - 16) * sizeof(float2);  // 18-wide half-OTF tile
  }
  return e;
}

}  // namespace vk
