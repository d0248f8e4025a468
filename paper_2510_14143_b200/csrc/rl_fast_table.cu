// Instantiations of the compile-time-length pass kernels (rl_fast.cuh) for
// the FFT lengths of the benchmark grids (96, 144, 192,
// 288, 576, 1080, 2160) plus a few common neighbours.  Any other 5-smooth
// length runs the generic Stockham kernels of rl_passes.cuh.
#define VK_NO_GENERIC_KERNELS
#include "fast_table.h"
#include "rl_cluster.cuh"
#include "rl_dataflow.cuh"

namespace vk {

namespace {

// TWG / YPREF / XMINB / XPB: x and y pass variants (rl_fast.cuh); ZTWG /
// ZPREF / ZMINB: the z pass's.  Chosen per length from B200 measurements.
template <int R1, int R2, int LX, int LZ, bool TWG = false, bool YPREF = true, int XMINB = 1, bool XPB = false,
          bool ZTWG = false, bool ZPREF = true, int ZMINB = 1, bool PDL = true, int ZPMINB = 2, int LY0 = 0,
          int ZTMA = 0,  // ZTMA: resident-CTA floor of the TMA z kernel (0 = no TMA variant)
          bool YTMA = false>
FastEntry make_entry() {
  constexpr int LY = LY0 ? LY0 : LX;  // y-pass lines per CTA (default: the x pass's)
  FastEntry e{};
  e.N = R1 * R2;
  e.pdl = PDL;
  e.R1 = R1;
  e.smem_xp = TWG ? FastCfg<R1, R2, LX>::smem_x : FastCfg<R1, R2, LX>::smem;
  e.Lx = LX;
  e.NTx = FastCfg<R1, R2, LX>::NT;
  e.smem_x = FastCfg<R1, R2, LX>::smem;
  e.Ly = LY;
  e.NTy = FastCfg<R1, R2, LY, true>::NT;
  e.smem_yp = (size_t)(FastCfg<R1, R2, LY, true>::DATA + (TWG ? 0 : R1 * R2)) * sizeof(float2);
  e.smem_yconv = (size_t)(FastCfg<R1, R2, LY, true>::DATA + (TWG ? 0 : R1 * R2) + (YPREF ? R1 * R2 * LY : 0)) *
                 sizeof(float2);
  e.xk = (const void*)xpass_fast<R1, R2, LX, TWG, XMINB, XPB>;
  e.yk = (const void*)ypass_fast<R1, R2, LY, TWG, YPREF>;
  e.Lz = LZ;
  e.NTz = FastCfg<R1, R2, LZ, true>::NT;
  e.smem_z = (size_t)(FastCfg<R1, R2, LZ, true>::DATA + (ZTWG ? 0 : R1 * R2) + (ZPREF ? R1 * R2 * LZ : 0)) *
             sizeof(float2);
  e.zk = (const void*)zpass_fast<R1, R2, LZ, ZTWG, ZPREF, ZMINB>;
  e.smem_zp = ZPipeCfg<R1, R2, LZ, ZTWG, ZPREF>::smem;
  e.zpk = (const void*)zpass_pipe<R1, R2, LZ, ZTWG, ZPREF, ZPMINB>;
  if constexpr (YTMA) {
    e.ytk = (const void*)ypass_tma<R1, R2, LY, TWG>;
    e.smem_yt = (size_t)(LY * YTma<R1 * R2, LY>::NP + (TWG ? 0 : ((R1 * R2 + 1) / 2) * 2)) * sizeof(float2);
  }
  if constexpr (ZTMA > 0 && LZ == 16) {
    e.ztk = (const void*)zpass_tma<R1, R2, ZTWG, ZTMA>;
    e.smem_zt = (size_t)(2 * R1 * R2 * 16 + (ZTWG ? 0 : R1 * R2)) * sizeof(float2);  // tile + OTF tile
  }
  return e;
}

const FastEntry kTable[] = {
    make_entry<8, 8, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 0, true>(),  // 64 (FRC half grids, small z)
    make_entry<8, 12, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 6, true>(),  // 96 (z: TMA 6; y bulk L=8)
    make_entry<12, 12, 16, 16, false, true, 1, false, true, false, 8, true, 2, 8, 6, true>(),  // 144 (z: TMA 6; y bulk L=8)
    make_entry<12, 16, 16, 16, false, true, 1, false, true, false, 5, true, 2, 8, 4, true>(),  // 192 (z: TMA tile, 4 CTAs/SM; y bulk L=8)
    make_entry<16, 16, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 0, true>(),  // 256 (y bulk L=8)
    make_entry<16, 18, 16, 16, false, true, 1, false, false, true, 1, true, 2, 8, 0, true>(),  // 288 (y: bulk, L=8)
    make_entry<24, 24, 8, 8, true, true, 5, false, false, true, 1, true, 2, 0, 0, true>(),  // 576: global twiddles -> 5 x/y CTAs/SM (y L=4: slower); y bulk copies
    make_entry<30, 36, 8, 4, false, true, 1, true, false, true, 1, true, 2, 4, 0, true>(),  // 1080 (Ix = 1000: partial chunks are common)
    // 2160: no smem twiddles / OTF tile -> 2 CTAs per SM; no PDL (CTAs parked
    // in griddepcontrol.wait would hold the scarce slots the batch lanes'
    // kernels need: C5 3.05e10 without vs 2.66e10 with, profiles/r01/pdl.log)
    make_entry<45, 48, 4, 2, true, false, 1, false, false, true, 1, false, 2, 2, 0, true>(),  // y L=2
};

}  // namespace

const FastEntry* fast_lookup(int n) {
  for (const auto& e : kTable)
    if (e.N == n) return &e;
  return nullptr;
}

template <int YR1, int YR2, int YL, int ZR1, int ZR2, int ZL>
DfEntry make_df() {
  using C = DfCfg<YR1, YR2, YL, ZR1, ZR2, ZL>;
  return DfEntry{C::NY, C::NZ, YL, ZL, C::NT, C::smem, (const void*)yzconv_dataflow<YR1, YR2, YL, ZR1, ZR2, ZL>};
}

const DfEntry kDfTable[] = {
    make_df<16, 18, 8, 8, 12, 16>(),    // C1/C3 grid: Wy 288, Wz 96
    make_df<24, 24, 8, 12, 16, 8>(),    // C2 grid: Wy 576, Wz 192
    make_df<30, 36, 4, 12, 12, 8>(),    // C4 grid: Wy 1080, Wz 144
};

template <int YR1, int YR2, int ZR1, int ZR2, int C, int RZ, int ZG, int NT>
ClEntry make_cl() {
  using K = ClCfg<YR1, YR2, ZR1, ZR2, C, RZ, ZG, NT>;
  return ClEntry{K::NY, K::NZ, C, RZ, NT, K::smem, (const void*)yzconv_cluster<YR1, YR2, ZR1, ZR2, C, RZ, ZG, NT>};
}

const ClEntry kClTable[] = {
    make_cl<16, 18, 8, 12, 4, 20, 24, 384>(),    // C1/C3 grid: Wy 288, Wz 96, Pz <= 80
    make_cl<24, 24, 12, 16, 12, 14, 24, 384>(),  // C2 grid: Wy 576, Wz 192, Pz <= 168
    make_cl<30, 36, 12, 12, 12, 10, 30, 384>(),  // C4 grid: Wy 1080, Wz 144, Pz <= 120
};

const ClEntry* cl_lookup(int ny, int nz, int pz) {
  for (const auto& e : kClTable)
    if (e.Ny == ny && e.Nz == nz && (pz + e.C - 1) / e.C <= e.RZ) return &e;
  return nullptr;
}

const DfEntry* df_lookup(int ny, int nz) {
  for (const auto& e : kDfTable)
    if (e.Ny == ny && e.Nz == nz) return &e;
  return nullptr;
}

cudaError_t fast_init_attributes() {
  for (const auto& e : kClTable) {
    cudaError_t r = cudaFuncSetAttribute(e.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem);
    if (r) return r;
    if (e.C > 8 && (r = cudaFuncSetAttribute(e.k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return r;
  }
  for (const auto& e : kDfTable) {
    cudaError_t r = cudaFuncSetAttribute(e.k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem);
    if (r) return r;
  }
  for (const auto& e : kTable) {
    cudaError_t r;
    if ((r = cudaFuncSetAttribute(e.xk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_xp))) return r;
    if ((r = cudaFuncSetAttribute(e.yk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yconv))) return r;
    if ((r = cudaFuncSetAttribute(e.zk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_z))) return r;
    if ((r = cudaFuncSetAttribute(e.zpk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_zp))) return r;
    if (e.ztk && (r = cudaFuncSetAttribute(e.ztk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_zt)))
      return r;
    if (e.ytk && (r = cudaFuncSetAttribute(e.ytk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yt)))
      return r;
    // prefer the full shared-memory carveout: occupancy is smem-limited
    for (const void* k : {e.xk, e.yk, e.zk, e.zpk})
      if ((r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100))) return r;
  }
  return cudaSuccess;
}

cudaError_t launch_otf_ramp(float2* otf, int Hx, size_t plane, int Wx, int cx, cudaStream_t s) {
  otf_ramp_kernel<<<148 * 8, 256, 0, s>>>(otf, Hx, plane, Wx, cx);
  return cudaGetLastError();
}

}  // namespace vk
