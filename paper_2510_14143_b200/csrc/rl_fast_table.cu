// Instantiations of the compile-time-length pass kernels (rl_fast.cuh) for
// the FFT lengths of the benchmark grids (96, 144, 192,
// 288, 576, 1080, 2160) plus a few common neighbours.  Any other 5-smooth
// length runs the generic Stockham kernels of rl_passes.cuh.
#define VK_NO_GENERIC_KERNELS
#define VK_FAST_TABLE_MAIN  // otf_ramp_kernel lives in this TU
#include "fast_table.h"
#include "rl_fast.cuh"
#include "rl_cluster.cuh"
#include "rl_dataflow.cuh"

namespace vk {

// rl_fast_len.cu, one object per length
FastEntry fast_entry_64();
FastEntry fast_entry_96();
FastEntry fast_entry_144();
FastEntry fast_entry_192();
FastEntry fast_entry_256();
FastEntry fast_entry_288();
FastEntry fast_entry_576();
FastEntry fast_entry_1080();
FastEntry fast_entry_2160();

namespace {

const FastEntry kTable[] = {
    fast_entry_64(),
    fast_entry_96(),
    fast_entry_144(),
    fast_entry_192(),
    fast_entry_256(),
    fast_entry_288(),
    fast_entry_576(),
    fast_entry_1080(),
    fast_entry_2160(),
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
    if (e.xtk && (r = cudaFuncSetAttribute(e.xtk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_xp)))
      return r;
    if ((r = cudaFuncSetAttribute(e.yk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yconv))) return r;
    if ((r = cudaFuncSetAttribute(e.zk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_z))) return r;
    if ((r = cudaFuncSetAttribute(e.zpk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_zp))) return r;
    if (e.ztk && (r = cudaFuncSetAttribute(e.ztk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_zt_half)))
      return r;
    if (e.ytk && (r = cudaFuncSetAttribute(e.ytk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yt)))
      return r;
    // prefer the full shared-memory carveout: occupancy is smem-limited
    for (const void* k : {e.xk, e.xtk, e.yk, e.zk, e.zpk})
      if (k && (r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100))) return r;
  }
  return cudaSuccess;
}

cudaError_t launch_otf_ramp(float2* otf, int Hx, size_t plane, int Wx, int cx, int Wy, int cy, cudaStream_t s) {
  otf_ramp_kernel<<<148 * 8, 256, 0, s>>>(otf, Hx, plane, Wx, cx, Wy, cy);
  return cudaGetLastError();
}

}  // namespace vk
