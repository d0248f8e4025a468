// Instantiations of the compile-time-length pass kernels (rl_fast.cuh) for
// the FFT lengths of the benchmark grids (96, 144, 192,
// 288, 576, 1080, 2160) plus a few common neighbours.  Any other 5-smooth
// length runs the generic Stockham kernels of rl_passes.cuh.
#define VK_NO_GENERIC_KERNELS
#define VK_FAST_TABLE_MAIN  // otf_ramp_kernel lives in this TU
#include "fast_table.h"
#include "rl_fast.cuh"

// Side builds for A/B runs may list a subset of lengths (build.py --lengths)
#ifndef VK_FAST_LENGTHS_DEF
#define VK_FAST_LENGTHS_DEF "fast_lengths.def"
#endif

namespace vk {

// rl_fast_len.cu, one object per length (fast_lengths.def)
#define VK_FAST_LEN(n) FastEntry fast_entry_##n();
#include VK_FAST_LENGTHS_DEF
#undef VK_FAST_LEN

namespace {

const FastEntry kTable[] = {
#define VK_FAST_LEN(n) fast_entry_##n(),
#include VK_FAST_LENGTHS_DEF
#undef VK_FAST_LEN
};

}  // namespace

const FastEntry* fast_lookup(int n) {
  for (const auto& e : kTable)
    if (e.N == n) return &e;
  return nullptr;
}

cudaError_t fast_init_attributes() {
  for (const auto& e : kTable) {
    cudaError_t r;
    if ((r = cudaFuncSetAttribute(e.xk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_xp))) return r;
    if (e.xtk && (r = cudaFuncSetAttribute(e.xtk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_xp)))
      return r;
    if ((r = cudaFuncSetAttribute(e.yk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yconv))) return r;
    if ((r = cudaFuncSetAttribute(e.zk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_z))) return r;
    if (e.ztk && (r = cudaFuncSetAttribute(e.ztk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_zt_half)))
      return r;
    if (e.ytk && (r = cudaFuncSetAttribute(e.ytk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_yt)))
      return r;
    // prefer the full shared-memory carveout: occupancy is smem-limited
    for (const void* k : {e.xk, e.xtk, e.yk, e.zk})
      if (k && (r = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100))) return r;
  }
  return cudaSuccess;
}

cudaError_t launch_otf_ramp(float2* otf, int Hx, size_t plane, int Wx, int cx, int Wy, int cy, cudaStream_t s) {
  otf_ramp_kernel<<<148 * 8, 256, 0, s>>>(otf, Hx, plane, Wx, cx, Wy, cy);
  return cudaGetLastError();
}

}  // namespace vk
