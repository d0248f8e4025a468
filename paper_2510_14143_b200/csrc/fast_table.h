// Lookup of compile-time-length pass kernels (rl_fast_table.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <cuda.h>  // CUtensorMap (TMA descriptors)

#include "rl_passes.cuh"

namespace vk {

// Kernel argument of zpass_tma: the S_B tensor map (param space, 64-byte
// aligned, __grid_constant__) and the usual z-pass arguments.
struct alignas(64) ZTmaArgs {
  CUtensorMap map;   // S: dims {Wy, zrows, Hx}, box {16, Pz, 1}, 8-byte elements
  CUtensorMap omap;  // OTF: dims {Wy, Wz, Hx}, box {16, Wz, 1} (when otf_tma)
  ZArgs z;
  int otf_tma;
  int tma_store;  // write the cropped tile back with one TMA tensor store (same map)
  // factored OTF of a separable PSF: fx[Hx], fy[Wy], fz[Wz] back to back,
  // O(kx, kz, ky) = (fx[kx] * fy[ky]) * fz[kz]; nullptr: read the OTF
  const float2* ofac;
  // ky-even OTF stored as columns 0..Wy/2 only (vk_rl.cu halve_otfs): tiles
  // above Wy/2 read the mirrored columns Wy-ky, reversed within the box
  int otf_half;
  // kx-chunked convolution: S is a ring slot holding kx planes [kx0, kx0 +
  // gridDim.y); the OTF / factor index is kx0 + blockIdx.y
  int kx0;
};

// Kernel argument of xpass_tma: the S_A tensor map {Py, Pz, Hx}, box
// {2L, 1, tbk} (8-byte elements), and the usual x-pass arguments.
struct alignas(64) XTmaArgs {
  CUtensorMap map;
  XArgs x;
};

struct FastEntry {
  int N, R1;            // N = R1 * R2 (pass-1 / pass-2 radices)
  bool pdl;             // launch with programmatic dependent launch
  size_t smem_xp;       // x-pass
  size_t smem_yp;       // y-pass FWD/INV
  int Lx, NTx;          // x-pass: lines per CTA, threads
  int Ly, NTy;          // y-pass
  size_t smem_x;        // x-pass, and y-pass FWD/INV
  size_t smem_yconv;    // y-pass CONV (adds the prefetched OTF tile)
  const void* xk;       // xpass_fast<R1,R2,Lx>(XArgs)
  const void* xtk;      // xpass_tma<R1,R2,Lx>(XTmaArgs): TMA-staged spectrum rows (RATIO/UPDATE)
  const void* yk;       // ypass_fast<R1,R2,Lx>(YArgs)
  int Lz, NTz;          // z-pass
  size_t smem_z;
  const void* zk;       // zpass_fast<R1,R2,Lz>(ZArgs)
  const void* ztk;      // zpass_tma<R1,R2>(ZTmaArgs): TMA-staged column tile (Lz = 16), or nullptr
  size_t smem_zt;
  size_t smem_zt_half;  // zpass_tma with a half OTF (wider OTF tile)
  const void* ytk;      // ypass_tma<R1,R2,Ly>(YArgs): bulk-copied lines (FWD/INV), or nullptr
  size_t smem_yt;
};

const FastEntry* fast_lookup(int n);
cudaError_t fast_init_attributes();

// OTF *= exp(+2 pi i cx kx / Wx) for every kx plane (layout [Hx][plane]).
cudaError_t launch_otf_ramp(float2* otf, int Hx, size_t plane, int Wx, int cx, int Wy, int cy, cudaStream_t s);

}  // namespace vk

