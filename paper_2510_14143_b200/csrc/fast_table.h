// Lookup of compile-time-length pass kernels (rl_fast_table.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace vk {

struct FastEntry {
  int N;
  int Lx, NTx;          // x-pass and y-pass: lines per CTA, threads
  size_t smem_x;        // x-pass, and y-pass FWD/INV
  size_t smem_yconv;    // y-pass CONV (adds the prefetched OTF tile)
  const void* xk;       // xpass_fast<R1,R2,Lx>(XArgs)
  const void* yk;       // ypass_fast<R1,R2,Lx>(YArgs)
  int Lz, NTz;          // z-pass
  size_t smem_z;
  const void* zk;       // zpass_fast<R1,R2,Lz>(ZArgs)
};

const FastEntry* fast_lookup(int n);
cudaError_t fast_init_attributes();

// OTF *= exp(+2 pi i cx kx / Wx) for every kx plane (layout [Hx][plane]).
cudaError_t launch_otf_ramp(float2* otf, int Hx, size_t plane, int Wx, int cx, cudaStream_t s);

}  // namespace vk
