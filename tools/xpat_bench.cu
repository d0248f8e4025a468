// micro-benchmark: x-pass access patterns on the S_A spectrum (C2 sizes); DESIGN.md §4 "kx-blocked S_A"
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xpat tools/xpat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int Hx = 289, Pz = 158, Py = 542, KB = (Hx + 7) / 8;
constexpr int SMEM = 41472;
// A: kx-plane-major [Hx][Pz][Py], float2 per thread, 8 lanes per 64 B (as xpass_fast)
__global__ void __launch_bounds__(192) patA(const float2* __restrict__ S, float2* __restrict__ O) {
  extern __shared__ float2 sm[];
  const int z = blockIdx.y, y0 = blockIdx.x * 16, l = threadIdx.x & 7;
  const unsigned plane = Pz * Py;
  const bool va = y0 + l < Py, vb = y0 + 8 + l < Py;
  const float2* Sa = S + (unsigned)z * Py + (va ? y0 + l : 0);
  const float2* Sb = S + (unsigned)z * Py + (vb ? y0 + 8 + l : 0);
  for (int kx0 = threadIdx.x / 8; kx0 < Hx; kx0 += 24 * 4) {
    float2 xa[4], xb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      xa[u] = (kx < Hx && va) ? Sa[kx * plane] : make_float2(0, 0);
      xb[u] = (kx < Hx && vb) ? Sb[kx * plane] : make_float2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      if (kx < Hx) { sm[kx * 17 + l] = xa[u]; sm[kx * 17 + 8 + l] = xb[u]; }
    }
  }
  __syncthreads();
  float2* Oa = O + (unsigned)z * Py + y0 + l;
  for (int kx = threadIdx.x / 8; kx < Hx; kx += 24) {
    if (va) Oa[kx * plane] = sm[kx * 17 + l];
    if (vb) Oa[kx * plane + 8] = sm[kx * 17 + 8 + l];
  }
}
// D: z-major [Pz][Hx][Py] (S_A candidate): the same 128-B pieces per kx,
// but the 289 pieces of a CTA lie 4.3 KB apart inside one z slab
__global__ void __launch_bounds__(192) patD(const float2* __restrict__ S, float2* __restrict__ O) {
  extern __shared__ float2 sm[];
  const int z = blockIdx.y, y0 = blockIdx.x * 16, l = threadIdx.x & 7;
  const bool va = y0 + l < Py, vb = y0 + 8 + l < Py;
  const float2* Sa = S + (size_t)z * Hx * Py + (va ? y0 + l : 0);
  const float2* Sb = S + (size_t)z * Hx * Py + (vb ? y0 + 8 + l : 0);
  for (int kx0 = threadIdx.x / 8; kx0 < Hx; kx0 += 24 * 4) {
    float2 xa[4], xb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      xa[u] = (kx < Hx && va) ? Sa[kx * Py] : make_float2(0, 0);
      xb[u] = (kx < Hx && vb) ? Sb[kx * Py] : make_float2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      if (kx < Hx) { sm[kx * 17 + l] = xa[u]; sm[kx * 17 + 8 + l] = xb[u]; }
    }
  }
  __syncthreads();
  float2* Oa = O + (size_t)z * Hx * Py + y0 + l;
  for (int kx = threadIdx.x / 8; kx < Hx; kx += 24) {
    if (va) Oa[kx * Py] = sm[kx * 17 + l];
    if (vb) Oa[kx * Py + 8] = sm[kx * 17 + 8 + l];
  }
}
// E: A with the grid walked z-fastest (consecutive CTAs: same y block, next z)
__global__ void __launch_bounds__(192) patE(const float2* __restrict__ S, float2* __restrict__ O) {
  extern __shared__ float2 sm[];
  const int z = blockIdx.x, y0 = blockIdx.y * 16, l = threadIdx.x & 7;
  const unsigned plane = Pz * Py;
  const bool va = y0 + l < Py, vb = y0 + 8 + l < Py;
  const float2* Sa = S + (unsigned)z * Py + (va ? y0 + l : 0);
  const float2* Sb = S + (unsigned)z * Py + (vb ? y0 + 8 + l : 0);
  for (int kx0 = threadIdx.x / 8; kx0 < Hx; kx0 += 24 * 4) {
    float2 xa[4], xb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      xa[u] = (kx < Hx && va) ? Sa[kx * plane] : make_float2(0, 0);
      xb[u] = (kx < Hx && vb) ? Sb[kx * plane] : make_float2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int kx = kx0 + u * 24;
      if (kx < Hx) { sm[kx * 17 + l] = xa[u]; sm[kx * 17 + 8 + l] = xb[u]; }
    }
  }
  __syncthreads();
  float2* Oa = O + (unsigned)z * Py + y0 + l;
  for (int kx = threadIdx.x / 8; kx < Hx; kx += 24) {
    if (va) Oa[kx * plane] = sm[kx * 17 + l];
    if (vb) Oa[kx * plane + 8] = sm[kx * 17 + 8 + l];
  }
}
// B: kx-blocked [KB][Pz][Py][8]: 16 rows x 8 kx = 1 KB contiguous per block
__global__ void __launch_bounds__(192) patB(const float4* __restrict__ S, float4* __restrict__ O) {
  extern __shared__ float4 sm4[];
  const int z = blockIdx.y, y0 = blockIdx.x * 16;
  const int nrow = min(16, Py - y0);
  const int per = nrow * 4;  // float4 per kb
  const int tot = KB * per;
  for (int i0 = threadIdx.x; i0 < tot; i0 += 192 * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int i = i0 + u * 192;
      if (i < tot) { int kb = i / per, r = i % per; v[u] = S[((size_t)(kb * Pz + z) * Py + y0) * 4 + r]; }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { int i = i0 + u * 192; if (i < tot) sm4[i] = v[u]; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tot; i += 192) {
    int kb = i / per, r = i % per;
    O[((size_t)(kb * Pz + z) * Py + y0) * 4 + r] = sm4[i];
  }
}
// C: contiguous float4 copy, same bytes per CTA
__global__ void __launch_bounds__(192) patC(const float4* __restrict__ S, float4* __restrict__ O, size_t n4) {
  extern __shared__ float4 sm4[];
  const size_t per = (n4 + gridDim.x * gridDim.y - 1) / (gridDim.x * gridDim.y);
  const size_t b = (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * per;
  const size_t e = b + per < n4 ? b + per : n4;
  for (size_t i0 = b + threadIdx.x; i0 < e; i0 += 192 * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t i = i0 + u * 192; if (i < e) v[u] = S[i]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t i = i0 + u * 192; if (i < e) sm4[(i - b) % 2592] = v[u]; }
  }
  __syncthreads();
  for (size_t i = b + threadIdx.x; i < e; i += 192) O[i] = sm4[(i - b) % 2592];
}
int main() {
  size_t nA = (size_t)Hx * Pz * Py, nB = (size_t)KB * 8 * Pz * Py;
  float2 *S, *O;
  cudaMalloc(&S, nB * 8); cudaMalloc(&O, nB * 8);
  cudaMemset(S, 0, nB * 8);
  char* flush; cudaMalloc(&flush, 512 << 20);
  for (auto k : {(const void*)patA, (const void*)patB, (const void*)patC, (const void*)patD, (const void*)patE})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  dim3 grid((Py + 15) / 16, Pz);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int which = 0; which < 5; ++which) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemset(flush, rep, 512 << 20);
      cudaEventRecord(e0);
      if (which == 0) patA<<<grid, 192, SMEM>>>(S, O);
      if (which == 1) patB<<<grid, 192, SMEM>>>((const float4*)S, (float4*)O);
      if (which == 2) patC<<<grid, 192, SMEM>>>((const float4*)S, (float4*)O, nA / 2);
      if (which == 3) patD<<<grid, 192, SMEM>>>(S, O);
      if (which == 4) patE<<<dim3(Pz, (Py + 15) / 16), 192, SMEM>>>(S, O);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep) best = ms < best ? ms : best;
    }
    double bytes = 2.0 * nA * 8;
    const char* names[] = {"A plane-major", "B kx-blocked", "C contiguous", "D z-major", "E plane-major z-fastest grid"};
    printf("%s %.4f ms  %.0f GB/s (alg bytes %.0f MB)\n", names[which], best, bytes / best / 1e6, bytes / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
