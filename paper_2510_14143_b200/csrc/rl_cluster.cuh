// Fused y/z convolution on thread-block clusters (3D plans).
//
// One convolution of the x-transformed field (deconv.cpp:135-147 minus the
// x transforms) is, per kx plane p (Pz x Py complex in S_A):
//     y-forward (rows, zero-padded Py -> Wy)
//     z-forward * OTF * z-inverse (columns, Pz -> Wz -> cropped Pz)
//     y-inverse (rows, Wy -> cropped Py)
// The intermediate plane (Pz x Wy complex, 728 KB at C2) does not fit one
// SM, so the 3-launch path writes and re-reads it through HBM twice.  Here a
// cluster of C CTAs (one per SM) holds it in DISTRIBUTED shared memory:
//
//   CTA r owns rows z in [r*RZr, (r+1)*RZr)  for the y transforms (Ybuf)
//          and columns ky in [r*CK, (r+1)*CK) for the z transforms (Zbuf)
//   1. rows S_A -> Ybuf (cp.async), y-forward in place
//   2. cluster.sync; each CTA gathers its ky columns of ALL rows from the
//      owners' Ybuf over DSMEM into Zbuf (a distributed transpose)
//   3. z-forward, x OTF (read once from HBM), z-inverse
//   4. cluster.sync; each CTA gathers its rows of ALL ky columns from the
//      owners' Zbuf over DSMEM back into Ybuf
//   5. y-inverse, cropped rows -> S_A
//
// HBM traffic per convolution drops from 16*S_p + 32*Hx*Pz*Wy + 8*S_otf to the
// minimum 16*S_p + 8*S_otf.  Clusters are persistent and
// walk kx planes with stride gridDim.x / C.
#pragma once
#include <cooperative_groups.h>

#include "fast_table.h"
#include "fft_reg.cuh"
#include "rl_fast.cuh"

namespace vk {

namespace cg = cooperative_groups;

// YR1*YR2 = Wy, ZR1*ZR2 = Wz, C = cluster size, RZ = max rows per CTA
// (ceil(Pz / C) <= RZ), ZG = z lines per transform group, NT threads.
template <int YR1, int YR2, int ZR1, int ZR2, int C, int RZ, int ZG, int NT>
struct ClCfg {
  static constexpr int NY = YR1 * YR2, NZ = ZR1 * ZR2;
  static constexpr int CK = NY / C;  // ky columns per CTA
  static_assert(NY % C == 0, "Wy must split evenly over the cluster");
  static_assert(CK % ZG == 0, "column groups must tile CK");
  static_assert(NT >= RZ * YR2 && NT >= ZG * ZR2, "one pass-1 butterfly per thread");
  static constexpr int LPY = RZ + 1, LPZ = CK + 1;  // padded pitches (reg::sw)
  static constexpr int YBUF = NY * LPY, ZBUF = NZ * LPZ;
  static constexpr size_t smem = (size_t)(NY + NZ + YBUF + ZBUF) * sizeof(float2);
};

template <int YR1, int YR2, int ZR1, int ZR2, int C, int RZ, int ZG, int NT>
__global__ void __launch_bounds__(NT, 1) yzconv_cluster(const ClArgs a) {
  using K = ClCfg<YR1, YR2, ZR1, ZR2, C, RZ, ZG, NT>;
  constexpr int NY = K::NY, NZ = K::NZ, CK = K::CK, LPY = K::LPY, LPZ = K::LPZ;
  extern __shared__ float2 smem[];
  float2* twy = smem;
  float2* twz = twy + NY;
  float2* Y = twz + NZ;      // [NY][LPY]: line lz = my row z0 + lz
  float2* Z = Y + K::YBUF;   // [NZ][LPZ]: line c = my column ky0 + c
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank();
  const int ncl = gridDim.x / C, cid = blockIdx.x / C;
  const Geom& g = a.g;
  const int RZr = (g.Pz + C - 1) / C;  // rows per CTA (<= RZ, host-checked)
  const int z0 = r * RZr;
  const int nz = max(0, min(RZr, g.Pz - z0));
  const int ky0 = r * CK;
  const int tid = threadIdx.x;
  reg::load_twiddles2<YR1, YR2>(twy, a.twy);
  reg::load_twiddles2<ZR1, ZR2>(twz, a.twz);

  for (int kx = cid; kx < g.Hx; kx += ncl) {
    // Launder the shared-memory bases each plane: otherwise ptxas hoists every
    // unrolled transform address out of the plane loop and spills them.
    asm volatile("" : "+l"(Y), "+l"(Z), "+l"(twy), "+l"(twz));
    // 1. my rows of the plane -> Ybuf (zero padded to Wy), y-forward
    const float2* src = a.SA + ((size_t)kx * g.Pz + z0) * g.Py;
    for (int lz = 0; lz < RZ; ++lz) {
      const float2* row = src + (size_t)lz * g.Py;
      for (int i = tid; i < NY; i += NT) {
        if (lz < nz && i < g.Py)
          cp_async8(&Y[i * LPY + lz], &row[i]);
        else
          Y[i * LPY + lz] = make_float2(0.f, 0.f);
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    reg::fft2<YR1, YR2, RZ, NT, false, LPY>(Y, twy);
    cl.sync();

    // 2. distributed transpose: my ky columns of every row, from the owners
#pragma unroll 1
    for (int o = 0; o < C; ++o) {
      const float2* rY = cl.map_shared_rank(Y, o);
      const int onz = max(0, min(RZr, g.Pz - o * RZr));
#pragma unroll 4
      for (int idx = tid; idx < RZ * CK; idx += NT) {
        const int c = idx / RZ, lz = idx - c * RZ;  // lz fastest: contiguous remote reads
        if (lz < onz) Z[(o * RZr + lz) * LPZ + c] = rY[(ky0 + c) * LPY + lz];
      }
    }
    for (int idx = tid; idx < (NZ - g.Pz) * CK; idx += NT) {
      const int zz = g.Pz + idx / CK, c = idx % CK;
      Z[zz * LPZ + c] = make_float2(0.f, 0.f);
    }
    __syncthreads();

    // 3. z-forward, OTF, z-inverse (column groups of ZG)
#pragma unroll 1
    for (int g0 = 0; g0 < CK; g0 += ZG) reg::fft2<ZR1, ZR2, ZG, NT, false, LPZ>(Z + g0, twz);
    {
      const float2* o = a.otf + (size_t)kx * NZ * NY + ky0;
#pragma unroll 4
      for (int idx = tid; idx < NZ * CK; idx += NT) {
        const int kz = idx / CK, c = idx - kz * CK;
        Z[kz * LPZ + c] = cmul(Z[kz * LPZ + c], __ldg(&o[(size_t)kz * NY + c]));
      }
    }
    __syncthreads();
#pragma unroll 1
    for (int g0 = 0; g0 < CK; g0 += ZG) reg::fft2<ZR1, ZR2, ZG, NT, true, LPZ>(Z + g0, twz);
    cl.sync();

    // 4. distributed transpose back: my rows of every ky column (crop cz)
#pragma unroll 1
    for (int o = 0; o < C; ++o) {
      const float2* rZ = cl.map_shared_rank(Z, o);
#pragma unroll 4
      for (int idx = tid; idx < RZ * CK; idx += NT) {
        const int lz = idx / CK, c = idx - lz * CK;  // c fastest: contiguous remote reads
        if (lz < nz) Y[(o * CK + c) * LPY + lz] = rZ[(z0 + lz + g.cz) * LPZ + c];
      }
    }
    __syncthreads();

    // 5. y-inverse, cropped rows -> S_A
    reg::fft2<YR1, YR2, RZ, NT, true, LPY>(Y, twy);
    float2* dst = a.SA + ((size_t)kx * g.Pz + z0) * g.Py;
    for (int lz = 0; lz < nz; ++lz) {
      float2* row = dst + (size_t)lz * g.Py;
      for (int j = tid; j < g.Py; j += NT) row[j] = Y[(j + g.cy) * LPY + lz];
    }
    __syncthreads();
  }
  cl.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace vk
