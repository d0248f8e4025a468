// On-device stopping metric: single-image Fourier ring/shell correlation.
//
// The reference's default StoppingRule metric is frc_resolution
// (include/voxelkit/deconv.hpp:36), evaluated every iteration on the f32 crop
// of the estimate as metrics::single_image_frc(even_view(current), spacing)
// (src/deconv.cpp:285-289, src/metrics.cpp:146-264):
//   * even_view trims a trailing odd voxel per axis;
//   * the image splits into two half-size sub-images on the (0,0,0) and
//     (1,1,1) checkerboard diagonals;
//   * both get an r2c FFT; per integer-radius ring j of width 1/n_max
//     (n_max = the largest half extent), num = sum w Re(A conj B),
//     den_a = sum w |A|^2, den_b = sum w |B|^2 with w = 2 for kx planes that
//     stand for a conjugate pair (1 for kx = 0 and the even-length Nyquist);
//   * correlation = num / sqrt(den_a den_b); the first crossing of 1/7 above
//     DC (linear interpolation) gives the resolution spacing*2 / nu.
// Here the split reads the P-domain estimate directly, the two spectra come
// from a sub-plan's r2c passes (the same kernels as the OTF build), and the
// ring sums are block-reduced in shared memory then added with FP64 atomics.
// Only the final curve walk (a few hundred bins) runs on the host.
#pragma once
#include "rl_passes.cuh"

namespace vk {

// est: P-domain estimate; the crop starts at (oz, oy, ox).  h*: half extents
// (1 for absent axes), s*: 1 where the axis exists (checkerboard shift).
__global__ void frc_split_kernel(const float* __restrict__ est, Geom g, int hz, int hy, int hx, int sz, int sy,
                                 int sx, float* __restrict__ even, float* __restrict__ odd) {
  const size_t n = (size_t)hz * hy * hx;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % hx);
    const size_t t = i / hx;
    const int y = (int)(t % hy), z = (int)(t / hy);
    const int ze = (sz ? 2 * z : 0) + g.oz, ye = (sy ? 2 * y : 0) + g.oy, xe = (sx ? 2 * x : 0) + g.ox;
    even[i] = est[((size_t)ze * g.Py + ye) * g.Px + xe];
    odd[i] = est[((size_t)(ze + sz) * g.Py + (ye + sy)) * g.Px + (xe + sx)];
  }
}

// Ring sums over two half spectra laid out [Hx][Wz][Wy] (OTF layout).
// bins: [3][nbins] = num, den_a, den_b.  Shared scratch: 3*nbins doubles.
__global__ void frc_bins_kernel(const float2* __restrict__ A, const float2* __restrict__ B, int Wz, int Wy, int Wx,
                                int Hx, double bin_freq, int nbins, double* __restrict__ bins) {
  extern __shared__ double hist[];
  for (int i = threadIdx.x; i < 3 * nbins; i += blockDim.x) hist[i] = 0.0;
  __syncthreads();
  const size_t n = (size_t)Hx * Wz * Wy;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int ky = (int)(i % Wy);
    const size_t t = i / Wy;
    const int kz = (int)(t % Wz), kx = (int)(t / Wz);
    const double fz = (double)min(kz, Wz - kz) / Wz;
    const double fy = (double)min(ky, Wy - ky) / Wy;
    const double fx = (double)min(kx, Wx - kx) / Wx;
    const double nu = sqrt(fz * fz + fy * fy + fx * fx);
    const long long bin = llround(nu / bin_freq);  // metrics.cpp:186-187
    if (bin < nbins) {
      const bool selfc = kx == 0 || ((Wx % 2 == 0) && 2 * kx == Wx);
      const double w = selfc ? 1.0 : 2.0;
      const float2 a = A[i], b = B[i];
      atomicAdd(&hist[bin], w * ((double)a.x * b.x + (double)a.y * b.y));
      atomicAdd(&hist[nbins + bin], w * ((double)a.x * a.x + (double)a.y * a.y));
      atomicAdd(&hist[2 * nbins + bin], w * ((double)b.x * b.x + (double)b.y * b.y));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * nbins; i += blockDim.x)
    if (hist[i] != 0.0) atomicAdd(&bins[i], hist[i]);
}

}  // namespace vk
