/*
 * vk_io.h — C ABI for the data formats either side of the deconvolution path
 * (SURVEY.md §8(f) row f2): NDIV volume files and the synthetic inputs the
 * reference CLI's `deconvolve` builds.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   vk_volume_info_read / vk_volume_read ... io::read_volume   (src/io.cpp:83-158)
 *   vk_volume_write ........................ io::write_volume  (src/io.cpp:53-81)
 *   vk_generate_blobs ...................... synth::generate_blobs (src/synth.cpp:199-224)
 *   vk_gaussian_psf ........................ synth::gaussian_psf   (src/synth.cpp:226-258)
 * The _device variants stream the payload between the file and device
 * memory through two pinned staging buffers, so the file read (write) of one
 * chunk overlaps the DMA of the previous one.
 *
 * NDIV layout (include/voxelkit/io.hpp:25-29): "NDIV", u32 LE header length
 * H, H bytes of JSON {"axes","elem","shape","spacing"?}, then the raw
 * little-endian row-major payload with no trailing bytes.  Headers are
 * written compact with sorted keys and shortest round-trip doubles, as the
 * reference's JSON library emits them, so write(read(f)) == f bytewise.
 * Status codes and messages follow the reference exceptions (vk_rl.h).
 */
#ifndef VK_IO_H_
#define VK_IO_H_

#include "vk_rl.h"

#ifdef __cplusplus
extern "C" {
#endif

#define VK_VOLUME_MAX_RANK 4

/* voxelkit::Elem (include/voxelkit/image.hpp) */
typedef enum vk_elem { VK_ELEM_F32 = 0, VK_ELEM_U16 = 1, VK_ELEM_U32 = 2, VK_ELEM_BOOL = 3 } vk_elem;

typedef struct vk_volume_info {
  int elem;                               /* vk_elem                       */
  int rank;                               /* 1..4 (X, YX, ZYX, CZYX)       */
  uint64_t shape[VK_VOLUME_MAX_RANK];
  int has_spacing;
  double spacing[VK_VOLUME_MAX_RANK];     /* valid when has_spacing        */
  uint64_t payload_offset;                /* read: byte offset of payload  */
  uint64_t payload_bytes;                 /* element count * element size  */
} vk_volume_info;

/* Header of an NDIV file (magic, header JSON, payload length and no trailing
 * bytes are all validated, as read_volume does before returning). */
vk_status vk_volume_info_read(const char* path, vk_volume_info* info);

/* Whole volume into host memory (dst_bytes >= payload_bytes). */
vk_status vk_volume_read(const char* path, vk_volume_info* info, void* dst, uint64_t dst_bytes);

/* Whole volume into device memory on the current device, chunked through
 * pinned staging on `stream`; returns after the last chunk has landed. */
vk_status vk_volume_read_device(const char* path, vk_volume_info* info, void* d_dst, uint64_t dst_bytes,
                                void* stream);

/* write_volume from host memory; info->payload_offset / payload_bytes are
 * ignored (derived from elem and shape). */
vk_status vk_volume_write(const char* path, const vk_volume_info* info, const void* src);

/* write_volume from device memory, D2H chunks overlapped with file writes. */
vk_status vk_volume_write_device(const char* path, const vk_volume_info* info, const void* d_src,
                                 void* stream);

/* synth::SynthSpec (include/voxelkit/synth.hpp:27-39) */
typedef struct vk_synth_spec {
  uint64_t shape[3]; /* ZYX */
  uint64_t n_objects;
  double radius_min, radius_max;
  uint64_t seed;
  double noise_sigma;
  double anisotropy;
  double inplane_margin;
} vk_synth_spec;

/* generate_blobs(spec).intensity into d_out (device, f32 ZYX) on `device`:
 * object placement replays the reference's mt19937_64 stream on the host;
 * rasterisation and the Gaussian noise (Box-Muller over the same stream)
 * run on the GPU.  spacing3 (may be NULL) receives {anisotropy, 1, 1}. */
vk_status vk_generate_blobs(int device, const vk_synth_spec* spec, float* d_out, double* spacing3,
                            void* stream);

/* gaussian_psf(shape, sigmas) into host memory (nsig == 1 broadcasts). */
vk_status vk_gaussian_psf(int rank, const uint64_t* shape, const double* sigmas, int nsig, float* out);

#ifdef __cplusplus
}
#endif

#endif /* VK_IO_H_ */
