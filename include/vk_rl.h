/*
 * vk_rl.h — C ABI of the B200-native Richardson–Lucy deconvolution path.
 *
 * This is the drop-in boundary for the reference's deconvolution API
 * (reference: proj/include/voxelkit/deconv.hpp:28-103, implemented in
 * proj/src/deconv.cpp).  Plain pointers and sizes only; no exception or C++
 * type crosses it.  Every entry point names the reference interface it
 * replaces.  The reference's C++ signatures are restored on top of this ABI by
 * paper_2510_14143_b200/host/deconv_b200.cpp.
 *
 * Conventions
 *  - Images are contiguous row-major float32, axes ZYX / YX / X (rank 1..3),
 *    exactly NdImage's layout (proj/include/voxelkit/image.hpp:46-48).
 *  - Functions suffixed _device take device pointers on the plan's GPU and a
 *    cudaStream_t (passed as void*, NULL = legacy default stream); the others
 *    take host pointers: pinned (page-locked) buffers are DMA'd directly,
 *    pageable ones are copied through the plan's ring of pinned chunks, the
 *    host copy of one chunk (split over a worker pool, VK_RL_HOST_THREADS)
 *    overlapping the DMA of the previous one.
 *  - Every function returns a vk_status.  On failure vk_last_error() returns
 *    the exact message the reference would put in the exception's what()
 *    (thread-local, valid until the next call on the same thread), and the
 *    contents of output buffers are unspecified (a pageable output may have
 *    been faulted in, i.e. zeroed, while the run was in flight).
 *  - A plan is not re-entrant (one run at a time, like RlTransforms,
 *    deconv.hpp:64-65); distinct plans may be used concurrently.
 */
#ifndef VK_RL_H_
#define VK_RL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VK_RL_ABI_VERSION 4
#define VK_MAX_RANK 3

/* Status codes; each maps to one reference exception type
 * (proj/include/voxelkit/errors.hpp:25-70). */
typedef enum vk_status {
  VK_OK = 0,
  VK_ERR_ARG = 1,              /* voxelkit::Error                 */
  VK_ERR_SHAPE = 2,            /* voxelkit::ShapeMismatch         */
  VK_ERR_NEGATIVE = 3,         /* voxelkit::NegativeInput         */
  VK_ERR_UNNORMALIZED_PSF = 4, /* voxelkit::UnnormalizedPsf       */
  VK_ERR_DEGENERATE_REF = 5,   /* voxelkit::DegenerateReference   */
  VK_ERR_TOO_SMALL = 6,        /* voxelkit::TooSmall              */
  VK_ERR_ODD_EXTENT = 7,       /* voxelkit::OddExtent             */
  VK_ERR_CUDA = 8,             /* CUDA runtime failure            */
  VK_ERR_OOM = 9,              /* device allocation failure       */
  VK_ERR_UNSUPPORTED = 10,     /* not implemented on this path    */
  VK_ERR_KERNEL_TOO_LARGE = 11, /* voxelkit::KernelTooLarge       */
  VK_ERR_BAD_MAGIC = 12,        /* voxelkit::BadMagic             */
  VK_ERR_HEADER_MISMATCH = 13,  /* voxelkit::HeaderMismatch       */
  VK_ERR_TRUNCATED = 14,        /* voxelkit::TruncatedPayload     */
  VK_ERR_PLACEMENT = 15,        /* voxelkit::PlacementFailure     */
  VK_ERR_EVEN_EXTENT = 16       /* voxelkit::EvenExtent           */
} vk_status;

/* deconv::StopMetric (deconv.hpp:28) */
typedef enum vk_stop_metric {
  VK_METRIC_SI_PSNR_VS_INPUT = 0,
  VK_METRIC_SSIM_VS_PREV = 1,
  VK_METRIC_FRC_RESOLUTION = 2
} vk_stop_metric;

/* deconv::StoppingRule (deconv.hpp:35-40), plus the physical x spacing the
 * reference takes from observed.spacing()->back() for the FRC metric
 * (deconv.cpp:285-289); 0 means "no spacing" (= 1.0). */
typedef struct vk_stop_rule {
  int metric; /* vk_stop_metric */
  double rel_tol;
  int patience;
  int max_iters;
  double spacing;
} vk_stop_rule;

/* deconv::IterationTrace (deconv.hpp:49-59).  Arrays are caller-allocated
 * with `capacity` >= rule.max_iters entries (any may be NULL). */
typedef struct vk_trace {
  int capacity;
  double* metric;         /* IterationRecord::value                  */
  double* wall_s;         /* IterationRecord::wall_time_s (device)   */
  double* log_likelihood; /* IterationTrace::log_likelihood          */
  int iters_run;          /* records.size()                          */
  int stop_reason;        /* 0 "max_iters", 1 "converged"            */
  uint64_t fft_shape[VK_MAX_RANK]; /* IterationTrace::fft_shape      */
} vk_trace;

typedef struct vk_rl_plan_s* vk_rl_plan;

/* Replaces RlTransforms::RlTransforms(shape, psf, threads) plus, with
 * pad_replicate = 1, padded_domain() of richardson_lucy
 * (deconv.cpp:110-131, 205-219, 331-332).
 *   pad_replicate = 1: `shape` is the IMAGE shape; the plan iterates on
 *                      P = I + 2 floor(K/2) (richardson_lucy).
 *   pad_replicate = 0: `shape` is the convolution domain itself (RlTransforms,
 *                      rl_step).
 * Validates the PSF rank (ShapeMismatch), builds both OTFs on `device`. */
vk_status vk_rl_plan_create(int device, int rank, const uint64_t* shape, int psf_rank,
                            const uint64_t* psf_shape, const float* psf, int pad_replicate,
                            vk_rl_plan* out);

/* RlTransforms::image_shape() / fft_shape() (deconv.hpp:73-74) plus the
 * iteration domain.  Arrays hold `rank` entries. */
vk_status vk_rl_plan_shapes(vk_rl_plan plan, int* rank, uint64_t* image_shape,
                            uint64_t* domain_shape, uint64_t* fft_shape);

/* Human-readable execution plan: FFT grid, kernel variant per axis, y/z
 * convolution strategy (for logs and the bench's config record). */
vk_status vk_rl_plan_describe(vk_rl_plan plan, char* buf, int len);

/* Bytes of device memory the plan holds. */
vk_status vk_rl_plan_device_bytes(vk_rl_plan plan, uint64_t* bytes);

vk_status vk_rl_plan_destroy(vk_rl_plan plan);

/* The loop of richardson_lucy (deconv.cpp:333-430) on a pad_replicate plan:
 * observed (image shape) -> estimate (image shape), trace filled.  Checks the
 * rule and observed >= 0 in the reference's order (deconv.cpp:306-318); the
 * PSF was checked when the plan was created. */
vk_status vk_rl_run(vk_rl_plan plan, const float* observed, float* estimate,
                    const vk_stop_rule* rule, int flat_init, vk_trace* trace);
vk_status vk_rl_run_device(vk_rl_plan plan, const float* d_observed, float* d_estimate,
                           const vk_stop_rule* rule, int flat_init, vk_trace* trace,
                           void* stream);

/* Independent volumes through one plan (one OTF, reused), e.g. the C3 / C5
 * batches.  traces may be NULL or an array of n. */
vk_status vk_rl_run_batch(vk_rl_plan plan, int n, const float* const* observed,
                          float* const* estimate, const vk_stop_rule* rule, int flat_init,
                          vk_trace* traces);

/* The same on device buffers.  The volumes run concurrently on the plan's
 * batch lanes (clones with their own work buffers and stream, one host thread
 * each; VK_RL_LANES overrides the count), so short per-volume grids overlap
 * and fill the GPU.  Inputs must be ready on `stream`; the call returns when
 * every estimate is written. */
vk_status vk_rl_run_batch_device(vk_rl_plan plan, int n, const float* const* d_observed,
                                 float* const* d_estimate, const vk_stop_rule* rule, int flat_init,
                                 vk_trace* traces, void* stream);
/* Lanes currently allocated (1 + clones). */
vk_status vk_rl_plan_lanes(vk_rl_plan plan, int* lanes);

/* rl_step(estimate, observed, transforms) (deconv.cpp:178-194) on a
 * pad_replicate = 0 plan: one multiplicative update on the plan's domain. */
vk_status vk_rl_step(vk_rl_plan plan, const float* estimate, const float* observed, float* out);
vk_status vk_rl_step_device(vk_rl_plan plan, const float* d_estimate, const float* d_observed,
                            float* d_out, void* stream);

/* richardson_lucy(observed, psf, rule, flat_init) (deconv.cpp:304-431) in one
 * call, with the reference's exact validation order: rule, rank, observed
 * negativity, PSF negativity, PSF sum.  The reference builds its transforms
 * per call (deconv.cpp:332); here the one-shot calls (this one,
 * vk_rl_step_psf, vk_fft_convolve) keep their plans in a process-wide LRU
 * cache keyed on (device, shapes, PSF values): VK_RL_PLAN_CACHE plans
 * (default 2; 0 = build and free per call, as the reference does). */
vk_status vk_richardson_lucy(int device, int rank, const uint64_t* shape, const float* observed,
                             int psf_rank, const uint64_t* psf_shape, const float* psf,
                             const vk_stop_rule* rule, int flat_init, float* estimate,
                             vk_trace* trace);

/* n independent volumes of one shape, each exactly as vk_richardson_lucy
 * would deconvolve it, through one cached plan and its batch lanes
 * (include/voxelkit_b200/deconv_batch.hpp; the C3 / C5 batches).  traces may
 * be NULL or an array of n.  On failure the message names the volume. */
vk_status vk_richardson_lucy_batch(int device, int rank, const uint64_t* shape, int n,
                                   const float* const* observed, int psf_rank,
                                   const uint64_t* psf_shape, const float* psf,
                                   const vk_stop_rule* rule, int flat_init, float* const* estimate,
                                   vk_trace* traces);

/* rl_step(estimate, observed, psf) registry form (deconv.cpp:196-200,
 * 437-449): transforms built for the call. */
vk_status vk_rl_step_psf(int device, int rank, const uint64_t* shape, const float* estimate,
                         const float* observed, int psf_rank, const uint64_t* psf_shape,
                         const float* psf, float* out);

/* filters::fft_convolve(img, kernel, circular) (filters.cpp:174-264) and its
 * registry op "fft_convolve" (filters.cpp:316-323) on the same transforms.
 * Linear: zero-padded to good_size(A + K - 1) per axis, the centred same-size
 * result (crop at (K-1)/2).  Circular: on the image grid itself with the
 * kernel centre wrapped to index 0 (KernelTooLarge if a kernel extent exceeds
 * the image's; extents must be 5-smooth on this path, else
 * VK_ERR_UNSUPPORTED).  The kernel is used as given (no sign or sum checks,
 * as in the reference).  Rank mismatch -> ShapeMismatch.  A conv plan is only
 * valid with the vk_conv_* calls. */
vk_status vk_conv_plan_create(int device, int rank, const uint64_t* shape, int kernel_rank,
                              const uint64_t* kernel_shape, const float* kernel, int circular,
                              vk_rl_plan* out);
vk_status vk_conv_run(vk_rl_plan plan, const float* image, float* out);
vk_status vk_conv_run_device(vk_rl_plan plan, const float* d_image, float* d_out, void* stream);
vk_status vk_fft_convolve(int device, int rank, const uint64_t* shape, const float* image,
                          int kernel_rank, const uint64_t* kernel_shape, const float* kernel,
                          int circular, float* out);

/* ---- Single-volume slab decomposition --------------------
 * richardson_lucy on a 3D volume split into `nslabs` z slabs of the padded
 * domain P, one plan per slab (per GPU).  Slab r owns P rows [own_begin,
 * own_end) and computes on [domain_begin, domain_end) = the owned rows plus
 * the correlations' reach (Kz-1-cz below, cz above, clipped to P).  After
 * every x pass the caller overwrites the halo rows of each plan's x-spectrum
 * S_A with the neighbours' owned rows (ncclSend/Recv, peer copies, ...):
 * rows are [kx][row][y] complex64 at `spectrum`, `kx_planes` planes of `rows`
 * rows of `row_elems` elements; halo_below rows start at local row 0, the
 * halo_above rows at rows - halo_above, and the matching source rows are the
 * neighbour's first / last owned rows.  Sums (stats, per-iteration LL and
 * si_psnr sums) are per slab; the caller adds them up (all-reduce).  The
 * stopping rule runs on the caller's side; si_psnr only.
 *
 *   begin(obs_local) -> stats[8]: Σr, Σr², min, max, Σ obs_p over owned rows,
 *                       negative flag, image voxels, owned P voxels
 *   start(iters, flat_init, mean)     -> x pass      [exchange]
 *   per iteration it = 1..:
 *     forward(obs, it)                -> x pass      [exchange]
 *     backward(obs, it, out or NULL)  -> x pass      [exchange unless last]
 *   crop(out) (after a non-final backward), sums(iters) -> acc[iters][4]:
 *     log-likelihood, Σx, Σx², Σx·r of the owned image rows. */
typedef struct vk_slab_info {
  int own_begin, own_end;        /* global P rows owned                    */
  int domain_begin, domain_end;  /* global P rows of the local domain      */
  int image_begin, image_end;    /* global image rows owned (obs / output) */
  int halo_below, halo_above;    /* halo rows of the local domain          */
  void* spectrum;                /* S_A (device)                           */
  uint64_t kx_planes, rows, row_elems;
} vk_slab_info;

vk_status vk_rl_slab_plan_create(int device, const uint64_t* shape, const uint64_t* psf_shape,
                                 const float* psf, int nslabs, int slab, vk_rl_plan* out,
                                 vk_slab_info* info);
vk_status vk_rl_slab_begin(vk_rl_plan plan, const float* d_observed_rows, double* stats, void* stream);
vk_status vk_rl_slab_start(vk_rl_plan plan, int iters, int flat_init, double mean, void* stream);
vk_status vk_rl_slab_forward(vk_rl_plan plan, const float* d_observed_rows, int iter, void* stream);
vk_status vk_rl_slab_backward(vk_rl_plan plan, const float* d_observed_rows, int iter, float* d_out_rows,
                              void* stream);
vk_status vk_rl_slab_crop(vk_rl_plan plan, float* d_out_rows, void* stream);
vk_status vk_rl_slab_sums(vk_rl_plan plan, int iters, double* acc, void* stream);
/* Halo traffic: S_A rows [row, row+n) of every kx plane to / from a packed
 * [kx_planes][n][row_elems] complex64 device buffer (for ncclSend/Recv), or
 * directly between two slab plans (same device or peers). */
vk_status vk_rl_slab_pack(vk_rl_plan plan, int row, int n, void* d_buf, void* stream);
vk_status vk_rl_slab_unpack(vk_rl_plan plan, int row, int n, const void* d_buf, void* stream);
vk_status vk_rl_slab_copy_rows(vk_rl_plan src, int src_row, vk_rl_plan dst, int dst_row, int n, void* stream);

/* Frees every idle plan held by the one-shot calls' cache (device memory). */
vk_status vk_plan_cache_clear(void);

/* fftx::good_size (fft_plan.cpp:41-49). */
uint64_t vk_good_size(uint64_t n);

/* Per-iteration kernel launches of the last run on this plan (evidence for
 * the bench's gpu_launches). */
vk_status vk_rl_plan_launches(vk_rl_plan plan, uint64_t* launches);

/* Kernel kinds for per-launch profiling. */
typedef enum vk_kernel_kind {
  VK_KIND_X_FWD = 0,    /* x-pass: R2C of the initial estimate          */
  VK_KIND_X_RATIO = 1,  /* x-pass: C2R -> ratio (+LL) -> R2C            */
  VK_KIND_X_UPDATE = 2, /* x-pass: C2R -> update/clip (+metric) -> R2C  */
  VK_KIND_Y_FWD = 3,    /* y-pass forward                               */
  VK_KIND_Z_CONV = 4,   /* z-pass forward * OTF * inverse               */
  VK_KIND_Y_INV = 5,    /* y-pass inverse                               */
  VK_KIND_Y_CONV = 6,   /* y-pass forward * OTF * inverse (rank <= 2)   */
  VK_KIND_YZ_DATAFLOW = 7, /* reserved (retired one-launch y/z schedule)   */
  VK_KIND_YZ_CLUSTER = 8,  /* reserved (retired cluster y/z schedule)       */
  VK_KIND_COUNT = 9
} vk_kernel_kind;

/* Enable/disable CUDA-event timing of every launch on this plan (events are
 * recorded on the launch stream around each kernel). */
vk_status vk_rl_plan_profile(vk_rl_plan plan, int enable);
/* Accumulated device ms and launch counts per kind since the last reset, and
 * the algorithmic HBM bytes of one launch of each kind (SURVEY.md §8(d):
 * spectra, observed and estimate; the OTF is not counted). */
vk_status vk_rl_plan_profile_read(vk_rl_plan plan, int n_kinds, double* ms_total, uint64_t* launches,
                                  uint64_t* alg_bytes_per_launch, int reset);

/* OTF bytes one launch of each kind reads (0 for a factored, separable OTF). */
vk_status vk_rl_plan_otf_bytes(vk_rl_plan plan, int n_kinds, uint64_t* otf_bytes_per_launch);

const char* vk_last_error(void);
int vk_abi_version(void);

/* Debug: with VK_RL_GUARD=1 in the environment every device buffer a plan
 * allocates carries a 64 KB guard band of a fixed pattern on each side.
 * Returns the number of bands found overwritten (freed buffers so far plus
 * the live ones checked now), or -1 when guards are off. */
int vk_debug_guard_check(void);

#ifdef __cplusplus
}
#endif

#endif /* VK_RL_H_ */
