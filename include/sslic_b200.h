/*
 * sslic_b200 — C ABI of the B200-native SSLIC hot path (sm_100a).
 *
 * Drop-in boundary for the reference's C++ SLIC interface
 * (/root/reference/proj/include/sslic/). Every entry point below names the
 * reference function it replaces. Plain pointers and sizes only; no torch or
 * C++ types cross this boundary. The C++ adapter over the reference's own
 * types is include/sslic_b200.hpp; the Python mirror is
 * paper_1806_08741_b200/__init__.py.
 *
 * Conventions
 *  - Layout is the reference's frozen layout (image.hpp:1-5): axis 0 fastest,
 *    channels interleaved; rank 1..4 (image.hpp:25).
 *  - Status codes mirror the reference's exception classes
 *    (SURVEY §8b "Errors"): SSLIC_EINVAL = std::invalid_argument,
 *    SSLIC_ELOGIC = std::logic_error, SSLIC_ERANGE = std::out_of_range.
 *    sslic_last_error() returns the thread's last message.
 *  - Host entry points take HOST buffers and copy; engine entry points work on
 *    DEVICE buffers and run on the caller's CUDA stream.
 *  - There is no CPU fallback: every compute entry point runs CUDA kernels and
 *    fails with SSLIC_ECUDA when no sm_100 device is usable.
 */
#ifndef SSLIC_B200_H
#define SSLIC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSLIC_OK 0
#define SSLIC_EINVAL (-1) /* std::invalid_argument (slic.hpp:52-64, image.hpp:238-249) */
#define SSLIC_ELOGIC (-2) /* std::logic_error (slic.hpp:330-331) */
#define SSLIC_ERANGE (-3) /* std::out_of_range (image.hpp:112-124) */
#define SSLIC_ECUDA (-4)
#define SSLIC_ENOMEM (-5)
/* io_error (io.hpp:40-56) by io_errc */
#define SSLIC_EIO_NOT_FOUND (-10) /* file_not_found */
#define SSLIC_EIO_HEADER (-11)    /* malformed_header */
#define SSLIC_EIO_SIZE (-12)      /* size_mismatch */
#define SSLIC_EIO_TYPE (-13)      /* unsupported_type */
#define SSLIC_EIO_WRITE (-14)     /* write_failed */

#define SSLIC_UNDEFINED 0xffffffffu /* LabelMap::kUndefined (image.hpp:291) */

typedef enum {
  SSLIC_U8 = 0,  /* io.hpp:67-71 uint8 volumes */
  SSLIC_U16 = 1, /* config 3 (not readable by the reference I/O; exact in fp64) */
  SSLIC_F32 = 2, /* io.hpp:67-71 float32 volumes */
  SSLIC_F64 = 3  /* NDImage's own storage (image.hpp:284) */
} sslic_dtype;

/* NDImage (image.hpp:236-285) in its native storage type. */
typedef struct {
  int rank;          /* 1..4 */
  int64_t dims[4];   /* extents, axis 0 fastest */
  int channels;      /* >= 1, interleaved */
  int dtype;         /* sslic_dtype */
  const void* data;  /* host or device pointer (see each entry point) */
} sslic_image;

/* SlicParams (slic.hpp:34-65). */
typedef struct {
  int64_t grid[4];            /* S per axis, 1 <= S <= dims */
  double weight_m;            /* m > 0 (default 10) */
  int max_iterations;         /* 0 => 10 for rank <= 2, 5 otherwise */
  int enforce_connectivity;   /* used by sslic_segment only */
  int has_residual_threshold; /* std::optional<double> residual_threshold */
  double residual_threshold;
} sslic_params;

const char* sslic_last_error(void);
const char* sslic_version(void);

/* k = prod ceil(d_a/S_a) (slic.hpp:212-216); 0 on invalid input. */
int64_t sslic_cluster_count(int rank, const int64_t* dims, const int64_t* grid);
int sslic_iterations_for(const sslic_params* p, int rank); /* SlicParams::iterations_for 47-50 */

/* run_slic (slic.hpp:384-415). img->data is HOST memory. Outputs (host):
 *   labels_out[N] (uint32), centers_out[k*(c+rank)], residuals_out[iterations],
 *   *iterations_done. The reference's `workers` maps to nothing: one device.
 * Host buffers may be pageable or pinned: large pageable buffers travel in
 * stripes over host threads and pinned staging (csrc/hostcopy.cu); pinned,
 * device-mapped label buffers of >= 2^24 voxels get the overlapped download.
 * An SSLIC_F64 image whose values are all uint8 / uint16 / float32 numbers (the
 * reference's NDImage stores doubles, image.hpp:236-285) is narrowed
 * losslessly on the device and runs the native-dtype kernels. */
int sslic_run_slic(const sslic_image* img, const sslic_params* params, int device,
                   uint32_t* labels_out, double* centers_out, double* residuals_out,
                   int* iterations_done);

/* run_slic followed by enforce_connectivity (tools/sslic.cpp:104-108).
 * *next_label_out = the sweep's next unused label. */
int sslic_segment(const sslic_image* img, const sslic_params* params, int device,
                  uint32_t* labels_out, double* centers_out, double* residuals_out,
                  int* iterations_done, uint32_t* next_label_out);

/* The tools/sslic.cpp pipeline (run_slic, enforce_connectivity when
 * params->enforce_connectivity, write_labels; tools/sslic.cpp:104-109) plus,
 * when contour_path is not NULL, write_volume(contour_path,
 * mask_label_contour(img, labels)) in float32 (tools/sslic.cpp:121-125,
 * io.hpp:362-392,432-454). The label count of the labels header and the
 * contour bitmask come out of the final relabel pass on the device (no extra
 * pass over the map). centers_out / residuals_out as sslic_run_slic. */
int sslic_segment_write(const sslic_image* img, const sslic_params* params, int device,
                        const char* labels_path, const char* contour_path, double* centers_out,
                        double* residuals_out, int* iterations_done, uint32_t* next_label_out);
/* init_centers (slic.hpp:206-230) [+ perturb_centers (236-267) when perturb].
 * centers_out: k*(c+rank) doubles (host). */
int sslic_init_centers(const sslic_image* img, const sslic_params* params, int perturb,
                       int device, double* centers_out);

/* perturb_centers (slic.hpp:236-267) of a caller-given table (host, in-out). */
int sslic_perturb_centers(const sslic_image* img, double* centers, int64_t k, int device);

/* convert_image_to_lab (color.hpp:54-66): 3-channel sRGB in [0, 255] to
 * CIE-Lab, npix*3 doubles into lab_out (host). SSLIC_EINVAL unless 3 channels.
 * Integral inputs reproduce the reference's transfer values bitwise; the cube
 * root is the device's (Lab within ~1e-13 of the reference). */
int sslic_convert_image_to_lab(const sslic_image* img, int device, double* lab_out);

/* mask_label_contour (io.hpp:432-454): copy of the image (fp64, npix*c into
 * out, host) with every voxel that has a face neighbour of a different label
 * zeroed in all channels. SSLIC_EINVAL if the label dims differ. */
int sslic_mask_label_contour(const sslic_image* img, int label_rank, const int64_t* label_dims,
                             const uint32_t* labels, int device, double* out);

/* gradient_magnitude_sq (color.hpp:71-102) at n coordinates (host, n*rank). */
int sslic_gradient_sq(const sslic_image* img, const int64_t* coords, int64_t n, int device,
                      double* out);

/* squared_distance (slic.hpp:189-200) for n (center, pixel, coord) triples,
 * evaluated by the device's exact distance routine (host buffers). */
int sslic_squared_distance(int channels, int rank, const int64_t* grid, double weight_m,
                           int64_t n, const double* centers, const double* pixels,
                           const int64_t* coords, int device, double* out);

/* One assign_labels pass over the whole image (slic.hpp:275-310) with
 * caller-owned labels/dists (host, in-out): the compat path used for the
 * "single pass bit-exact given identical centres" gate. */
int sslic_assign_pass(const sslic_image* img, const sslic_params* params, const double* centers,
                      int64_t k, int device, uint32_t* labels, double* dists);

/* accumulate_region over the whole image + merge (slic.hpp:315-346, 133-143).
 * sums_out[k*(c+rank)] (double), counts_out[k]. ELOGIC on undefined labels. */
int sslic_accumulate(const sslic_image* img, const uint32_t* labels, int64_t k, int device,
                     double* sums_out, int64_t* counts_out);

/* reduce_and_update (slic.hpp:352-372) on merged sums/counts: centers in-out,
 * residual out. */
int sslic_reduce_and_update(double* centers, int64_t k, int stride, const double* sums,
                            const int64_t* counts, int device, double* residual_out);

/* enforce_connectivity (connectivity.hpp:265-273). Host buffers. */
int sslic_enforce_connectivity(int rank, const int64_t* dims, const uint32_t* labels_in,
                               const double* centers, int channels, int64_t k,
                               const int64_t* grid, int device, uint32_t* labels_out,
                               uint32_t* next_label_out);

/* ------------------------------------------------------------------------ */
/* Device-resident engine: the per-iteration loop on HBM-resident data, one  */
/* z-slab (last axis) per GPU. Used by bench.py and multi-GPU runs.          */
/* ------------------------------------------------------------------------ */
typedef struct sslic_engine sslic_engine;

/* img->dims are the FULL image; img->data is a DEVICE pointer to planes
 * [data_begin, data_end) of the last axis, which must cover
 * [slab_begin-2, slab_end+2) clipped to the image (the perturbation halo).
 * stream: cudaStream_t (NULL = legacy default). */
int sslic_engine_create(const sslic_image* img, const sslic_params* params, int device,
                        int64_t slab_begin, int64_t slab_end, int64_t data_begin,
                        int64_t data_end, void* stream, sslic_engine** out);
int sslic_engine_destroy(sslic_engine* e);

/* init_centers + perturb_centers for the clusters whose initial cell centre
 * lies in this slab (zeros elsewhere). With several slabs, sum the tables
 * across ranks (exact: one non-zero term per entry) then commit. */
int sslic_engine_init(sslic_engine* e);
/* Back to iteration 0 (every label undefined, zero sums): the same engine
 * then runs another whole run from sslic_engine_init (bench: timed runs
 * over the configured iteration window). */
int sslic_engine_reset(sslic_engine* e);
int sslic_engine_centers_buffer(sslic_engine* e, double** dev_ptr, int64_t* count);
int sslic_engine_commit_centers(sslic_engine* e);

/* Fused assign_labels + accumulate_region over the slab (one iteration's
 * map phase). Per-cluster partial sums land in the int64 partials buffer
 * (k*(c+rank+1)); sum it across ranks before sslic_engine_update. */
int sslic_engine_assign(sslic_engine* e);
int sslic_engine_partials(sslic_engine* e, int64_t** dev_ptr, int64_t* count);
/* reduce_and_update on the (reduced) partials; residual kept on device. */
int sslic_engine_update(sslic_engine* e);
/* assign + update (single slab covering the whole image). */
int sslic_engine_iterate(sslic_engine* e, int iterations);
/* Same, captured as one CUDA graph and launched once (single-GPU loops);
 * ms_out (nullable) receives the device time of the launch. */
int sslic_engine_iterate_graph(sslic_engine* e, int iterations, float* ms_out);

int sslic_engine_iterations_done(sslic_engine* e);
/* Copies residuals of the iterations done so far (host). Synchronizes. */
int sslic_engine_residuals(sslic_engine* e, double* host_out);
/* Slab labels (plain uint32, tags stripped) into a DEVICE buffer. */
int sslic_engine_labels(sslic_engine* e, uint32_t* dev_out);
int sslic_engine_centers(sslic_engine* e, double* host_out);
/* Number of voxels whose label was undefined at the last accumulation
 * (the reference throws std::logic_error for any). Synchronizes. */
int64_t sslic_engine_undefined_count(sslic_engine* e);
/* Kernel launches issued by the engine so far (bench.py's gpu_launches). */
int64_t sslic_engine_launch_count(sslic_engine* e);
/* Device time (ms, CUDA events on the engine stream) of the i-th assign
 * kernel launch since creation; *n_out = launches recorded. Synchronizes. */
int sslic_engine_assign_ms(sslic_engine* e, int i, float* ms_out, int* n_out);
/* Value range of the engine's data: max |value| over its planes for float
 * images (the dtype maximum for u8/u16). Multi-GPU: set every rank's engine
 * to the MAX over ranks (after create, before init) so that the fixed-point
 * per-cluster sums that are allreduced share one scale and the fp32 filter
 * margins cover centres built from every rank's voxels -- the z-slab split
 * of the reference's exact accumulate_region / reduce_and_update
 * (slic.hpp:315-372). */
int sslic_engine_value_range(sslic_engine* e, double* absmax_out);
int sslic_engine_set_value_range(sslic_engine* e, double absmax);
/* Force the exact fp64 assignment kernel (1) or allow the fast fp32-filter
 * kernel where supported (0, default). Both produce identical labels. */
int sslic_engine_set_exact(sslic_engine* e, int exact);
/* Fast-path statistics of the last assign: voxels re-decided in fp64 and
 * CTAs that took the crowded-region exact fallback. Synchronizes. */
int sslic_engine_fast_stats(sslic_engine* e, double* ambiguous, double* overflow_blocks,
                            double* changed);
/* Enable counting of candidate evaluations / window volumes in assign. */
int sslic_engine_set_stats(sslic_engine* e, int on);
/* Assignment evaluation statistics of the last assign (bench roofline):
 * *evals = candidate evaluations actually performed, *window_evals =
 * sum_k |W_k ∩ slab| (the algorithmic count). Synchronizes. */
int sslic_engine_eval_stats(sslic_engine* e, double* evals, double* window_evals);

/* ---- multi-GPU (z-slabs, one NCCL allreduce of the int64 per-cluster
 * partials per iteration) ------------------------------------
 * The reference parallelises run_slic(img, params, workers) over slabs with
 * an ordered merge of per-slab accumulators (slic.hpp:384-415,
 * parallel.hpp:52-94); here the slabs are z-slabs of a 3-D volume, one per
 * GPU, and results are bitwise the single-GPU result for any device count. */

/* run_slic over `n_devices` GPUs of this process (devices: their indices, or
 * NULL for 0..n-1): one host thread per device, ncclCommInitAll. img / labels
 * / centres / residuals as sslic_run_slic (host buffers, full image).
 * n_devices > 1 needs a rank-3 image with at least n_devices planes. */
int sslic_run_slic_multi(const sslic_image* img, const sslic_params* params, int n_devices,
                         const int* devices, uint32_t* labels_out, double* centers_out,
                         double* residuals_out, int* iterations_done);
/* One rank of a one-process-per-GPU job (torchrun): img->dims are the FULL
 * image; img->data points at plane `data_first_plane` of it (0: the whole
 * host image) and must hold this rank's slab plus a 2-plane halo (only those
 * planes are uploaded, sslic_slab_bounds gives the slab); labels_out
 * receives this rank's slab (sslic_slab_bounds); centres / residuals /
 * iterations_done (nullable) are the same on every rank. nccl_id: the
 * NCCL_UNIQUE_ID_BYTES from sslic_nccl_unique_id on one rank, given to all
 * (may be NULL when world == 1: no communicator). Collective: every rank must
 * call it. The communicator is cached per (id, rank, world, device) for the
 * process lifetime, so successive calls with one id skip its setup. */
int sslic_run_slic_rank(const sslic_image* img, const sslic_params* params, int rank, int world,
                        const void* nccl_id, int device, int64_t data_first_plane,
                        uint32_t* labels_out, double* centers_out, double* residuals_out,
                        int* iterations_done);
/* Number of visible CUDA devices (0 when none). */
int sslic_device_count(void);
/* ncclGetUniqueId into out (bytes >= 128). */
int sslic_nccl_unique_id(void* out, int64_t bytes);
/* The z-slab [lo, hi) of `rank` (slabs rounded to multiples of `align` planes
 * when there are at least `world` such units). */
int sslic_slab_bounds(int64_t last, int world, int rank, int64_t align, int64_t* lo,
                      int64_t* hi);
/* Attach an NCCL communicator to an engine (collective over the ranks):
 * sslic_engine_start, _iterate and _iterate_graph then run the value-range
 * MAX, the SUM of the init tables and the per-iteration SUM of the partials
 * on the engine's stream (inside the captured graph). nccl_id == NULL (world
 * 1) detaches. A 1-rank communicator is valid (the NCCL path on one GPU). */
int sslic_engine_attach_nccl(sslic_engine* e, const void* nccl_id, int rank, int world);
/* init + perturb of the slab's clusters, the synced table, anchors and bins
 * (with a communicator: value-range MAX first, table SUM before the commit). */
int sslic_engine_start(sslic_engine* e);

/* Seeded synthetic volumes for the five BASELINE configs, generated on the
 * device straight into HBM (planes [z_begin, z_end) of the last axis). */
int sslic_synth_generate(int config, int rank, const int64_t* dims, int channels, int dtype,
                         uint64_t seed, int64_t z_begin, int64_t z_end, void* dev_out,
                         void* stream);

/* ---- detached-header raw volumes (io.hpp:57-202, 337-428) ----------------
 * Types uint8 / uint16 / float32 for images, uint32 for label maps; little
 * endian. PNG paths fail with SSLIC_EIO_TYPE (this build has no libpng). */
typedef struct {
  int rank;
  int64_t dims[4];
  int channels;
  int dtype;      /* sslic_dtype of an image volume; -1 for a label map */
  int label_map;  /* type uint32 */
} sslic_volume_info;

/* parse_volume_header (io.hpp:123-190). */
int sslic_volume_info_read(const char* header_path, sslic_volume_info* out);
/* read_volume (io.hpp:337-360) without the fp64 widening: planes
 * [plane_begin, plane_end) of the last axis, native dtype, into dst — host
 * memory when device < 0, else device memory on that device, streamed from
 * disk through pinned staging (a z-slab rank reads only its planes). */
int sslic_volume_read(const char* header_path, int64_t plane_begin, int64_t plane_end, void* dst,
                      int device);
/* write_volume (io.hpp:362-392) in the image's own dtype (u8/u16/f32; host). */
int sslic_volume_write(const char* header_path, const sslic_image* img);
/* write_labels / read_labels (io.hpp:396-428): uint32 label maps (host). */
int sslic_labels_write(const char* header_path, int rank, const int64_t* dims,
                       const uint32_t* labels);
int sslic_labels_read(const char* header_path, uint32_t* labels_out);

#ifdef __cplusplus
}
#endif
#endif
