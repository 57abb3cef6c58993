/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the SSLIC hot path.
 *
 * A plain-C restatement of the reference algorithm
 * (/root/reference/proj/include/sslic/{slic,color,connectivity}.hpp), used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker. Nothing in the product path (paper_1806_08741_b200/) links, loads
 * or calls this code.
 *
 * Parity pinning: the restatement is checked against
 *   (1) the reference itself, compiled from its own headers into
 *       oracle/_ref/libsslic_ref.so by oracle/Makefile (ref_harness.cpp), and
 *   (2) golden fixtures in tests/golden/ produced by that reference build
 *       (tests/golden/make_golden.py), including the reference test-suite
 *       corpora regenerated from their seeds.
 *
 * Layout follows image.hpp:1-5: axis 0 fastest, channels interleaved.
 * All arithmetic is fp64 compiled with -ffp-contract=off, as the reference
 * library target requires (proj/CMakeLists.txt:18-20).
 */
#ifndef SSLIC_ORACLE_H
#define SSLIC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_UNDEFINED 0xffffffffu

/* k = prod ceil(d_a / S_a)   (slic.hpp:206-215) */
int64_t orc_cluster_count(int rank, const int64_t* dims, const int64_t* grid);

/* init_centers (slic.hpp:206-230). centers: k*(c+rank) doubles. */
void orc_init_centers(int rank, const int64_t* dims, int channels, const double* data,
                      const int64_t* grid, double* centers);

/* gradient_magnitude_sq (color.hpp:71-102) at a flat offset. */
double orc_gradient_sq(int rank, const int64_t* dims, int channels, const double* data,
                       const int64_t* coord);

/* perturb_centers (slic.hpp:236-267), in place. */
void orc_perturb_centers(int rank, const int64_t* dims, int channels, const double* data,
                         double* centers, int64_t k);

/* squared_distance_raw (slic.hpp:156-171). */
double orc_distance(const double* center, const double* pixel, const int64_t* coord,
                    int channels, int rank, const int64_t* grid, double m_sq);

/* assign_labels over the full image (slic.hpp:275-310), labels/dists in-out. */
void orc_assign(int rank, const int64_t* dims, int channels, const double* data,
                const double* centers, int64_t k, const int64_t* grid, double weight_m,
                uint32_t* labels, double* dists);

/* accumulate_region per slab + ordered merge (slic.hpp:315-346, 133-143).
 * slab_rows = S_last reproduces run_slic's decomposition; <= 0 = one pass.
 * sums: k*(c+rank) doubles (zeroed here), counts: k int64.
 * Returns 0, or -1 when a pixel carries the undefined label (the reference
 * throws std::logic_error, slic.hpp:330-331), or -2 when a label >= k. */
int orc_accumulate(int rank, const int64_t* dims, int channels, const double* data,
                   const uint32_t* labels, int64_t k, int64_t slab_rows, double* sums,
                   int64_t* counts);

/* reduce_and_update (slic.hpp:352-372) on an already merged accumulator.
 * Updates centers in place and returns the residual. */
double orc_update(double* centers, int64_t k, int stride, const double* sums,
                  const int64_t* counts);

/* run_slic (slic.hpp:384-415). iterations: 0 => 10 for rank<=2, else 5.
 * residuals: capacity >= iterations. Returns 0, or a negative status
 * (-1 undefined label during accumulation, -3 invalid parameter). */
int orc_run_slic(int rank, const int64_t* dims, int channels, const double* data,
                 const int64_t* grid, double weight_m, int max_iterations, int has_threshold,
                 double threshold, uint32_t* labels, double* centers, double* residuals,
                 int* iterations_done);

/* size_threshold (connectivity.hpp:34-38) */
int64_t orc_size_threshold(int rank, const int64_t* grid);

/* mask_label_contour (io.hpp:432-454): pixels with a face neighbour of a
 * different label are zeroed in every channel, the rest copied. */
void orc_mask_label_contour(int rank, const int64_t* dims, int channels, const double* img,
                            const uint32_t* labels, double* out);

/* srgb_to_cielab (color.hpp:21-52) for n interleaved RGB pixels in [0, 255]. */
void orc_srgb_to_lab(int64_t n, const double* rgb, double* lab);

/* finalize_cluster_components (connectivity.hpp:125-173): markers (N bytes) in-out. */
void orc_finalize(int rank, const int64_t* dims, const uint32_t* labels, const double* centers,
                  int channels, int64_t k, const int64_t* grid, uint8_t* markers);

/* sweep_relabel (connectivity.hpp:182-261), labels/markers in-out. Returns next label. */
uint32_t orc_sweep(int rank, const int64_t* dims, uint32_t* labels, uint8_t* markers,
                   int64_t min_size, uint32_t k_start);

/* enforce_connectivity (connectivity.hpp:265-273): labels_out = relabelled copy. */
uint32_t orc_enforce_connectivity(int rank, const int64_t* dims, const uint32_t* labels_in,
                                  const double* centers, int channels, int64_t k,
                                  const int64_t* grid, uint32_t* labels_out);

/* Seeded synthetic config volume (planes [z_begin, z_end)), the same bytes
 * as the device generator (synth_ref.c; bench reference arm / cpu_baseline). */
int orc_synth_generate(int config, int rank, const int64_t* dims, int channels, uint64_t seed,
                       int64_t z_begin, int64_t z_end, void* out, int threads);

#ifdef __cplusplus
}
#endif
#endif
