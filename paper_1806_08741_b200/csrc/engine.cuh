// Host-side engine owning the device state of one SLIC run on one slab.
#pragma once

#include <vector>

#include "common.cuh"
#include "kernels_exact.cuh"

namespace sslic_b200 {

enum class AssignPath { kExact = 0, kFast = 1 };
struct FastParams;  // kernels_fast.cuh

class Engine {
 public:
  // img.data: DEVICE pointer to planes [data_begin, data_end) of the last
  // axis (borrowed). force_dist: keep an explicit fp64 DistanceMap.
  Engine(const sslic_image& img, const sslic_params& p, int device, int64_t slab_begin,
         int64_t slab_end, int64_t data_begin, int64_t data_end, cudaStream_t stream,
         bool force_dist = false, int64_t k_override = -1);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // Back to the state after construction (iteration 0, every label
  // undefined, zero sums), so one engine runs several whole runs.
  void reset();
  // K1 on the owned clusters (zeros elsewhere).
  void init(bool perturb);
  // Load a caller-given centre table (host) as the current table.
  void set_centers_host(const double* h);
  // Anchors + candidate bins of the current table.
  void commit();
  // Pipelined start (whole-volume rank-3 fast path, used by run_slic while
  // the image is still arriving in z chunks): pipeline_ok() holds when
  // perturbation cannot move an anchor out of its initial cell (S >= 3 and
  // no 1-plane last cell on every axis), so iteration 0's bins are the
  // identity; init_pipeline() sets them, init_range(z0, z1) perturbs the
  // clusters whose initial centre lies in planes [z0, z1) and publishes
  // their anchors and fp32 split, assign_rows(r0, r1) runs iteration 0's
  // fused assign on region rows [r0, r1). Then update() as usual.
  bool pipeline_ok() const;
  void init_pipeline();
  void init_range(int64_t z0, int64_t z1);
  void assign_rows(int64_t r0, int64_t r1);
  int region_z() const;
  int64_t region_rows() const;
  // One map phase: fused assign + accumulate into partials (zeroed first).
  void assign(bool accumulate = true);
  // Accumulate only (labels as given).
  // reduce_and_update from partials; pushes the new table; residual on device.
  void update();

  double* current_centers() const;
  int64_t centers_count() const { return g_.k * g_.stride; }
  unsigned long long* partials() const { return acc_; }
  int64_t partials_count() const { return g_.k * (g_.stride + 1); }
  uint32_t* label_words() const { return labels_; }
  double* dists() const { return dists_; }
  int64_t slab_voxels() const { return (g_.slab_end - g_.slab_begin) * g_.plane; }
  void unpack_labels(uint32_t* dev_out);
  void copy_centers_to_host(double* h);
  void residuals_to_host(double* h, int n);
  int64_t undefined_count();
  // Tag mode: some assign since construction left a voxel undefined (latched
  // by the fused update; reading it synchronizes).
  bool undefined_seen();
  int64_t out_of_range_count();
  void eval_stats(double* evals, double* window_evals);
  // Fast path: voxels re-decided in fp64, crowded CTAs (last assign).
  void fast_stats(double* ambiguous, double* overflow_blocks, double* changed);
  // Device time (ms) of the i-th assign kernel launch (CUDA events on stream).
  float assign_ms(int i);
  int assign_calls() const { return n_assign_; }
  void set_value_shift(int s) { shift_ = s; }
  // max |value| over this engine's data (float dtypes; the dtype max for
  // u8/u16) and its override with the MAX over ranks (multi-GPU)
  double value_range() const;
  void set_value_range(double absmax);
  int value_shift() const { return shift_; }
  void set_path(AssignPath p) { path_ = p; }
  // The fast fp32-filter kernel applies to this geometry/dtype/mode.
  bool fast_supported() const;
  // Count candidate evaluations and window volumes in assign() (bench).
  void set_collect_stats(bool on) { collect_stats_ = on; }
  AssignPath path() const { return path_; }

  const Geom& geom() const { return g_; }
  int iterations_done() const { return iter_; }
  int max_iterations() const { return max_iter_; }
  bool dist_mode() const { return dist_mode_; }
  LabelCodec codec() const { return codec_; }
  int64_t launches() const { return launches_; }
  cudaStream_t stream() const { return stream_; }
  int device() const { return device_; }

 private:
  void launch_check(const char* what);
  void launch_assign_kernel(bool accumulate);
  FastParams fast_params();
  void launch_exact_kernel(bool accumulate, int64_t nv, const double* hist);
  void compute_shift();
  int fixed_shift(double absmax) const;
  void derive_value_params();

  Geom g_{};
  const void* img_ = nullptr;
  cudaStream_t stream_ = nullptr;
  int device_ = 0;
  int max_iter_ = 0;
  int iter_ = 0;
  int shift_ = 0;
  bool dist_mode_ = false;
  AssignPath path_ = AssignPath::kExact;
  bool collect_stats_ = false;
  LabelCodec codec_{32, 0xffffffffu};

  double* centers_ = nullptr;  // tag mode: (max_iter+1) tables; dist mode: 2 tables
  int n_tables_ = 0;
  uint32_t* labels_ = nullptr;
  double* dists_ = nullptr;
  unsigned long long* acc_ = nullptr;   // this iteration's int64 deltas (allreduced)
  unsigned long long* sums_ = nullptr;  // persistent exact per-cluster sums
  int* anchors_ = nullptr;
  int* cell_of_ = nullptr;
  int* cell_count_ = nullptr;
  int* cell_start_ = nullptr;
  int* cursor_ = nullptr;
  int* items_ = nullptr;
  void* scan_tmp_ = nullptr;
  size_t scan_tmp_bytes_ = 0;
  double* block_partials_ = nullptr;
  double* residuals_ = nullptr;
  unsigned long long* counters_ = nullptr;  // [0] undefined, [1] out-of-range, [2] evals, [3] window
  int64_t launches_ = 0;
  float2* hist32_ = nullptr;  // hi/lo fp32 split of every history table
  int* chg_ = nullptr;        // per cluster: first table index of its current centre
  int* region_cand_ = nullptr;  // fast path: per-region candidate lists
  float key_scale_ = 1.f;       // fast path: 2^-k operand scaling of the fp32 keys
  bool fast_ok_scale_ = true;
  unsigned* update_done_ = nullptr;  // last-block counter of k_update_fused
  int max_cand_ = 0;                  // 0: kFastMaxCand
  float* img32_ = nullptr;            // fast path over an fp64 image: f32 working copy
  double pix_err_ = 0.0;              // bound of its rounding (|v| 2^-24)
  bool acc_zero_ = false;            // deltas already zero (fused update)
  bool words_fresh_ = false;         // every label word is undefined (constructor / reset)
  bool rows_assigned_ = false;       // assign_rows ran since the last reset (pipelined start)
  double vmax_ = 0.0;
  float abs_margin_ = 0.f;
  std::vector<cudaEvent_t> ev_start_, ev_stop_;
  int n_assign_ = 0;
};

}  // namespace sslic_b200
