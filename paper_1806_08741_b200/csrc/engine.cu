// Engine: device state + launch sequence of the SSLIC iteration loop
// (run_slic, slic.hpp:384-415) for one slab on one GPU.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "kernels_fast_main.cuh"

namespace sslic_b200 {

namespace {
template <class T>
T* dalloc(size_t n, cudaStream_t s) {
  void* p = nullptr;
  if (n == 0) n = 1;
  SSLIC_CUDA_CHECK(cudaMallocAsync(&p, n * sizeof(T), s));
  return static_cast<T*>(p);
}
inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

Engine::Engine(const sslic_image& img, const sslic_params& p, int device, int64_t slab_begin,
               int64_t slab_end, int64_t data_begin, int64_t data_end, cudaStream_t stream,
               bool force_dist, int64_t k_override)
    : img_(img.data), stream_(stream), device_(device) {
  SSLIC_CUDA_CHECK(cudaSetDevice(device));
  const int rank = img.rank;
  g_.rank = rank;
  g_.channels = img.channels;
  g_.stride = img.channels + rank;
  g_.dtype = img.dtype;
  int64_t acc = 1;
  g_.k = 1;
  for (int a = 0; a < kMaxRank; ++a) {
    const bool used = a < rank;
    g_.dims[a] = used ? img.dims[a] : 1;
    g_.grid[a] = used ? (int)p.grid[a] : 1;
    g_.cells[a] = (int)((g_.dims[a] + g_.grid[a] - 1) / g_.grid[a]);
    g_.strides[a] = acc;
    acc *= g_.dims[a];
    g_.k *= g_.cells[a];
  }
  g_.ncells = g_.k;
  if (k_override >= 0) g_.k = k_override;
  g_.m_sq = p.weight_m * p.weight_m;
  g_.plane = acc / g_.dims[rank - 1];
  g_.slab_begin = slab_begin;
  g_.slab_end = slab_end;
  g_.data_begin = data_begin;
  g_.data_end = data_end;
  max_iter_ = p.max_iterations > 0 ? p.max_iterations : (rank <= 2 ? 10 : 5);

  // Tag mode needs label ids < 2^label_bits - 1 (so 0xffffffff stays free)
  // and max_iter+1 tags, plus (max_iter+1) history tables in HBM.
  int lb = 1;
  while (((int64_t)1 << lb) - 1 <= g_.k) ++lb;  // label < k <= 2^lb - 2
  const int tag_bits = 32 - lb;
  const double hist_bytes = (double)(max_iter_ + 1) * g_.k * g_.stride * 8.0;
  dist_mode_ = force_dist || tag_bits < 1 || (int64_t)max_iter_ + 1 > ((int64_t)1 << tag_bits) - 1 ||
               hist_bytes > 8e9;
  codec_.label_bits = dist_mode_ ? 32 : lb;
  codec_.label_mask = dist_mode_ ? 0xffffffffu : (uint32_t)(((uint64_t)1 << lb) - 1);

  cudaStream_t s = stream_;
  n_tables_ = dist_mode_ ? 2 : max_iter_ + 1;
  centers_ = dalloc<double>((size_t)n_tables_ * g_.k * g_.stride, s);
  const int64_t nv = slab_voxels();
  labels_ = dalloc<uint32_t>(nv, s);
  SSLIC_CUDA_CHECK(cudaMemsetAsync(labels_, 0xff, nv * sizeof(uint32_t), s));
  words_fresh_ = true;
  rows_assigned_ = false;
  if (dist_mode_) {
    dists_ = dalloc<double>(nv, s);  // filled with +inf below (DistanceMap, image.hpp:323)
  } else {
    hist32_ = dalloc<float2>((size_t)n_tables_ * g_.k * hist32_stride(g_.stride), s);
    chg_ = dalloc<int>(g_.k, s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(chg_, 0, g_.k * sizeof(int), s));
  }
  acc_ = dalloc<unsigned long long>(partials_count(), s);
  sums_ = dalloc<unsigned long long>(partials_count(), s);
  SSLIC_CUDA_CHECK(cudaMemsetAsync(sums_, 0, partials_count() * sizeof(unsigned long long), s));
  anchors_ = dalloc<int>(g_.k * kMaxRank, s);
  cell_of_ = dalloc<int>(g_.k, s);
  cell_count_ = dalloc<int>(g_.ncells + 1, s);
  cell_start_ = dalloc<int>(g_.ncells + 1, s);
  cursor_ = dalloc<int>(g_.ncells, s);
  items_ = dalloc<int>(g_.k, s);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp_bytes_, cell_count_, cell_start_,
                                (int)(g_.ncells + 1), s);
  scan_tmp_ = dalloc<char>(scan_tmp_bytes_, s);
  block_partials_ = dalloc<double>(blocks_for(g_.k, 256), s);
  residuals_ = dalloc<double>(max_iter_, s);
  counters_ = dalloc<unsigned long long>(8, s);
  SSLIC_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 8 * sizeof(unsigned long long), s));
  update_done_ = dalloc<unsigned>(2, s);  // [0] last-block counter, [1] undefined latch
  SSLIC_CUDA_CHECK(cudaMemsetAsync(update_done_, 0, 2 * sizeof(unsigned), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(acc_, 0, partials_count() * sizeof(unsigned long long), s));
  acc_zero_ = true;
  if (dist_mode_) {
    k_fill_f64<<<blocks_for(nv, 256), 256, 0, s>>>(dists_, nv, __builtin_huge_val());
    launch_check("fill dists");
  }
  compute_shift();
  derive_value_params();
  path_ = fast_path_supported(g_) && !dist_mode_ && fast_ok_scale_ ? AssignPath::kFast
                                                                    : AssignPath::kExact;
  if (path_ == AssignPath::kFast)
    region_cand_ = dalloc<int>((size_t)fast_region_count(g_) * kRegionCandStride, s);
  // test hook: SSLIC_FAST_MAX_CAND lowers the candidate capacity of a region
  // (more regions take the exact crowded fallback)
  if (const char* mc = std::getenv("SSLIC_FAST_MAX_CAND")) max_cand_ = std::atoi(mc);
  if (path_ == AssignPath::kFast && g_.dtype == SSLIC_F64) {
    // f32 working copy of an fp64 image for the fast sweep (round to nearest;
    // the rounding is in the fast margins)
    const int64_t nvals = (g_.data_end - g_.data_begin) * g_.plane * g_.channels;
    img32_ = dalloc<float>((size_t)nvals, s);
    k_f64_to_f32<<<blocks_for(nvals, 256), 256, 0, s>>>(static_cast<const double*>(img_), img32_,
                                                        nvals);
    launch_check("f64 working copy");
  }
}

Engine::~Engine() {
  cudaSetDevice(device_);
  cudaStream_t s = stream_;
  void* ptrs[] = {centers_, labels_, dists_, acc_, anchors_, cell_of_, cell_count_,
                  cell_start_, cursor_, items_, scan_tmp_, block_partials_, residuals_,
                  counters_, hist32_, chg_, sums_, region_cand_, update_done_, img32_};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  for (cudaEvent_t e : ev_start_) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_stop_) cudaEventDestroy(e);
}

bool Engine::fast_supported() const {
  return fast_path_supported(g_) && !dist_mode_ && fast_ok_scale_ && region_cand_ != nullptr;
}

void Engine::launch_check(const char* what) {
  ++launches_;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(SSLIC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void Engine::compute_shift() {
  if (g_.dtype == SSLIC_U8 || g_.dtype == SSLIC_U16) {
    shift_ = 0;
    return;
  }
  const int64_t nvals = (g_.data_end - g_.data_begin) * g_.plane * g_.channels;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(counters_ + 4, 0, sizeof(unsigned long long), stream_));
  k_absmax<<<148 * 4, 256, 0, stream_>>>(img_, g_.dtype, nvals, counters_ + 4);
  launch_check("absmax");
  unsigned long long bits = 0;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&bits, counters_ + 4, sizeof(bits), cudaMemcpyDeviceToHost,
                                   stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  double m;
  std::memcpy(&m, &bits, sizeof(m));
  shift_ = fixed_shift(m);
  vmax_ = m;
}

// Fixed-point scale 2^shift of float intensities. Each |v| 2^shift stays
// below 2^(40 - h), where 2^h bounds a cluster's population (its window,
// prod_a min(2 S_a + 1, dims_a): a voxel only joins a cluster whose window
// covers it), so every per-cluster int64 sum and delta stays below 2^40 x
// population <= 2^62 (grid = extent on an 8M-voxel float image
// used to wrap). h = 0 up to 2^22 members (every fast-path geometry).
int Engine::fixed_shift(double m) const {
  int e = 0;
  if (m > 0.0) std::frexp(m, &e);  // m < 2^e
  double pop = 1.0;
  for (int a = 0; a < g_.rank; ++a)
    pop *= (double)std::min<int64_t>(2 * g_.grid[a] + 1, g_.dims[a]);
  int h = 0;
  while (std::ldexp(1.0, 22 + h) < pop) ++h;
  return 40 - h - e;
}

// Parameters derived from the value range: the fixed-point shift of float
// intensities, the fp32 filter's absolute margin and key scale.
void Engine::derive_value_params() {
  if (g_.dtype == SSLIC_U8) vmax_ = 255.0;
  if (g_.dtype == SSLIC_U16) vmax_ = 65535.0;
  {
    // absolute fp32 margin for the hi/lo centre split (DESIGN.md error bound)
    const double e = vmax_ * std::ldexp(1.0, -48);
    const double M = fast_margin(g_.channels);
    double am = 8.0 * e * e / M + e * e + 1e-37;
    if (g_.dtype == SSLIC_F64) {
      // rounding of the f32 working copy (kernels_fast_main.cuh, fast margin)
      const double ep = vmax_ * std::ldexp(1.0, -24);
      const double eps0 = (g_.channels + 14) * std::ldexp(1.0, -24);
      am += g_.channels * (1.0 / eps0 + 1.0) * ep * ep;
      pix_err_ = ep;
    }
    abs_margin_ = (float)am;
    // key scale 2^-k: the largest possible fp32 distance of a covered
    // candidate, C (2 vmax + 1)^2 + m^2 rank 4, must map below 2^-67
    // (kernels_fast.cuh "Keys"). Exact power-of-two scaling.
    const double dmax = g_.channels * (2.0 * vmax_ + 1.0) * (2.0 * vmax_ + 1.0) +
                        g_.m_sq * g_.rank * 4.0 + 1.0;
    const int k = (int)std::ceil((std::log2(dmax) + 67.0) / 2.0);
    key_scale_ = (float)std::ldexp(1.0, -k);
    if (!(k < 120)) fast_ok_scale_ = false;  // absurd ranges: keep the exact path
  }
}

double Engine::value_range() const { return vmax_; }

// Multi-GPU: every rank must use the same value range (the fixed-point
// shift of the summed deltas, and the filter margins of centres built from
// every rank's voxels), i.e. the MAX over ranks of value_range().
void Engine::set_value_range(double m) {
  if (g_.dtype == SSLIC_U8 || g_.dtype == SSLIC_U16) return;  // fixed: dtype max, shift 0
  if (!(m >= 0.0)) throw Error(SSLIC_EINVAL, "engine: value range must be >= 0");
  shift_ = fixed_shift(m);
  vmax_ = m;
  derive_value_params();
  if (!fast_ok_scale_) path_ = AssignPath::kExact;
}

double* Engine::current_centers() const {
  const int slot = dist_mode_ ? (iter_ & 1) : iter_;
  return centers_ + (size_t)slot * g_.k * g_.stride;
}

void Engine::reset() {
  cudaStream_t s = stream_;
  const int64_t nv = slab_voxels();
  iter_ = 0;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(labels_, 0xff, nv * sizeof(uint32_t), s));
  words_fresh_ = true;
  rows_assigned_ = false;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(sums_, 0, partials_count() * sizeof(unsigned long long), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(acc_, 0, partials_count() * sizeof(unsigned long long), s));
  acc_zero_ = true;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 8 * sizeof(unsigned long long), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(update_done_, 0, 2 * sizeof(unsigned), s));
  if (chg_) SSLIC_CUDA_CHECK(cudaMemsetAsync(chg_, 0, g_.k * sizeof(int), s));
  if (dist_mode_) {
    k_fill_f64<<<blocks_for(nv, 256), 256, 0, s>>>(dists_, nv, __builtin_huge_val());
    launch_check("fill dists");
  }
}

void Engine::init(bool perturb) {
  k_init_perturb<<<blocks_for(g_.k, 128), 128, 0, stream_>>>(g_, img_, current_centers(),
                                                             perturb ? 1 : 0);
  launch_check("init_perturb");
}

void Engine::set_centers_host(const double* h) {
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(current_centers(), h, centers_count() * sizeof(double),
                                   cudaMemcpyHostToDevice, stream_));
}

void Engine::commit() {
  cudaStream_t s = stream_;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cell_count_, 0, (g_.ncells + 1) * sizeof(int), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cursor_, 0, g_.ncells * sizeof(int), s));
  k_anchors<<<blocks_for(g_.k, 256), 256, 0, s>>>(g_, current_centers(), anchors_, cell_of_,
                                                  cell_count_);
  launch_check("anchors");
  SSLIC_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_tmp_, scan_tmp_bytes_, cell_count_,
                                                 cell_start_, (int)(g_.ncells + 1), s));
  ++launches_;
  k_bin_fill<<<blocks_for(g_.k, 256), 256, 0, s>>>(g_.k, cell_of_, cell_start_, cursor_, items_);
  launch_check("bin_fill");
  k_bin_sort_reset<<<blocks_for(g_.ncells + 1, 256), 256, 0, s>>>(g_.ncells, cell_start_, items_,
                                                                  cell_count_, cursor_);
  launch_check("bin_sort");
  if (!dist_mode_) {
    const int s2 = hist32_stride(g_.stride);
    k_split32<<<blocks_for(g_.k * s2, 256), 256, 0, s>>>(
        current_centers(), hist32_ + (size_t)iter_ * g_.k * s2, g_.k, g_.stride);
    launch_check("split32");
  }
}

bool Engine::pipeline_ok() const {
  if (g_.rank != 3 || dist_mode_ || path_ != AssignPath::kFast || g_.k != g_.ncells) return false;
  if (g_.slab_begin != 0 || g_.slab_end != g_.dims[2] || g_.data_begin != 0) return false;
  if (g_.dtype != SSLIC_U8 && g_.dtype != SSLIC_U16) return false;  // no image-wide pre-pass
  for (int a = 0; a < g_.rank; ++a)
    if (g_.grid[a] < 3 || g_.dims[a] % g_.grid[a] == 1) return false;
  return true;
}

int Engine::region_z() const {
  int R[3];
  region_extents(g_, R);
  return R[2];
}

int64_t Engine::region_rows() const { return (g_.dims[2] + region_z() - 1) / region_z(); }

void Engine::init_pipeline() {
  if (!pipeline_ok()) throw Error(SSLIC_EINVAL, "engine: pipelined start not applicable");
  k_identity_bins<<<blocks_for(g_.ncells + 1, 256), 256, 0, stream_>>>(g_.ncells, cell_start_,
                                                                       items_);
  launch_check("identity_bins");
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cell_count_, 0, (g_.ncells + 1) * sizeof(int), stream_));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cursor_, 0, g_.ncells * sizeof(int), stream_));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 8 * sizeof(unsigned long long), stream_));
  if (!acc_zero_)
    SSLIC_CUDA_CHECK(
        cudaMemsetAsync(acc_, 0, partials_count() * sizeof(unsigned long long), stream_));
  acc_zero_ = false;
}

void Engine::init_range(int64_t z0, int64_t z1) {
  if (z1 <= z0) return;
  k_init_perturb<<<blocks_for(g_.k, 128), 128, 0, stream_>>>(g_, img_, current_centers(), 1, z0,
                                                             z1);
  launch_check("init_perturb(range)");
  const int s2 = hist32_stride(g_.stride);
  k_anchors_split_range<<<blocks_for(g_.k, 256), 256, 0, stream_>>>(
      g_, current_centers(), anchors_, hist32_ + (size_t)iter_ * g_.k * s2, s2, z0, z1);
  launch_check("anchors_split(range)");
}

void Engine::assign_rows(int64_t r0, int64_t r1) {
  if (r1 <= r0) return;
  // (each region row is assigned once per iteration, so the rows of
  // iteration 0 still hold undefined words: the first-iteration kernel applies)
  launch_fast_assign(fast_params(), stream_, r0, r1);
  rows_assigned_ = true;
  ++launches_;
  launch_check("assign_fast(rows)");
}

void Engine::assign(bool accumulate) {
  if (!dist_mode_ && iter_ >= max_iter_)
    throw Error(SSLIC_EINVAL, "engine: iteration budget exhausted (history tables)");
  cudaStream_t s = stream_;
  // the fused update leaves the deltas zeroed; otherwise clear them here
  if (accumulate && !acc_zero_)
    SSLIC_CUDA_CHECK(cudaMemsetAsync(acc_, 0, partials_count() * sizeof(unsigned long long), s));
  if (accumulate) acc_zero_ = false;
  SSLIC_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 8 * sizeof(unsigned long long), s));
  const int64_t nv = slab_voxels();
  const double* hist = dist_mode_ ? nullptr : centers_;
  if (collect_stats_) {
    k_window_volume<<<blocks_for(g_.k, 256), 256, 0, s>>>(g_, anchors_, counters_ + 3);
    launch_check("window_volume");
  }
  // Device-side timing of the assign kernel alone (bench roofline).
  if ((int)ev_start_.size() <= n_assign_) {
    cudaEvent_t a, b;
    SSLIC_CUDA_CHECK(cudaEventCreate(&a));
    SSLIC_CUDA_CHECK(cudaEventCreate(&b));
    ev_start_.push_back(a);
    ev_stop_.push_back(b);
  }
  // inside a graph capture the timing events must be external record nodes
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  SSLIC_CUDA_CHECK(cudaStreamIsCapturing(s, &cap));
  const unsigned rf = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
  SSLIC_CUDA_CHECK(cudaEventRecordWithFlags(ev_start_[n_assign_], s, rf));
  launch_assign_kernel(accumulate);
  SSLIC_CUDA_CHECK(cudaEventRecordWithFlags(ev_stop_[n_assign_], s, rf));
  ++n_assign_;
}

void Engine::launch_assign_kernel(bool accumulate) {
  cudaStream_t s = stream_;
  const int64_t nv = slab_voxels();
  const double* hist = dist_mode_ ? nullptr : centers_;
  if (path_ == AssignPath::kFast && accumulate && !dist_mode_) {
    FastParams P = fast_params();
    if (rows_assigned_) P.first = 0;  // some rows may already hold labels
    launch_fast_assign(P, s);
    words_fresh_ = false;
    ++launches_;  // k_region_cand + k_assign_fast
    launch_check("assign_fast");
    return;
  }
  words_fresh_ = false;
  launch_exact_kernel(accumulate, nv, hist);
}

FastParams Engine::fast_params() {
    const double* hist = dist_mode_ ? nullptr : centers_;
    FastParams P{};
    P.g = g_;
    P.img = img32_ ? static_cast<const void*>(img32_) : img_;
    P.img_exact = img_;
    P.pix_err = (float)(pix_err_ * key_scale_);
    P.centers = current_centers();
    P.history = hist;
    P.hist32 = hist32_;
    P.chg = chg_;
    P.anchors = anchors_;
    P.cell_start = cell_start_;
    P.items = items_;
    P.labels = labels_;
    P.codec = codec_;
    P.tag_now = (uint32_t)iter_;
    P.shift = shift_;
    P.acc = acc_;
    P.counters = counters_;
    P.eval_count = collect_stats_ ? counters_ + 2 : nullptr;
    P.abs_margin = abs_margin_;
    P.cur32 = hist32_ + (size_t)iter_ * g_.k * hist32_stride(g_.stride);
    P.key_scale = key_scale_;
    P.key_scale2 = key_scale_ * key_scale_;
    P.abs_margin = abs_margin_ * P.key_scale2;
    P.region_cand = region_cand_;
    P.max_cand = max_cand_;
    P.vmax = (float)vmax_;
    P.first = words_fresh_ && iter_ == 0 ? 1 : 0;
    return P;
}

void Engine::launch_exact_kernel(bool accumulate, int64_t nv, const double* hist) {
  cudaStream_t s = stream_;
  const unsigned nb = blocks_for(nv, 256);
  if (dist_mode_) {
    if (accumulate)
      k_assign_exact<true, true><<<nb, 256, 0, s>>>(g_, img_, current_centers(), hist, anchors_,
                                                    cell_start_, items_, labels_, dists_, codec_,
                                                    (uint32_t)iter_, shift_, acc_, counters_,
                                                    collect_stats_ ? counters_ + 2 : nullptr);
    else
      k_assign_exact<true, false><<<nb, 256, 0, s>>>(g_, img_, current_centers(), hist, anchors_,
                                                     cell_start_, items_, labels_, dists_, codec_,
                                                     (uint32_t)iter_, shift_, acc_, counters_,
                                                     collect_stats_ ? counters_ + 2 : nullptr);
  } else {
    if (accumulate)
      k_assign_exact<false, true><<<nb, 256, 0, s>>>(g_, img_, current_centers(), hist, anchors_,
                                                     cell_start_, items_, labels_, dists_, codec_,
                                                     (uint32_t)iter_, shift_, acc_, counters_,
                                                     collect_stats_ ? counters_ + 2 : nullptr);
    else
      k_assign_exact<false, false><<<nb, 256, 0, s>>>(g_, img_, current_centers(), hist,
                                                      anchors_, cell_start_, items_, labels_,
                                                      dists_, codec_, (uint32_t)iter_, shift_,
                                                      acc_, counters_,
                                                      collect_stats_ ? counters_ + 2 : nullptr);
  }
  launch_check("assign_exact");
}

void Engine::update() {
  if (iter_ >= max_iter_) throw Error(SSLIC_EINVAL, "engine: all iterations already done");
  cudaStream_t s = stream_;
  double* old_c = current_centers();
  const int next_slot = dist_mode_ ? ((iter_ + 1) & 1) : iter_ + 1;
  double* new_c = centers_ + (size_t)next_slot * g_.k * g_.stride;
  const unsigned nb = blocks_for(g_.k, 256);
  if (!dist_mode_) {
    // one fused launch (update + residual + hi/lo split + anchors/cell
    // counts), then the bins: scan, fill, sort (+ counter reset)
    const int s2 = hist32_stride(g_.stride);
    k_update_fused<<<nb, 256, 0, s>>>(g_, shift_, acc_, sums_, old_c, new_c, block_partials_,
                                      chg_, iter_ + 1, hist32_ + (size_t)(iter_ + 1) * g_.k * s2,
                                      s2, anchors_, cell_of_, cell_count_, update_done_,
                                      residuals_ + iter_, counters_, update_done_ + 1);
    launch_check("update_fused");
    acc_zero_ = true;
    ++iter_;
    SSLIC_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(scan_tmp_, scan_tmp_bytes_, cell_count_,
                                                   cell_start_, (int)(g_.ncells + 1), s));
    ++launches_;
    k_bin_fill<<<blocks_for(g_.k, 256), 256, 0, s>>>(g_.k, cell_of_, cell_start_, cursor_,
                                                     items_);
    launch_check("bin_fill");
    k_bin_sort_reset<<<blocks_for(g_.ncells + 1, 256), 256, 0, s>>>(
        g_.ncells, cell_start_, items_, cell_count_, cursor_);
    launch_check("bin_sort");
    return;
  }
  k_update<<<nb, 256, 0, s>>>(g_, shift_, acc_, sums_, old_c, new_c, block_partials_, chg_,
                              iter_ + 1);
  launch_check("update");
  k_residual_final<<<1, 1024, 0, s>>>(block_partials_, (int)nb, residuals_ + iter_);
  launch_check("residual");
  ++iter_;
  commit();
}

void Engine::unpack_labels(uint32_t* dev_out) {
  const int64_t nv = slab_voxels();
  k_unpack_labels<<<blocks_for(nv, 256), 256, 0, stream_>>>(nv, labels_, codec_, dev_out);
  launch_check("unpack_labels");
}

void Engine::copy_centers_to_host(double* h) {
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(h, current_centers(), centers_count() * sizeof(double),
                                   cudaMemcpyDeviceToHost, stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

void Engine::residuals_to_host(double* h, int n) {
  if (n <= 0) return;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(h, residuals_, n * sizeof(double), cudaMemcpyDeviceToHost,
                                   stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

bool Engine::undefined_seen() {
  unsigned v = 0;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&v, update_done_ + 1, sizeof(v), cudaMemcpyDeviceToHost,
                                   stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return v != 0;
}

int64_t Engine::undefined_count() {
  unsigned long long v = 0;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&v, counters_, sizeof(v), cudaMemcpyDeviceToHost, stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return (int64_t)v;
}

int64_t Engine::out_of_range_count() {
  unsigned long long v = 0;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&v, counters_ + 1, sizeof(v), cudaMemcpyDeviceToHost, stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  return (int64_t)v;
}

float Engine::assign_ms(int i) {
  if (i < 0 || i >= n_assign_) throw Error(SSLIC_EINVAL, "assign_ms: no such assign call");
  SSLIC_CUDA_CHECK(cudaEventSynchronize(ev_stop_[i]));
  float ms = 0.f;
  SSLIC_CUDA_CHECK(cudaEventElapsedTime(&ms, ev_start_[i], ev_stop_[i]));
  return ms;
}

void Engine::fast_stats(double* ambiguous, double* overflow_blocks, double* changed) {
  unsigned long long v[3] = {0, 0, 0};
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(v, counters_ + 5, sizeof(v), cudaMemcpyDeviceToHost, stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  *ambiguous = (double)v[0];
  *overflow_blocks = (double)v[1];
  if (changed) *changed = (double)v[2];
}

void Engine::eval_stats(double* evals, double* window_evals) {
  unsigned long long v[2] = {0, 0};
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(v, counters_ + 2, sizeof(v), cudaMemcpyDeviceToHost, stream_));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(stream_));
  *evals = (double)v[0];
  *window_evals = (double)v[1];
}

}  // namespace sslic_b200
