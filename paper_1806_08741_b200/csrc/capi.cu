// C ABI (include/sslic_b200.h) over the Engine. Host entry points copy host
// buffers to the device, run the CUDA path and copy results back; every
// failure is reported as a status code mirroring the reference's exception
// classes, with the message in sslic_last_error().
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <new>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.cuh"
#include "color.cuh"
#include "connectivity.cuh"
#include "engine.cuh"

using namespace sslic_b200;

namespace sslic_b200 {
std::string& last_error() {
  thread_local std::string msg;
  return msg;
}
}  // namespace sslic_b200

namespace {

size_t dtype_size(int dt) {
  switch (dt) {
    case SSLIC_U8: return 1;
    case SSLIC_U16: return 2;
    case SSLIC_F32: return 4;
    case SSLIC_F64: return 8;
    default: return 0;
  }
}

int64_t pixel_count(const sslic_image& img) {
  int64_t n = 1;
  for (int a = 0; a < img.rank; ++a) n *= img.dims[a];
  return n;
}

// NDImage constructor checks (image.hpp:238-249).
void validate_image(const sslic_image* img) {
  if (!img) throw Error(SSLIC_EINVAL, "image: null descriptor");
  if (img->rank < 1 || img->rank > kMaxRank)
    throw Error(SSLIC_EINVAL, "NDImage: rank must be in [1, 4]");
  for (int a = 0; a < img->rank; ++a)
    if (img->dims[a] < 1) throw Error(SSLIC_EINVAL, "NDImage: extents must be positive");
  if (img->channels < 1) throw Error(SSLIC_EINVAL, "NDImage: channels must be >= 1");
  if (dtype_size(img->dtype) == 0) throw Error(SSLIC_EINVAL, "image: unknown dtype");
  if (!img->data) throw Error(SSLIC_EINVAL, "image: null data");
}

// SlicParams::validate (slic.hpp:52-64).
void validate_params(const sslic_params* p, const sslic_image* img) {
  if (!p) throw Error(SSLIC_EINVAL, "SlicParams: null");
  for (int a = 0; a < img->rank; ++a) {
    if (p->grid[a] < 1) throw Error(SSLIC_EINVAL, "SlicParams: grid sizes must be >= 1");
    if (p->grid[a] > img->dims[a])
      throw Error(SSLIC_EINVAL,
                  "SlicParams: grid size exceeds image extent on axis " + std::to_string(a));
  }
  if (!(p->weight_m > 0.0)) throw Error(SSLIC_EINVAL, "SlicParams: weight_m must be positive");
  if (p->max_iterations < 0)
    throw Error(SSLIC_EINVAL, "SlicParams: max_iterations must be positive (or 0 for default)");
}

struct DeviceBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DeviceBuf(size_t bytes, cudaStream_t st) : s(st) {
    SSLIC_CUDA_CHECK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
  }
  ~DeviceBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Keep freed device memory in the stream-ordered pool across calls (the
// default release threshold returns it to the driver at every sync, so each
// whole-run call would re-map gigabytes).
}  // namespace
namespace sslic_b200 {
void keep_pool_memory(int device) {
  static bool done[64] = {};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  done[device] = true;
}
}  // namespace sslic_b200
namespace {

struct Stream {
  cudaStream_t s = nullptr;
  explicit Stream(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(SSLIC_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= n) throw Error(SSLIC_EINVAL, "device index out of range");
    SSLIC_CUDA_CHECK(cudaSetDevice(device));
    keep_pool_memory(device);
    SSLIC_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~Stream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
  void sync() { SSLIC_CUDA_CHECK(cudaStreamSynchronize(s)); }
};

__global__ void k_count_nonfinite(const void* data, int dtype, int64_t n, unsigned long long* out) {
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad += isfinite(load_value(data, dtype, i)) ? 0 : 1;
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, bad);
}

// Uploads a host image; checks finiteness like the NDImage constructor.
// SSLIC_TIMING=1: per-phase wall times of the whole-run entry points (stderr).
struct PhaseTimer {
  const char* what;
  bool on;
  std::chrono::steady_clock::time_point t0;
  std::string line;
  explicit PhaseTimer(const char* w) : what(w), on(std::getenv("SSLIC_TIMING") != nullptr) {
    t0 = std::chrono::steady_clock::now();
  }
  void mark(Stream& st, const char* phase) {
    if (!on) return;
    st.sync();
    const auto t = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s %.1f ms", phase,
                  std::chrono::duration<double, std::milli>(t - t0).count());
    line += buf;
    t0 = t;
  }
  ~PhaseTimer() {
    if (on) std::fprintf(stderr, "[sslic] %s:%s\n", what, line.c_str());
  }
};

// fp64 images are the reference's storage (NDImage holds doubles,
// image.hpp:236-285) whatever the data really is. When every value is a
// uint8 / uint16 / float32 number the volume is narrowed to that type ON THE
// DEVICE, losslessly, and takes the native-dtype kernels: flags[0] non-finite
// values, [1] not uint8, [2] not uint16, [3] not float32.
__global__ void k_narrow_probe(const double* v, int64_t n, unsigned* flags) {
  unsigned f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = v[i];
    const bool integral = x == trunc(x);
    f |= isfinite(x) ? 0u : 1u;
    f |= (integral && x >= 0.0 && x <= 255.0) ? 0u : 2u;
    f |= (integral && x >= 0.0 && x <= 65535.0) ? 0u : 4u;
    f |= ((double)(float)x == x) ? 0u : 8u;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) {
    if (f & 1u) atomicOr(flags, 1u);
    if (f & 2u) atomicOr(flags + 1, 1u);
    if (f & 4u) atomicOr(flags + 2, 1u);
    if (f & 8u) atomicOr(flags + 3, 1u);
  }
}
template <typename T>
__global__ void k_narrow_convert(const double* v, int64_t n, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)v[i];
}

// narrowed_dtype (optional): fp64 input may come back as a uint8 / uint16 /
// float32 device image (see k_narrow_probe); *narrowed_dtype is its type.
std::unique_ptr<DeviceBuf> upload_image(const sslic_image* img, Stream& st,
                                        int* narrowed_dtype = nullptr) {
  const int64_t nvals = pixel_count(*img) * img->channels;
  const size_t bytes = (size_t)nvals * dtype_size(img->dtype);
  auto buf = std::make_unique<DeviceBuf>(bytes, st.s);
  int dev = 0;
  SSLIC_CUDA_CHECK(cudaGetDevice(&dev));
  copy_to_device(buf->p, img->data, bytes, dev, st.s);  // (pageable callers: striped)
  if (narrowed_dtype) *narrowed_dtype = img->dtype;
  if (narrowed_dtype && img->dtype == SSLIC_F64 && std::getenv("SSLIC_NO_NARROW") == nullptr) {
    DeviceBuf flags(4 * sizeof(unsigned), st.s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(flags.p, 0, 4 * sizeof(unsigned), st.s));
    k_narrow_probe<<<148 * 8, 256, 0, st.s>>>(buf->as<double>(), nvals, flags.as<unsigned>());
    SSLIC_CUDA_CHECK(cudaGetLastError());
    unsigned f[4] = {0, 0, 0, 0};
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(f, flags.p, sizeof f, cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (f[0]) throw Error(SSLIC_EINVAL, "NDImage: non-finite value");
    const int dt = !f[1] ? SSLIC_U8 : !f[2] ? SSLIC_U16 : !f[3] ? SSLIC_F32 : SSLIC_F64;
    if (dt == SSLIC_F64) return buf;  // genuinely fp64 data (checked finite above)
    auto out = std::make_unique<DeviceBuf>((size_t)nvals * dtype_size(dt), st.s);
    if (dt == SSLIC_U8)
      k_narrow_convert<uint8_t><<<148 * 8, 256, 0, st.s>>>(buf->as<double>(), nvals,
                                                          out->as<uint8_t>());
    else if (dt == SSLIC_U16)
      k_narrow_convert<uint16_t><<<148 * 8, 256, 0, st.s>>>(buf->as<double>(), nvals,
                                                           out->as<uint16_t>());
    else
      k_narrow_convert<float><<<148 * 8, 256, 0, st.s>>>(buf->as<double>(), nvals,
                                                        out->as<float>());
    SSLIC_CUDA_CHECK(cudaGetLastError());
    *narrowed_dtype = dt;
    return out;  // (the fp64 copy is released in stream order)
  }
  if (img->dtype == SSLIC_F32 || img->dtype == SSLIC_F64) {
    DeviceBuf cnt(sizeof(unsigned long long), st.s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st.s));
    k_count_nonfinite<<<148 * 4, 256, 0, st.s>>>(buf->p, img->dtype, nvals,
                                                 cnt.as<unsigned long long>());
    SSLIC_CUDA_CHECK(cudaGetLastError());
    unsigned long long bad = 0;
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(&bad, cnt.p, sizeof(bad), cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (bad) throw Error(SSLIC_EINVAL, "NDImage: non-finite value");
  }
  return buf;
}

sslic_image device_view(const sslic_image* img, const void* dev) {
  sslic_image v = *img;
  v.data = dev;
  for (int a = img->rank; a < kMaxRank; ++a) v.dims[a] = 1;
  return v;
}

sslic_params default_params_for(const sslic_image* img, const int64_t* grid, double m) {
  sslic_params p{};
  for (int a = 0; a < kMaxRank; ++a) p.grid[a] = a < img->rank ? grid[a] : 1;
  p.weight_m = m;
  return p;
}

// The run_slic loop over a whole-image engine. Returns iterations done.
// Writes the labels that changed since the snapshot straight into the
// (pinned, device-mapped) host map.
__global__ void k_patch_labels_host(int64_t n, const uint32_t* before, const uint32_t* after,
                                    uint32_t* host) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = after[i];
    if (v != before[i]) host[i] = v;
  }
}

// run_slic's loop for a pinned host label map: the labels after iteration
// iters-4 are unpacked into a snapshot whose download (PCIe) overlaps the last
// iterations on a second stream; afterwards the voxels whose label changed
// since (~0.1-1 %) are written straight into the mapped host map. Same result
// as downloading the final map.
// Labels that differ between the snapshot and the final map, as (index,
// label) pairs written through a mapped pinned staging buffer (coalesced
// 8-byte stores; PCIe handles these far better than scattered 4-byte
// writes into the caller's map). Each block walks 4096-label tiles and
// reserves its tile's entries with one atomic; entries past `cap` are
// counted but not written (the caller then copies the whole map).
// (amask != ~0: `after` holds engine label words, decoded like
// LabelCodec::label -- the final map needs no separate unpack pass)
__global__ void k_change_list(int64_t n, const uint32_t* before, const uint32_t* after,
                              unsigned long long* count, int64_t cap, uint2* out,
                              uint32_t idx0 = 0, uint32_t amask = 0xffffffffu) {
  constexpr int kPer = 16;
  __shared__ unsigned long long base;
  __shared__ int warp_tot[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t tile = blockIdx.x * (int64_t)(256 * kPer); tile < n;
       tile += (int64_t)gridDim.x * 256 * kPer) {
    uint32_t chg = 0;
    uint32_t val[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t i = tile + j * 256 + tid;
      val[j] = 0;
      if (i < n) {
        const uint32_t w = after[i];
        const uint32_t a = w == 0xffffffffu ? w : (w & amask);
        val[j] = a;
        if (a != before[i]) chg |= 1u << j;
      }
    }
    const int mine = __popc(chg);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int before_w = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      before_w += w < warp ? warp_tot[w] : 0;
      tot += warp_tot[w];
    }
    if (tid == 0) base = tot ? atomicAdd(count, (unsigned long long)tot) : 0ull;
    __syncthreads();
    int64_t pos = (int64_t)base + before_w + incl - mine;
#pragma unroll
    for (int j = 0; j < kPer; ++j)
      if (chg >> j & 1u) {
        if (pos < cap) out[pos] = make_uint2(idx0 + (uint32_t)(tile + j * 256 + tid), val[j]);
        ++pos;
      }
    __syncthreads();  // warp_tot / base reuse
  }
}

// The per-piece list counts into mapped host memory (read by the host as
// soon as the lists are built, without queueing behind the snapshot DMA).
__global__ void k_copy_counts(const unsigned long long* cnt, int k, unsigned long long* host_cnt) {
  if ((int)threadIdx.x < k) host_cnt[threadIdx.x] = cnt[threadIdx.x];
}

// Page-locked, device-mapped host staging kept across calls (grown on demand).
struct MappedStage {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t want) {
    if (want > bytes) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      bytes = 0;
      SSLIC_CUDA_CHECK(cudaHostAlloc(&p, want, cudaHostAllocMapped | cudaHostAllocPortable));
      bytes = want;
    }
    return p;
  }
};
MappedStage& mapped_stage() {
  static MappedStage* s = new MappedStage();  // never destroyed (exit-order safe)
  return *s;
}


// Host threads applying per-chunk change lists as the chunks become ready
// (the main thread calls ready(c) once chunk c's snapshot copy and list have
// landed); chunks touch disjoint label ranges, so they may overlap.
struct ChunkApplier {
  uint32_t* labels;
  std::vector<const uint2*> lists;
  std::vector<int64_t> counts;
  std::atomic<int> n_ready{0};
  std::atomic<bool> cancel{false};
  std::vector<std::thread> th;
  ChunkApplier(uint32_t* l, int chunks) : labels(l), lists(chunks), counts(chunks, 0) {}
  // an exception between start() and join() must not leave joinable threads
  ~ChunkApplier() {
    cancel.store(true, std::memory_order_release);
    join();
  }
  void start() {
    int t = (int)std::thread::hardware_concurrency();
    t = t < 1 ? 1 : (t > 32 ? 32 : t);
    const int K = (int)lists.size();
    for (int w = 0; w < t; ++w)
      th.emplace_back([this, w, t, K] {
        for (int c = 0; c < K; ++c) {
          while (n_ready.load(std::memory_order_acquire) <= c) {
            if (cancel.load(std::memory_order_acquire)) return;
            std::this_thread::yield();
          }
          const uint2* list = lists[c];
          const int64_t cnt = counts[c], a = cnt * w / t, b = cnt * (w + 1) / t;
          for (int64_t i = a; i < b; ++i) {
            if (i + 32 < b) __builtin_prefetch(labels + list[i + 32].x, 1, 0);
            labels[list[i].x] = list[i].y;
          }
        }
      });
  }
  void ready(int c) { n_ready.store(c + 1, std::memory_order_release); }
  void join() {
    for (auto& x : th) x.join();
    th.clear();
  }
};

// Owned non-blocking stream / timing-free event (released on every exit path).
struct OwnedStream {
  cudaStream_t s = nullptr;
  OwnedStream() { SSLIC_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~OwnedStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
  OwnedStream(const OwnedStream&) = delete;
  OwnedStream& operator=(const OwnedStream&) = delete;
};
struct OwnedEvent {
  cudaEvent_t e = nullptr;
  OwnedEvent() { SSLIC_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~OwnedEvent() {
    if (e) cudaEventDestroy(e);
  }
  OwnedEvent(const OwnedEvent&) = delete;
  OwnedEvent& operator=(const OwnedEvent&) = delete;
};

// SSLIC_TIMING: device-event marks on the streams (no host syncs in between)
struct EventMarks {
  bool on = std::getenv("SSLIC_TIMING") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(cudaStream_t s, const std::string& what) {
    if (!on) return;
    cudaEvent_t e;
    SSLIC_CUDA_CHECK(cudaEventCreate(&e));
    SSLIC_CUDA_CHECK(cudaEventRecord(e, s));
    ev.emplace_back(what, e);
  }
  ~EventMarks() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    std::string line;
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventSynchronize(ev[i].second);
      cudaEventElapsedTime(&ms, ev[0].second, ev[i].second);
      char buf[96];
      std::snprintf(buf, sizeof buf, " %s@%.1f", ev[i].first.c_str(), ms);
      line += buf;
    }
    for (auto& p : ev) cudaEventDestroy(p.second);
    std::fprintf(stderr, "[sslic] overlapped loop (ms from start):%s\n", line.c_str());
  }
};

// Pipelined start of a whole-volume run (Engine::pipeline_ok): the image
// travels host -> device in z chunks on a copy stream, and each chunk's
// arrival releases the perturbation of the clusters whose gradient hood it
// completes and iteration 0's assign of the region rows whose planes and
// candidate centres are then all present; iteration 0's update closes it.
// The H2D copy thus overlaps init + iteration 0 instead of preceding them.
void pipelined_start(Engine& e, const sslic_image* img, void* dev, Stream& st, EventMarks& em) {
  const int64_t d = img->dims[2];
  const size_t plane_bytes =
      (size_t)img->dims[0] * img->dims[1] * img->channels * dtype_size(img->dtype);
  const int64_t S = e.geom().grid[2], cells = e.geom().cells[2];
  const int64_t RZ = e.region_z(), rows = e.region_rows();
  constexpr int kChunks = 8;
  OwnedStream copy_stream;
  const cudaStream_t cs = copy_stream.s;
  OwnedEvent evs[kChunks + 1];
  cudaEvent_t ev[kChunks + 1];
  for (int i = 0; i <= kChunks; ++i) ev[i] = evs[i].e;
  SSLIC_CUDA_CHECK(cudaEventRecord(ev[kChunks], st.s));  // the device buffer exists
  SSLIC_CUDA_CHECK(cudaStreamWaitEvent(cs, ev[kChunks], 0));
  e.init_pipeline();
  int64_t z_init = 0, rows_done = 0;
  for (int c = 0; c < kChunks; ++c) {
    const int64_t p0 = d * c / kChunks, p1 = d * (c + 1) / kChunks;
    const bool last = c == kChunks - 1;
    if (p1 > p0)
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dev) + p0 * plane_bytes,
                                       static_cast<const char*>(img->data) + p0 * plane_bytes,
                                       (p1 - p0) * plane_bytes, cudaMemcpyHostToDevice, cs));
    SSLIC_CUDA_CHECK(cudaEventRecord(ev[c], cs));
    SSLIC_CUDA_CHECK(cudaStreamWaitEvent(st.s, ev[c], 0));
    // a cluster's perturbation reads planes [z - 2, z + 2] of its initial z
    const int64_t zi = last ? d : std::max(z_init, p1 - 2);
    e.init_range(z_init, zi);
    z_init = zi;
    // region rows whose planes have arrived and whose candidate clusters
    // (anchor cells up to (zhi + S) / S, k_region_cand) are perturbed
    int64_t r = rows_done;
    while (r < rows && !last) {
      const int64_t zhi = std::min((r + 1) * RZ, d) - 1;
      const int64_t chi = std::min((zhi + S) / S, cells - 1);
      const int64_t zc = std::min(chi * S + S / 2, d - 1);
      if (zhi >= p1 || zc >= z_init) break;
      ++r;
    }
    if (last) r = rows;
    e.assign_rows(rows_done, r);
    rows_done = r;
    em.mark(st.s, "chunk" + std::to_string(c));
  }
  e.update();
  em.mark(st.s, "it0");
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(cs));
}

int run_loop_overlapped(Engine& e, Stream& st, uint32_t* labels_out, int64_t n,
                        const sslic_image* pipelined_img = nullptr, void* dev = nullptr) {
  EventMarks em;
  em.mark(st.s, "start");
  if (pipelined_img) {
    pipelined_start(e, pipelined_img, dev, st, em);
  } else {
    e.init(true);
    e.commit();
    em.mark(st.s, "init");
  }
  const int iters = e.max_iterations();
  // the labels after iteration iters - 5 (iters - 4 for short runs) are
  // copied while the last iterations run (4.3 GB at PCIe speed take ~6 of
  // config 3's iterations); later changes travel as a change list
  const int snap = iters >= 8 ? iters - 5 : iters - 4;
  for (int it = e.iterations_done(); it < snap; ++it) {
    e.assign(true);
    e.update();
    em.mark(st.s, "it" + std::to_string(it));
  }
  DeviceBuf snapbuf(n * sizeof(uint32_t), st.s);
  e.unpack_labels(snapbuf.as<uint32_t>());
  em.mark(st.s, "snap");
  // The snapshot goes down in kPieces pieces on the DMA engine, submitted by
  // the host two at a time, so that the change lists (built on the device
  // after the last iteration) jump the queue as soon as they exist. Host
  // threads apply each piece's list once that piece and the lists have
  // landed, overlapping the remaining pieces' copies.
  constexpr int kPieces = 32, kInFlight = 2;
  const bool listed = n < ((int64_t)1 << 32);
  OwnedEvent ready_ev;
  const cudaEvent_t ready = ready_ev.e;
  SSLIC_CUDA_CHECK(cudaEventRecord(ready, st.s));
  OwnedStream copy_stream;
  const cudaStream_t cs = copy_stream.s;
  SSLIC_CUDA_CHECK(cudaStreamWaitEvent(cs, ready, 0));
  for (int it = std::max(snap, e.iterations_done()); it < iters; ++it) {
    e.assign(true);
    e.update();
    em.mark(st.s, "it" + std::to_string(it));
  }
  DeviceBuf fin(n * sizeof(uint32_t), st.s);  // unpacked only where needed
  if (!listed) {
    e.unpack_labels(fin.as<uint32_t>());  // >= 2^32 voxels: snapshot, then the changed labels via the mapped map
    OwnedEvent copied_ev;
    const cudaEvent_t copied = copied_ev.e;
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out, snapbuf.p, n * sizeof(uint32_t),
                                     cudaMemcpyDeviceToHost, cs));
    SSLIC_CUDA_CHECK(cudaEventRecord(copied, cs));
    SSLIC_CUDA_CHECK(cudaStreamWaitEvent(st.s, copied, 0));
    k_patch_labels_host<<<148 * 8, 256, 0, st.s>>>(n, snapbuf.as<uint32_t>(),
                                                    fin.as<uint32_t>(), labels_out);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    st.sync();
    if (e.undefined_seen())
      throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
    return e.iterations_done();
  }
  const int K = kPieces;
  std::vector<int64_t> c0(K + 1), cap(K), off(K, 0);
  for (int c = 0; c <= K; ++c) c0[c] = n * c / K;
  int64_t total_cap = 0;
  for (int c = 0; c < K; ++c) {
    cap[c] = (c0[c + 1] - c0[c]) / 20 + 1024;  // up to 5% (more -> the piece is copied whole)
    off[c] = total_cap;
    total_cap += cap[c];
  }
  DeviceBuf dlist((size_t)total_cap * sizeof(uint2), st.s);
  DeviceBuf cntb(K * sizeof(unsigned long long), st.s);
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cntb.p, 0, K * sizeof(unsigned long long), st.s));
  for (int c = 0; c < K; ++c) {
    k_change_list<<<148 * 2, 256, 0, st.s>>>(
        c0[c + 1] - c0[c], snapbuf.as<uint32_t>() + c0[c], e.label_words() + c0[c],
        cntb.as<unsigned long long>() + c, cap[c], dlist.as<uint2>() + off[c], (uint32_t)c0[c],
        e.codec().label_mask);
    SSLIC_CUDA_CHECK(cudaGetLastError());
  }
  MappedStage& ms = mapped_stage();
  std::lock_guard<std::mutex> lock(ms.mu);
  char* stage = static_cast<char*>(ms.get((size_t)total_cap * sizeof(uint2) + 64 * 8));
  auto* cnt_h = reinterpret_cast<unsigned long long*>(stage);
  uint2* list_h = reinterpret_cast<uint2*>(stage + 64 * 8);
  k_copy_counts<<<1, 32, 0, st.s>>>(cntb.as<unsigned long long>(), K, cnt_h);
  SSLIC_CUDA_CHECK(cudaGetLastError());
  OwnedEvent built_ev, lists_in_ev;
  const cudaEvent_t built = built_ev.e, lists_in = lists_in_ev.e;
  SSLIC_CUDA_CHECK(cudaEventRecord(built, st.s));
  em.mark(st.s, "lists");
  std::vector<OwnedEvent> copied_evs(K);
  std::vector<cudaEvent_t> copied(K);
  for (int c = 0; c < K; ++c) copied[c] = copied_evs[c].e;
  ChunkApplier ap(labels_out, K);
  for (int c = 0; c < K; ++c) ap.lists[c] = list_h + off[c];
  ap.start();
  std::vector<char> whole(K, 0);
  bool lists_sent = false;
  unsigned long long total = 0;
  auto send_lists = [&]() {  // counts are in host memory once `built` completed
    for (int c = 0; c < K; ++c) {
      total += cnt_h[c];
      if ((int64_t)cnt_h[c] <= cap[c]) {
        ap.counts[c] = (int64_t)cnt_h[c];
        if (cnt_h[c])
          SSLIC_CUDA_CHECK(cudaMemcpyAsync(list_h + off[c], dlist.as<uint2>() + off[c],
                                           cnt_h[c] * sizeof(uint2), cudaMemcpyDeviceToHost,
                                           cs));
      } else {
        whole[c] = 1;
      }
    }
    SSLIC_CUDA_CHECK(cudaEventRecord(lists_in, cs));
    em.mark(cs, "lists-d2h");
    lists_sent = true;
  };
  SSLIC_CUDA_CHECK(cudaEventSynchronize(ready));  // the snapshot exists
  int submitted = 0, landed = 0, applied = 0;
  while (applied < K) {
    while (submitted < K && submitted - landed < kInFlight) {
      const int c = submitted++;
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out + c0[c], snapbuf.as<uint32_t>() + c0[c],
                                       (c0[c + 1] - c0[c]) * sizeof(uint32_t),
                                       cudaMemcpyDeviceToHost, cs));
      SSLIC_CUDA_CHECK(cudaEventRecord(copied[c], cs));
    }
    if (!lists_sent && cudaEventQuery(built) == cudaSuccess) send_lists();
    if (landed < submitted) {
      SSLIC_CUDA_CHECK(cudaEventSynchronize(copied[landed]));
      ++landed;
    }
    if (lists_sent && landed > applied && cudaEventQuery(lists_in) == cudaSuccess) {
      while (applied < landed) ap.ready(applied++);
    } else if (landed == K) {
      if (!lists_sent) {
        SSLIC_CUDA_CHECK(cudaEventSynchronize(built));
        send_lists();
      }
      SSLIC_CUDA_CHECK(cudaEventSynchronize(lists_in));
    }
  }
  ap.join();
  bool any_whole = false;
  for (int c = 0; c < K; ++c)
    if (whole[c]) {  // too many changes in this piece: its final labels, whole
      if (!any_whole) {
        e.unpack_labels(fin.as<uint32_t>());
        st.sync();
      }
      any_whole = true;
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out + c0[c], fin.as<uint32_t>() + c0[c],
                                       (c0[c + 1] - c0[c]) * sizeof(uint32_t),
                                       cudaMemcpyDeviceToHost, cs));
    }
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(cs));
  st.sync();
  if (em.on)
    std::fprintf(stderr, "[sslic] change lists: %llu entries (%.2f%% of the map)%s\n", total,
                 100.0 * (double)total / (double)n, any_whole ? ", some pieces copied whole" : "");
  if (e.undefined_seen())
    throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
  return e.iterations_done();
}

// The host buffer is page-locked and mapped into the device address space.
bool host_pinned_mapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer == p;
}

int run_loop(Engine& e, const sslic_params* p, Stream& st) {
  e.init(true);
  e.commit();
  const int iters = e.max_iterations();
  // Tag mode: the fused update latches "an assignment left a voxel
  // undefined" on the device, so the loop needs no host sync per iteration;
  // the reference's logic_error (slic.hpp:330-331) is raised after it.
  const bool latched = !e.dist_mode();
  for (int it = 0; it < iters; ++it) {
    e.assign(true);
    if (!latched && e.undefined_count() > 0)  // slic.hpp:330-331
      throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
    e.update();
    if (p->has_residual_threshold) {
      double r = 0.0;
      std::vector<double> rs(e.iterations_done());
      e.residuals_to_host(rs.data(), e.iterations_done());
      r = rs.back();
      if (r <= p->residual_threshold) break;  // slic.hpp:411
    }
  }
  st.sync();
  if (latched && e.undefined_seen())
    throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
  return e.iterations_done();
}

__global__ void k_update_from_sums(int64_t k, int stride, const double* sums,
                                   const int64_t* counts, double* centers, double* partial) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double part = 0.0;
  if (id < k && counts[id] != 0) {
    for (int i = 0; i < stride; ++i) {
      const double v = __ddiv_rn(sums[id * stride + i], (double)counts[id]);
      const double d = __dsub_rn(v, centers[id * stride + i]);
      centers[id * stride + i] = v;
      part = __dadd_rn(part, __dmul_rn(d, d));
    }
  }
  __shared__ double red[256];
  red[threadIdx.x] = part;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

}  // namespace


extern "C" {

const char* sslic_last_error(void) { return sslic_b200::last_error().c_str(); }
const char* sslic_version(void) { return "sslic_b200 0.1 (sm_100a)"; }

int64_t sslic_cluster_count(int rank, const int64_t* dims, const int64_t* grid) {
  if (rank < 1 || rank > kMaxRank || !dims || !grid) return 0;
  int64_t k = 1;
  for (int a = 0; a < rank; ++a) {
    if (grid[a] < 1 || dims[a] < 1) return 0;
    k *= (dims[a] + grid[a] - 1) / grid[a];
  }
  return k;
}

int sslic_iterations_for(const sslic_params* p, int rank) {
  if (!p) return 0;
  return p->max_iterations > 0 ? p->max_iterations : (rank <= 2 ? 10 : 5);
}

int sslic_run_slic(const sslic_image* img, const sslic_params* params, int device,
                   uint32_t* labels_out, double* centers_out, double* residuals_out,
                   int* iterations_done) {
  return guarded([&] {
    validate_image(img);
    validate_params(params, img);
    PhaseTimer pt("run_slic");
    Stream st(device);
    const int64_t n = pixel_count(*img);
    const int64_t last = img->dims[img->rank - 1];
    // the overlapped download keeps a label snapshot on the device (4 B per
    // voxel) next to the image and the label words: only when it fits
    size_t free_b = 0, total_b = 0;
    SSLIC_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const double need = (double)n * (4.0 + 4.0 + img->channels * (double)dtype_size(img->dtype));
    const bool overlapped = !params->has_residual_threshold && n >= ((int64_t)1 << 24) &&
                            host_pinned_mapped(labels_out) && need < 0.9 * (double)free_b;
    // pipelined upload (u8/u16 volumes: no image-wide pre-pass before init)
    const size_t img_bytes = (size_t)n * img->channels * dtype_size(img->dtype);
    std::unique_ptr<DeviceBuf> dimg;
    int dtype_dev = img->dtype;
    bool pipelined = false;
    if (overlapped && img->rank == 3 && (img->dtype == SSLIC_U8 || img->dtype == SSLIC_U16) &&
        std::getenv("SSLIC_NO_PIPELINED_UPLOAD") == nullptr) {
      dimg = std::make_unique<DeviceBuf>(img_bytes, st.s);
      pipelined = true;
    } else {
      dimg = upload_image(img, st, &dtype_dev);  // (fp64 storage of narrower data: narrowed)
      pt.mark(st, "upload");
    }
    sslic_image v = device_view(img, dimg->p);
    v.dtype = dtype_dev;
    Engine e(v, *params, device, 0, last, 0, last, st.s);
    if (pipelined && !(e.pipeline_ok() && !e.dist_mode() && e.max_iterations() >= 4)) {
      SSLIC_CUDA_CHECK(
          cudaMemcpyAsync(dimg->p, img->data, img_bytes, cudaMemcpyHostToDevice, st.s));
      pipelined = false;
    }
    pt.mark(st, "engine");
    int done = 0;
    if (!e.dist_mode() && overlapped && e.max_iterations() >= 4) {
      done = run_loop_overlapped(e, st, labels_out, n, pipelined ? img : nullptr, dimg->p);
      pt.mark(st, pipelined ? "pipelined upload + iterations + overlapped label download"
                            : "iterations + overlapped label download");
    } else {
      done = run_loop(e, params, st);
      pt.mark(st, "iterations");
      // the engine is done with its words and the image: unpack in place
      dimg.reset();
      uint32_t* lab = e.label_words();
      e.unpack_labels(lab);
      copy_to_host(labels_out, lab, n * sizeof(uint32_t), device, st.s);
      st.sync();
      pt.mark(st, "labels D2H");
    }
    e.copy_centers_to_host(centers_out);
    if (residuals_out) e.residuals_to_host(residuals_out, done);
    if (iterations_done) *iterations_done = done;
    return SSLIC_OK;
  });
}

int sslic_segment(const sslic_image* img, const sslic_params* params, int device,
                  uint32_t* labels_out, double* centers_out, double* residuals_out,
                  int* iterations_done, uint32_t* next_label_out) {
  return guarded([&] {
    validate_image(img);
    validate_params(params, img);
    Stream st(device);
    PhaseTimer pt("segment");
    int dtype_dev = img->dtype;
    auto dimg = upload_image(img, st, &dtype_dev);
    sslic_image v = device_view(img, dimg->p);
    v.dtype = dtype_dev;
    const int64_t last = img->dims[img->rank - 1];
    Engine e(v, *params, device, 0, last, 0, last, st.s);
    const int done = run_loop(e, params, st);
    pt.mark(st, "upload + iterations");
    const int64_t n = pixel_count(*img);
    // Memory-lean tail (config 5: 17.4 G voxels): the image is no longer
    // read, the label words are unpacked in place and relabelled in place,
    // so the connectivity pass needs only the node ids on top of the map.
    dimg.reset();
    uint32_t* lab = e.label_words();
    e.unpack_labels(lab);
    uint32_t next = (uint32_t)e.geom().k;
    if (params->enforce_connectivity) {
      next = enforce_connectivity_device(e.geom(), lab, e.current_centers(), lab, st.s);
      pt.mark(st, "connectivity");
    }
    copy_to_host(labels_out, lab, n * sizeof(uint32_t), device, st.s);
    st.sync();
    pt.mark(st, "labels D2H");
    e.copy_centers_to_host(centers_out);
    if (residuals_out) e.residuals_to_host(residuals_out, done);
    if (iterations_done) *iterations_done = done;
    if (next_label_out) *next_label_out = next;
    return SSLIC_OK;
  });
}

int sslic_segment_write(const sslic_image* img, const sslic_params* params, int device,
                        const char* labels_path, const char* contour_path, double* centers_out,
                        double* residuals_out, int* iterations_done, uint32_t* next_label_out) {
  return guarded([&] {
    validate_image(img);
    validate_params(params, img);
    if (!labels_path) throw Error(SSLIC_EINVAL, "segment_write: null labels path");
    Stream st(device);
    PhaseTimer pt("segment_write");
    int dtype_dev = img->dtype;
    auto dimg = upload_image(img, st, &dtype_dev);
    sslic_image v = device_view(img, dimg->p);
    v.dtype = dtype_dev;
    const int64_t last = img->dims[img->rank - 1];
    Engine e(v, *params, device, 0, last, 0, last, st.s);
    const int done = run_loop(e, params, st);
    pt.mark(st, "upload + iterations");
    const int64_t n = pixel_count(*img);
    dimg.reset();
    uint32_t* lab = e.label_words();
    e.unpack_labels(lab);
    // the final pass also yields the label count and the contour bitmask
    const int64_t words = (n + 31) / 32;
    DeviceBuf dmax(sizeof(unsigned), st.s), dbits(contour_path ? words * 4 : 4, st.s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(dmax.p, 0, sizeof(unsigned), st.s));
    if (contour_path) SSLIC_CUDA_CHECK(cudaMemsetAsync(dbits.p, 0, words * 4, st.s));
    LabelOutputs outs;
    outs.max_label = dmax.as<unsigned>();
    outs.boundary = contour_path ? dbits.as<uint32_t>() : nullptr;
    uint32_t next = (uint32_t)e.geom().k;
    if (params->enforce_connectivity)
      next = enforce_connectivity_device(e.geom(), lab, e.current_centers(), lab, st.s, outs);
    else
      label_outputs_device(e.geom(), lab, outs, st.s);
    pt.mark(st, params->enforce_connectivity ? "connectivity (fused outputs)" : "outputs");
    std::vector<uint32_t> host((size_t)n);
    std::vector<uint32_t> bits(contour_path ? (size_t)words : 0);
    unsigned mx = 0;
    copy_to_host(host.data(), lab, n * sizeof(uint32_t), device, st.s);
    if (contour_path)
      SSLIC_CUDA_CHECK(
          cudaMemcpyAsync(bits.data(), dbits.p, words * 4, cudaMemcpyDeviceToHost, st.s));
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(&mx, dmax.p, sizeof mx, cudaMemcpyDeviceToHost, st.s));
    e.copy_centers_to_host(centers_out);  // (synchronizes)
    if (residuals_out) e.residuals_to_host(residuals_out, done);
    pt.mark(st, "D2H");
    write_labels_counted(labels_path, img->rank, img->dims, host.data(), (uint64_t)mx + 1);
    if (contour_path) write_contour_f32(contour_path, img, bits.data());
    pt.mark(st, "files");
    if (iterations_done) *iterations_done = done;
    if (next_label_out) *next_label_out = next;
    return SSLIC_OK;
  });
}

int sslic_init_centers(const sslic_image* img, const sslic_params* params, int perturb,
                       int device, double* centers_out) {
  return guarded([&] {
    validate_image(img);
    validate_params(params, img);
    Stream st(device);
    auto dimg = upload_image(img, st);
    const sslic_image v = device_view(img, dimg->p);
    const int64_t last = img->dims[img->rank - 1];
    Engine e(v, *params, device, 0, last, 0, last, st.s, true);
    e.init(perturb != 0);
    e.copy_centers_to_host(centers_out);
    return SSLIC_OK;
  });
}

int sslic_perturb_centers(const sslic_image* img, double* centers, int64_t k, int device) {
  return guarded([&] {
    validate_image(img);
    Stream st(device);
    auto dimg = upload_image(img, st);
    Geom g{};
    g.rank = img->rank;
    g.channels = img->channels;
    g.stride = img->channels + img->rank;
    g.dtype = img->dtype;
    int64_t acc = 1;
    for (int a = 0; a < kMaxRank; ++a) {
      g.dims[a] = a < img->rank ? img->dims[a] : 1;
      g.strides[a] = acc;
      acc *= g.dims[a];
      g.grid[a] = g.cells[a] = 1;
    }
    g.k = k;
    g.plane = acc / g.dims[img->rank - 1];
    g.slab_begin = g.data_begin = 0;
    g.slab_end = g.data_end = g.dims[img->rank - 1];
    DeviceBuf c(k * g.stride * sizeof(double), st.s);
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(c.p, centers, k * g.stride * sizeof(double),
                                     cudaMemcpyHostToDevice, st.s));
    if (k > 0) {
      k_perturb_table<<<(unsigned)((k + 127) / 128), 128, 0, st.s>>>(g, dimg->p, c.as<double>());
      SSLIC_CUDA_CHECK(cudaGetLastError());
    }
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(centers, c.p, k * g.stride * sizeof(double),
                                     cudaMemcpyDeviceToHost, st.s));
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_convert_image_to_lab(const sslic_image* img, int device, double* lab_out) {
  return guarded([&] {
    validate_image(img);
    if (img->channels != 3)
      throw Error(SSLIC_EINVAL, "convert_image_to_lab: image must have 3 channels");
    Stream st(device);
    auto dimg = upload_image(img, st);
    const int64_t npix = pixel_count(*img);
    double table[256];
    sslic_b200::srgb_linear_table(table);
    DeviceBuf dt(sizeof(table), st.s), dout(npix * 3 * sizeof(double), st.s);
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(dt.p, table, sizeof(table), cudaMemcpyHostToDevice, st.s));
    sslic_b200::srgb_to_lab_device(dimg->p, img->dtype, npix, dt.as<double>(),
                                   dout.as<double>(), st.s);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    copy_to_host(lab_out, dout.p, npix * 3 * sizeof(double), device, st.s);
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_mask_label_contour(const sslic_image* img, int label_rank, const int64_t* label_dims,
                             const uint32_t* labels, int device, double* out) {
  return guarded([&] {
    validate_image(img);
    bool same = label_rank == img->rank && label_dims != nullptr;
    for (int a = 0; same && a < img->rank; ++a) same = label_dims[a] == img->dims[a];
    if (!same) throw Error(SSLIC_EINVAL, "mask_label_contour: image and label dims differ");
    Stream st(device);
    auto dimg = upload_image(img, st);
    const int64_t n = pixel_count(*img);
    sslic_b200::Geom g{};
    g.rank = img->rank;
    g.channels = img->channels;
    g.dtype = img->dtype;
    int64_t acc = 1;
    for (int a = 0; a < kMaxRank; ++a) {
      g.dims[a] = a < img->rank ? img->dims[a] : 1;
      g.strides[a] = acc;
      acc *= g.dims[a];
    }
    DeviceBuf dl(n * sizeof(uint32_t), st.s), dout(n * img->channels * sizeof(double), st.s);
    copy_to_device(dl.p, labels, n * sizeof(uint32_t), device, st.s);
    sslic_b200::mask_label_contour_device(g, dimg->p, dl.as<uint32_t>(),
                                          dout.as<double>(), st.s);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    copy_to_host(out, dout.p, n * img->channels * sizeof(double), device, st.s);
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_gradient_sq(const sslic_image* img, const int64_t* coords, int64_t n, int device,
                      double* out) {
  return guarded([&] {
    validate_image(img);
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < img->rank; ++a)
        if (coords[i * img->rank + a] < 0 || coords[i * img->rank + a] >= img->dims[a])
          throw Error(SSLIC_ERANGE, "linear_index: coordinate outside image");
    Stream st(device);
    auto dimg = upload_image(img, st);
    sslic_params p = default_params_for(img, img->dims, 10.0);
    const sslic_image v = device_view(img, dimg->p);
    const int64_t last = img->dims[img->rank - 1];
    Engine e(v, p, device, 0, last, 0, last, st.s, true);
    DeviceBuf dc(n * img->rank * sizeof(int64_t), st.s), dout(n * sizeof(double), st.s);
    copy_to_device(dc.p, coords, n * img->rank * sizeof(int64_t), device, st.s);
    if (n > 0) {
      k_gradient_points<<<(unsigned)((n + 127) / 128), 128, 0, st.s>>>(
          e.geom(), dimg->p, dc.as<int64_t>(), n, dout.as<double>());
      SSLIC_CUDA_CHECK(cudaGetLastError());
    }
    copy_to_host(out, dout.p, n * sizeof(double), device, st.s);
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_squared_distance(int channels, int rank, const int64_t* grid, double weight_m,
                           int64_t n, const double* centers, const double* pixels,
                           const int64_t* coords, int device, double* out) {
  return guarded([&] {
    if (rank < 1 || rank > kMaxRank || channels < 1)
      throw Error(SSLIC_EINVAL, "squared_distance: center size must be channels + rank");
    Stream st(device);
    Geom g{};
    g.rank = rank;
    g.channels = channels;
    g.stride = channels + rank;
    for (int a = 0; a < kMaxRank; ++a) g.grid[a] = a < rank ? (int)grid[a] : 1;
    g.m_sq = weight_m * weight_m;
    DeviceBuf dc(n * g.stride * sizeof(double), st.s), dp(n * channels * sizeof(double), st.s),
        dx(n * rank * sizeof(int64_t), st.s), dout(n * sizeof(double), st.s);
    copy_to_device(dc.p, centers, n * g.stride * sizeof(double), device, st.s);
    copy_to_device(dp.p, pixels, n * channels * sizeof(double), device, st.s);
    copy_to_device(dx.p, coords, n * rank * sizeof(int64_t), device, st.s);
    if (n > 0) {
      k_distance_points<<<(unsigned)((n + 127) / 128), 128, 0, st.s>>>(
          g, n, dc.as<double>(), dp.as<double>(), dx.as<int64_t>(), dout.as<double>());
      SSLIC_CUDA_CHECK(cudaGetLastError());
    }
    copy_to_host(out, dout.p, n * sizeof(double), device, st.s);
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_assign_pass(const sslic_image* img, const sslic_params* params, const double* centers,
                      int64_t k, int device, uint32_t* labels, double* dists) {
  return guarded([&] {
    validate_image(img);
    for (int a = 0; a < img->rank; ++a)
      if (params->grid[a] < 1) throw Error(SSLIC_EINVAL, "SlicParams: grid sizes must be >= 1");
    Stream st(device);
    auto dimg = upload_image(img, st);
    // The engine sizes its table from the grid; a caller table may differ in
    // k, so build the engine with a grid whose cell count we override below.
    const sslic_image v = device_view(img, dimg->p);
    const int64_t last = img->dims[img->rank - 1];
    sslic_params p = *params;
    p.max_iterations = 1;
    Engine e(v, p, device, 0, last, 0, last, st.s, true, k);
    e.set_centers_host(centers);
    e.commit();
    const int64_t n = pixel_count(*img);
    copy_to_device(e.label_words(), labels, n * sizeof(uint32_t), device, st.s);
    copy_to_device(e.dists(), dists, n * sizeof(double), device, st.s);
    e.assign(false);
    copy_to_host(labels, e.label_words(), n * sizeof(uint32_t), device, st.s);
    copy_to_host(dists, e.dists(), n * sizeof(double), device, st.s);
    st.sync();
    return SSLIC_OK;
  });
}

int sslic_accumulate(const sslic_image* img, const uint32_t* labels, int64_t k, int device,
                     double* sums_out, int64_t* counts_out) {
  return guarded([&] {
    validate_image(img);
    if (k < 0) throw Error(SSLIC_EINVAL, "accumulate: k must be >= 0");
    Stream st(device);
    auto dimg = upload_image(img, st);
    const sslic_image v = device_view(img, dimg->p);
    const int64_t last = img->dims[img->rank - 1];
    // A grid giving exactly k cells is not needed: the engine only uses k for
    // the accumulator size, so use grid = dims (k = 1) and then resize.
    sslic_params p = default_params_for(img, img->dims, 10.0);
    p.max_iterations = 1;
    Engine e(v, p, device, 0, last, 0, last, st.s, true);
    Geom g = e.geom();
    g.k = k;
    const int64_t n = pixel_count(*img);
    DeviceBuf acc((k * (g.stride + 1) + 2) * sizeof(unsigned long long), st.s);
    DeviceBuf dl(n * sizeof(uint32_t), st.s);
    copy_to_device(dl.p, labels, n * sizeof(uint32_t), device, st.s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(acc.p, 0, (k * (g.stride + 1) + 2) * sizeof(unsigned long long),
                                     st.s));
    unsigned long long* a = acc.as<unsigned long long>();
    k_accumulate<<<(unsigned)((n + 255) / 256), 256, 0, st.s>>>(
        g, dimg->p, dl.as<uint32_t>(), LabelCodec{32, 0xffffffffu}, e.value_shift(), a + 2, a,
        a + 1);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    std::vector<long long> h(k * (g.stride + 1) + 2);
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(h.data(), acc.p, h.size() * sizeof(long long),
                                     cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (h[0]) throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
    if (h[1]) throw Error(SSLIC_EINVAL, "accumulate: label >= k");
    for (int64_t id = 0; id < k; ++id) {
      const long long* r = h.data() + 2 + id * (g.stride + 1);
      for (int i = 0; i < g.stride; ++i)
        sums_out[id * g.stride + i] =
            i < g.channels ? std::ldexp((double)r[i], -e.value_shift()) : (double)r[i];
      counts_out[id] = r[g.stride];
    }
    return SSLIC_OK;
  });
}

int sslic_reduce_and_update(double* centers, int64_t k, int stride, const double* sums,
                            const int64_t* counts, int device, double* residual_out) {
  return guarded([&] {
    if (k < 0 || stride < 1) throw Error(SSLIC_EINVAL, "reduce_and_update: bad table shape");
    Stream st(device);
    DeviceBuf dc(k * stride * sizeof(double), st.s), ds(k * stride * sizeof(double), st.s),
        dn(k * sizeof(int64_t), st.s);
    const int nb = (int)((k + 255) / 256);
    DeviceBuf part((nb + 1) * sizeof(double), st.s);
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(dc.p, centers, k * stride * sizeof(double),
                                     cudaMemcpyHostToDevice, st.s));
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(ds.p, sums, k * stride * sizeof(double),
                                     cudaMemcpyHostToDevice, st.s));
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(dn.p, counts, k * sizeof(int64_t), cudaMemcpyHostToDevice,
                                     st.s));
    double r = 0.0;
    if (k > 0) {
      k_update_from_sums<<<nb, 256, 0, st.s>>>(k, stride, ds.as<double>(), dn.as<int64_t>(),
                                               dc.as<double>(), part.as<double>());
      k_residual_final<<<1, 1024, 0, st.s>>>(part.as<double>(), nb, part.as<double>() + nb);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(&r, part.as<double>() + nb, sizeof(double),
                                       cudaMemcpyDeviceToHost, st.s));
    }
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(centers, dc.p, k * stride * sizeof(double),
                                     cudaMemcpyDeviceToHost, st.s));
    st.sync();
    if (residual_out) *residual_out = r;
    return SSLIC_OK;
  });
}

int sslic_enforce_connectivity(int rank, const int64_t* dims, const uint32_t* labels_in,
                               const double* centers, int channels, int64_t k,
                               const int64_t* grid, int device, uint32_t* labels_out,
                               uint32_t* next_label_out) {
  return guarded([&] {
    if (rank < 1 || rank > kMaxRank || channels < 1 || k < 0)
      throw Error(SSLIC_EINVAL, "enforce_connectivity: bad shape");
    Stream st(device);
    Geom g{};
    g.rank = rank;
    g.channels = channels;
    g.stride = channels + rank;
    int64_t acc = 1;
    for (int a = 0; a < kMaxRank; ++a) {
      g.dims[a] = a < rank ? dims[a] : 1;
      g.grid[a] = a < rank ? (int)grid[a] : 1;
      if (g.dims[a] < 1 || g.grid[a] < 1) throw Error(SSLIC_EINVAL, "bad dims/grid");
      g.cells[a] = (int)((g.dims[a] + g.grid[a] - 1) / g.grid[a]);
      g.strides[a] = acc;
      acc *= g.dims[a];
    }
    g.k = k;
    g.ncells = 1;
    for (int a = 0; a < kMaxRank; ++a) g.ncells *= g.cells[a];
    g.plane = acc / g.dims[rank - 1];
    g.slab_begin = g.data_begin = 0;
    g.slab_end = g.data_end = g.dims[rank - 1];
    const int64_t n = acc;
    // relabelled in place on the device (4 bytes per voxel + the node ids)
    DeviceBuf din(n * sizeof(uint32_t), st.s), dc(k * g.stride * sizeof(double), st.s);
    copy_to_device(din.p, labels_in, n * sizeof(uint32_t), device, st.s);  // (pageable: striped)
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(dc.p, centers, k * g.stride * sizeof(double),
                                     cudaMemcpyHostToDevice, st.s));
    const uint32_t next = enforce_connectivity_device(g, din.as<uint32_t>(), dc.as<double>(),
                                                      din.as<uint32_t>(), st.s);
    copy_to_host(labels_out, din.p, n * sizeof(uint32_t), device, st.s);
    st.sync();
    if (next_label_out) *next_label_out = next;
    return SSLIC_OK;
  });
}

// ---- engine -----------------------------------------------------------------

int sslic_engine_create(const sslic_image* img, const sslic_params* params, int device,
                        int64_t slab_begin, int64_t slab_end, int64_t data_begin,
                        int64_t data_end, void* stream, sslic_engine** out) {
  return guarded([&] {
    validate_image(img);
    validate_params(params, img);
    const int64_t last = img->dims[img->rank - 1];
    if (slab_begin < 0 || slab_end > last || slab_begin >= slab_end)
      throw Error(SSLIC_EINVAL, "engine: bad slab range");
    const int64_t need_lo = slab_begin - 2 < 0 ? 0 : slab_begin - 2;
    const int64_t need_hi = slab_end + 2 > last ? last : slab_end + 2;
    if (data_begin > need_lo || data_end < need_hi)
      throw Error(SSLIC_EINVAL, "engine: data planes must cover the slab plus a 2-plane halo");
    sslic_image v = device_view(img, img->data);
    auto h = std::make_unique<sslic_engine>();
    h->e = std::make_unique<Engine>(v, *params, device, slab_begin, slab_end, data_begin,
                                    data_end, static_cast<cudaStream_t>(stream));
    *out = h.release();
    return SSLIC_OK;
  });
}

int sslic_engine_destroy(sslic_engine* e) {
  return guarded([&] {
    delete e;
    return SSLIC_OK;
  });
}

int sslic_engine_reset(sslic_engine* e) {
  return guarded([&] {
    SSLIC_CUDA_CHECK(cudaSetDevice(e->e->device()));
    e->e->reset();
    return SSLIC_OK;
  });
}

int sslic_engine_init(sslic_engine* e) {
  return guarded([&] {
    e->e->init(true);
    return SSLIC_OK;
  });
}

int sslic_engine_centers_buffer(sslic_engine* e, double** dev_ptr, int64_t* count) {
  return guarded([&] {
    *dev_ptr = e->e->current_centers();
    *count = e->e->centers_count();
    return SSLIC_OK;
  });
}

int sslic_engine_commit_centers(sslic_engine* e) {
  return guarded([&] {
    e->e->commit();
    return SSLIC_OK;
  });
}

int sslic_engine_assign(sslic_engine* e) {
  return guarded([&] {
    e->e->assign(true);
    return SSLIC_OK;
  });
}

int sslic_engine_partials(sslic_engine* e, int64_t** dev_ptr, int64_t* count) {
  return guarded([&] {
    *dev_ptr = reinterpret_cast<int64_t*>(e->e->partials());
    *count = e->e->partials_count();
    return SSLIC_OK;
  });
}

int sslic_engine_update(sslic_engine* e) {
  return guarded([&] {
    e->e->update();
    return SSLIC_OK;
  });
}

int sslic_engine_iterate(sslic_engine* e, int iterations) {
  return guarded([&] {
    SSLIC_CUDA_CHECK(cudaSetDevice(e->e->device()));
    for (int i = 0; i < iterations; ++i) {
      e->e->assign(true);
      comm_sum_partials(e->comm, *e->e);  // attached NCCL communicator (multi.cu)
      e->e->update();
    }
    return SSLIC_OK;
  });
}

int sslic_engine_iterate_graph(sslic_engine* e, int iterations, float* ms_out) {
  return guarded([&] {
    // Capture `iterations` assign+update steps on the engine's stream into
    // one CUDA graph, then launch it once: the per-kernel launch gaps of a
    // small volume disappear. The iterations execute at the launch (the
    // capture only records them); ms_out is the launch's device time.
    sslic_b200::Engine& en = *e->e;
    SSLIC_CUDA_CHECK(cudaSetDevice(en.device()));
    cudaStream_t s = en.stream();
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    SSLIC_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      for (int i = 0; i < iterations; ++i) {
        en.assign(true);
        comm_sum_partials(e->comm, en);  // the NCCL allreduce is a graph node
        en.update();
      }
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    SSLIC_CUDA_CHECK(cudaStreamEndCapture(s, &graph));
    SSLIC_CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
    cudaEvent_t a, b;
    SSLIC_CUDA_CHECK(cudaEventCreate(&a));
    SSLIC_CUDA_CHECK(cudaEventCreate(&b));
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    SSLIC_CUDA_CHECK(cudaEventRecord(a, s));
    SSLIC_CUDA_CHECK(cudaGraphLaunch(exec, s));
    SSLIC_CUDA_CHECK(cudaEventRecord(b, s));
    SSLIC_CUDA_CHECK(cudaEventSynchronize(b));
    float ms = 0.f;
    SSLIC_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    if (ms_out) *ms_out = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    return SSLIC_OK;
  });
}

int sslic_engine_iterations_done(sslic_engine* e) { return e ? e->e->iterations_done() : 0; }

int sslic_engine_residuals(sslic_engine* e, double* host_out) {
  return guarded([&] {
    e->e->residuals_to_host(host_out, e->e->iterations_done());
    return SSLIC_OK;
  });
}

int sslic_engine_labels(sslic_engine* e, uint32_t* dev_out) {
  return guarded([&] {
    e->e->unpack_labels(dev_out);
    return SSLIC_OK;
  });
}

int sslic_engine_centers(sslic_engine* e, double* host_out) {
  return guarded([&] {
    e->e->copy_centers_to_host(host_out);
    return SSLIC_OK;
  });
}

int64_t sslic_engine_undefined_count(sslic_engine* e) {
  int64_t v = -1;
  guarded([&] {
    v = e->e->undefined_count();
    return SSLIC_OK;
  });
  return v;
}

int64_t sslic_engine_launch_count(sslic_engine* e) { return e ? e->e->launches() : 0; }

int sslic_engine_assign_ms(sslic_engine* e, int i, float* ms_out, int* n_out) {
  return guarded([&] {
    if (n_out) *n_out = e->e->assign_calls();
    if (ms_out) *ms_out = e->e->assign_ms(i);
    return SSLIC_OK;
  });
}

int sslic_engine_value_range(sslic_engine* e, double* absmax_out) {
  return guarded([&] {
    if (!absmax_out) throw Error(SSLIC_EINVAL, "null output");
    *absmax_out = e->e->value_range();
    return SSLIC_OK;
  });
}

int sslic_engine_set_value_range(sslic_engine* e, double absmax) {
  return guarded([&] {
    e->e->set_value_range(absmax);
    return SSLIC_OK;
  });
}

int sslic_engine_set_exact(sslic_engine* e, int exact) {
  return guarded([&] {
    const bool fast_ok = e->e->fast_supported();
    e->e->set_path(exact || !fast_ok ? AssignPath::kExact : AssignPath::kFast);
    return SSLIC_OK;
  });
}

int sslic_engine_fast_stats(sslic_engine* e, double* ambiguous, double* overflow_blocks,
                            double* changed) {
  return guarded([&] {
    e->e->fast_stats(ambiguous, overflow_blocks, changed);
    return SSLIC_OK;
  });
}

int sslic_engine_set_stats(sslic_engine* e, int on) {
  return guarded([&] {
    e->e->set_collect_stats(on != 0);
    return SSLIC_OK;
  });
}

int sslic_engine_eval_stats(sslic_engine* e, double* evals, double* window_evals) {
  return guarded([&] {
    e->e->eval_stats(evals, window_evals);
    return SSLIC_OK;
  });
}

}  // extern "C"
