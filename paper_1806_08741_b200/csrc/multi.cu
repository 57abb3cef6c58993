// Multi-GPU run_slic behind the C ABI (north_star "slabs along
// the slowest axis across the 8 GPUs of one box ... per-cluster partial sums
// combined by an NCCL allreduce over NVLink each iteration").
//
// The reference parallelises run_slic(img, params, workers) over slabs with
// an ordered merge of per-slab accumulators (slic.hpp:384-415,
// parallel.hpp:52-94). Here each GPU owns one z-slab of the volume (its
// planes plus the 2-plane perturbation halo are the only image bytes it
// holds) and the per-iteration exchange is one ncclAllReduce of the int64
// per-cluster deltas; every rank then runs the identical update. Integer sums
// are associative, so labels, centres and residuals are bitwise the
// single-GPU result for any device count.
//
// Two launch shapes share one per-rank body (run_rank):
//  * sslic_run_slic_multi: one process, one host thread per device,
//    communicators from ncclCommInitAll;
//  * sslic_run_slic_rank: one process per GPU (torchrun), communicator from
//    ncclCommInitRank on a unique id the caller distributes.
// Engines can also be attached to a communicator (sslic_engine_attach_nccl):
// sslic_engine_start / _iterate / _iterate_graph then run the collectives on
// the engine's stream, inside the captured CUDA graph.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.cuh"

using namespace sslic_b200;

namespace sslic_b200 {

struct RankComm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  double* scratch = nullptr;  // one device double (value-range MAX)
};

namespace {

#define SSLIC_NCCL_CHECK(expr)                                                        \
  do {                                                                                \
    const ncclResult_t r_ = (expr);                                                   \
    if (r_ != ncclSuccess)                                                            \
      throw Error(SSLIC_ECUDA, std::string("NCCL: ") + ncclGetErrorString(r_) + " (" + \
                                   #expr + ")");                                      \
  } while (0)

size_t dsize(int dt) {
  switch (dt) {
    case SSLIC_U8: return 1;
    case SSLIC_U16: return 2;
    case SSLIC_F32: return 4;
    case SSLIC_F64: return 8;
    default: return 0;
  }
}

}  // namespace

void comm_destroy(RankComm* c) {
  if (!c) return;
  if (c->scratch) cudaFree(c->scratch);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

void comm_sync_value_range(RankComm* c, Engine& e) {
  if (!c) return;  // (a 1-rank communicator still runs: the path is exercised on one GPU)
  const double v = e.value_range();
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(c->scratch, &v, sizeof v, cudaMemcpyHostToDevice, e.stream()));
  SSLIC_NCCL_CHECK(ncclAllReduce(c->scratch, c->scratch, 1, ncclFloat64, ncclMax, c->comm,
                                 e.stream()));
  double m = 0.0;
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&m, c->scratch, sizeof m, cudaMemcpyDeviceToHost, e.stream()));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(e.stream()));
  e.set_value_range(m);
}

// Init tables: each rank wrote its slab's clusters and zeros elsewhere, so
// the fp64 SUM has one non-zero term per entry (exact).
void comm_sum_centers(RankComm* c, Engine& e) {
  if (!c) return;  // (a 1-rank communicator still runs: the path is exercised on one GPU)
  SSLIC_NCCL_CHECK(ncclAllReduce(e.current_centers(), e.current_centers(),
                                 (size_t)e.centers_count(), ncclFloat64, ncclSum, c->comm,
                                 e.stream()));
}

// int64 deltas as uint64: two's-complement addition is the same operation.
void comm_sum_partials(RankComm* c, Engine& e) {
  if (!c) return;  // (a 1-rank communicator still runs: the path is exercised on one GPU)
  SSLIC_NCCL_CHECK(ncclAllReduce(e.partials(), e.partials(), (size_t)e.partials_count(),
                                 ncclUint64, ncclSum, c->comm, e.stream()));
}

namespace {

RankComm* make_comm(ncclComm_t comm, int rank, int world) {
  auto* c = new RankComm();
  c->comm = comm;
  c->rank = rank;
  c->world = world;
  if (cudaMalloc(&c->scratch, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    comm_destroy(c);
    throw Error(SSLIC_ENOMEM, "device allocation failed (NCCL scratch)");
  }
  return c;
}

// run_slic_rank's communicators, kept for the process lifetime (never
// destroyed: exit-order safe, like the mapped staging in capi.cu)
struct CommCache {
  std::mutex mu;
  std::map<std::string, RankComm*> map;
};
CommCache& comm_cache() {
  static CommCache* c = new CommCache();
  return *c;
}

struct CommOwner {
  RankComm* c = nullptr;
  ~CommOwner() { comm_destroy(c); }
};

struct DevMem {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevMem(size_t bytes, cudaStream_t st) : s(st) {
    SSLIC_CUDA_CHECK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
  }
  ~DevMem() {
    if (p) cudaFreeAsync(p, s);
  }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
};

struct RankStream {
  cudaStream_t s = nullptr;
  explicit RankStream(int device) {
    SSLIC_CUDA_CHECK(cudaSetDevice(device));
    keep_pool_memory(device);  // whole-run calls must not re-map gigabytes each time
    SSLIC_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~RankStream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

__global__ void k_nonfinite(const void* data, int dtype, int64_t n, unsigned long long* out) {
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad += isfinite(load_value(data, dtype, i)) ? 0 : 1;
  for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(out, bad);
}

void check_rank_args(const sslic_image* img, int world) {
  if (world < 1) throw Error(SSLIC_EINVAL, "run_slic: device count must be >= 1");
  if (world > 1 && img->rank != 3)
    throw Error(SSLIC_EINVAL, "multi-GPU run_slic splits 3-D volumes into z-slabs (rank 3)");
  if (world > 1 && img->dims[2] < world)
    throw Error(SSLIC_EINVAL, "multi-GPU run_slic: fewer planes than devices");
}

// One rank's whole run: upload the slab (+ halo) from the host image, engine,
// synced start, iterations with the partials allreduce, slab labels out.
// labels_out: this rank's slab (host). centers/residuals/done: nullable.
void run_rank(const sslic_image* img, const sslic_params* p, int rank, int world, RankComm* comm,
              int device, uint32_t* labels_out, double* centers_out, double* residuals_out,
              int* done_out, int64_t data_first_plane = 0) {
  RankStream st(device);
  const int last_axis = img->rank - 1;
  const int64_t last = img->dims[last_axis];
  int64_t s0 = 0, s1 = last;
  if (world > 1) slab_bounds(last, world, rank, p->grid[last_axis], &s0, &s1);
  const int64_t d0 = std::max<int64_t>(0, s0 - 2), d1 = std::min<int64_t>(last, s1 + 2);
  int64_t plane = 1;
  for (int a = 0; a < last_axis; ++a) plane *= img->dims[a];
  const size_t plane_bytes = (size_t)plane * img->channels * dsize(img->dtype);
  if (d0 < data_first_plane)
    throw Error(SSLIC_EINVAL, "run_slic_rank: host planes must cover the slab plus its halo");
  DevMem dimg((size_t)(d1 - d0) * plane_bytes, st.s);
  copy_to_device(dimg.p,
                 static_cast<const char*>(img->data) + (d0 - data_first_plane) * plane_bytes,
                 (size_t)(d1 - d0) * plane_bytes, device, st.s);
  if (img->dtype == SSLIC_F32 || img->dtype == SSLIC_F64) {  // NDImage checks (image.hpp:238-249)
    DevMem cnt(sizeof(unsigned long long), st.s);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st.s));
    k_nonfinite<<<148 * 4, 256, 0, st.s>>>(dimg.p, img->dtype,
                                           (d1 - d0) * plane * img->channels,
                                           static_cast<unsigned long long*>(cnt.p));
    SSLIC_CUDA_CHECK(cudaGetLastError());
    unsigned long long bad = 0;
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(&bad, cnt.p, sizeof bad, cudaMemcpyDeviceToHost, st.s));
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(st.s));
    if (bad) throw Error(SSLIC_EINVAL, "NDImage: non-finite value");
  }
  sslic_image v = *img;
  v.data = dimg.p;
  for (int a = img->rank; a < kMaxRank; ++a) v.dims[a] = 1;
  Engine e(v, *p, device, s0, s1, d0, d1, st.s);
  comm_sync_value_range(comm, e);
  e.init(true);
  comm_sum_centers(comm, e);
  e.commit();
  const int iters = e.max_iterations();
  for (int it = 0; it < iters; ++it) {
    e.assign(true);
    if (e.dist_mode() && e.undefined_count() > 0)  // slic.hpp:330-331
      throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
    comm_sum_partials(comm, e);
    e.update();
    if (p->has_residual_threshold) {  // identical residuals on every rank
      std::vector<double> rs(e.iterations_done());
      e.residuals_to_host(rs.data(), e.iterations_done());
      if (rs.back() <= p->residual_threshold) break;  // slic.hpp:411
    }
  }
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(st.s));
  if (!e.dist_mode() && e.undefined_seen())
    throw Error(SSLIC_ELOGIC, "accumulate_region: pixel with undefined label");
  const int64_t nv = (s1 - s0) * plane;
  DevMem lab((size_t)nv * sizeof(uint32_t), st.s);
  e.unpack_labels(static_cast<uint32_t*>(lab.p));
  copy_to_host(labels_out, lab.p, (size_t)nv * sizeof(uint32_t), device, st.s);
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(st.s));
  if (centers_out) e.copy_centers_to_host(centers_out);
  if (residuals_out) e.residuals_to_host(residuals_out, e.iterations_done());
  if (done_out) *done_out = e.iterations_done();
}

}  // namespace
}  // namespace sslic_b200

extern "C" {

int sslic_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sslic_nccl_unique_id(void* out, int64_t bytes) {
  return guarded([&] {
    if (!out || bytes < (int64_t)sizeof(ncclUniqueId))
      throw Error(SSLIC_EINVAL, "nccl unique id: buffer smaller than NCCL_UNIQUE_ID_BYTES");
    ncclUniqueId id;
    SSLIC_NCCL_CHECK(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof id);
    return SSLIC_OK;
  });
}

int sslic_slab_bounds(int64_t last, int world, int rank, int64_t align, int64_t* lo,
                      int64_t* hi) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world || last < 1 || align < 1 || !lo || !hi)
      throw Error(SSLIC_EINVAL, "slab_bounds: bad arguments");
    slab_bounds(last, world, rank, align, lo, hi);
    return SSLIC_OK;
  });
}

int sslic_run_slic_multi(const sslic_image* img, const sslic_params* params, int n_devices,
                         const int* devices, uint32_t* labels_out, double* centers_out,
                         double* residuals_out, int* iterations_done) {
  return guarded([&] {
    if (!img || !params || !labels_out || !centers_out)
      throw Error(SSLIC_EINVAL, "run_slic_multi: null argument");
    check_rank_args(img, n_devices);
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw Error(SSLIC_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    std::vector<int> devs(n_devices);
    for (int r = 0; r < n_devices; ++r) {
      devs[r] = devices ? devices[r] : r;
      if (devs[r] < 0 || devs[r] >= count) throw Error(SSLIC_EINVAL, "device index out of range");
    }
    std::vector<ncclComm_t> comms(n_devices);
    SSLIC_NCCL_CHECK(ncclCommInitAll(comms.data(), n_devices, devs.data()));
    std::vector<CommOwner> owners(n_devices);
    for (int r = 0; r < n_devices; ++r) {
      SSLIC_CUDA_CHECK(cudaSetDevice(devs[r]));
      owners[r].c = make_comm(comms[r], r, n_devices);
    }
    const int last_axis = img->rank - 1;
    int64_t plane = 1;
    for (int a = 0; a < last_axis; ++a) plane *= img->dims[a];
    std::vector<int> status(n_devices, SSLIC_OK);
    std::vector<std::string> msg(n_devices);
    std::vector<int> done(n_devices, 0);
    std::once_flag abort_once;
    std::vector<std::thread> th;
    for (int r = 0; r < n_devices; ++r) {
      th.emplace_back([&, r] {
        int64_t s0, s1;
        slab_bounds(img->dims[last_axis], n_devices, r, params->grid[last_axis], &s0, &s1);
        status[r] = guarded([&] {
          run_rank(img, params, r, n_devices, owners[r].c, devs[r], labels_out + s0 * plane,
                   r == 0 ? centers_out : nullptr, r == 0 ? residuals_out : nullptr, &done[r]);
          return SSLIC_OK;
        });
        if (status[r] != SSLIC_OK) {
          msg[r] = last_error();
          // the other ranks may wait in a collective this rank never joins
          std::call_once(abort_once, [&] {
            for (auto& o : owners) {
              ncclCommAbort(o.c->comm);
              o.c->comm = nullptr;
            }
          });
        }
      });
    }
    for (auto& t : th) t.join();
    for (int r = 0; r < n_devices; ++r)
      if (status[r] != SSLIC_OK) throw Error(status[r], msg[r]);
    if (iterations_done) *iterations_done = done[0];
    return SSLIC_OK;
  });
}

int sslic_run_slic_rank(const sslic_image* img, const sslic_params* params, int rank, int world,
                        const void* nccl_id, int device, int64_t data_first_plane,
                        uint32_t* labels_out, double* centers_out, double* residuals_out,
                        int* iterations_done) {
  return guarded([&] {
    if (!img || !params || !labels_out) throw Error(SSLIC_EINVAL, "run_slic_rank: null argument");
    if (rank < 0 || rank >= world) throw Error(SSLIC_EINVAL, "run_slic_rank: bad rank");
    check_rank_args(img, world);
    if (world > 1 && !nccl_id) throw Error(SSLIC_EINVAL, "run_slic_rank: null NCCL unique id");
    if (data_first_plane < 0) throw Error(SSLIC_EINVAL, "run_slic_rank: negative first plane");
    RankComm* comm = nullptr;
    if (nccl_id) {
      // Communicators are cached per (unique id, rank, world, device) for the
      // life of the process: repeated calls with the same id (one job's
      // successive volumes) skip ncclCommInitRank. A new id makes a new one.
      SSLIC_CUDA_CHECK(cudaSetDevice(device));
      std::string key(static_cast<const char*>(nccl_id), sizeof(ncclUniqueId));
      key += std::to_string(rank) + "/" + std::to_string(world) + "@" + std::to_string(device);
      std::lock_guard<std::mutex> lk(comm_cache().mu);
      auto it = comm_cache().map.find(key);
      if (it == comm_cache().map.end()) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof id);
        ncclComm_t c;
        SSLIC_NCCL_CHECK(ncclCommInitRank(&c, world, id, rank));
        it = comm_cache().map.emplace(key, make_comm(c, rank, world)).first;
      }
      comm = it->second;
    }
    run_rank(img, params, rank, world, comm, device, labels_out, centers_out, residuals_out,
             iterations_done, data_first_plane);
    return SSLIC_OK;
  });
}

int sslic_engine_attach_nccl(sslic_engine* e, const void* nccl_id, int rank, int world) {
  return guarded([&] {
    if (!e || rank < 0 || rank >= world) throw Error(SSLIC_EINVAL, "attach_nccl: bad arguments");
    comm_destroy(e->comm);
    e->comm = nullptr;
    if (!nccl_id) {
      if (world > 1) throw Error(SSLIC_EINVAL, "attach_nccl: null NCCL unique id");
      return SSLIC_OK;  // detached
    }
    SSLIC_CUDA_CHECK(cudaSetDevice(e->e->device()));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    ncclComm_t comm;
    SSLIC_NCCL_CHECK(ncclCommInitRank(&comm, world, id, rank));
    e->comm = make_comm(comm, rank, world);
    return SSLIC_OK;
  });
}

int sslic_engine_start(sslic_engine* e) {
  return guarded([&] {
    Engine& en = *e->e;
    SSLIC_CUDA_CHECK(cudaSetDevice(en.device()));
    comm_sync_value_range(e->comm, en);
    en.init(true);
    comm_sum_centers(e->comm, en);
    en.commit();
    return SSLIC_OK;
  });
}

}  // extern "C"
