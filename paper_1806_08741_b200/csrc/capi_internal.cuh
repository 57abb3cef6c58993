// Shared by the C ABI translation units: status/exception mapping and the
// thread's last error message (sslic_last_error).
#pragma once

#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "engine.cuh"

namespace sslic_b200 {

std::string& last_error();  // thread-local, defined in capi.cu

template <class F>
int guarded(F&& f) {
  try {
    last_error().clear();
    return f();
  } catch (const Error& e) {
    last_error() = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    last_error() = "host allocation failed";
    return SSLIC_ENOMEM;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return SSLIC_EINVAL;
  }
}

// Z-slab of `rank` among `world` ranks along the last axis, rounded to
// multiples of `align` planes when there are at least `world` such units
// (paper_1806_08741_b200/sharded.py slab_bounds is the same split).
inline void slab_bounds(int64_t last, int world, int rank, int64_t align, int64_t* lo,
                        int64_t* hi) {
  int64_t units = (last + align - 1) / align;
  if (units < world) {
    align = 1;
    units = last;
  }
  *lo = std::min(units * rank / world * align, last);
  *hi = std::min(units * (rank + 1) / world * align, last);
}

// Host <-> device copies that stripe large PAGEABLE buffers over host threads
// and pinned staging (hostcopy.cu); small or pinned buffers: cudaMemcpyAsync.
void copy_to_device(void* dev, const void* host, size_t bytes, int device, cudaStream_t s);
void copy_to_host(void* host, const void* dev, size_t bytes, int device, cudaStream_t s);

// Keep freed device memory in the stream-ordered pool across calls (capi.cu).
void keep_pool_memory(int device);

// Output files of the fused final pass (io.cu).
void write_labels_counted(const char* path, int rank, const int64_t* dims,
                          const uint32_t* labels, uint64_t count);
void write_contour_f32(const char* path, const sslic_image* img, const uint32_t* boundary);

// NCCL plumbing (multi.cu): one communicator per engine/rank. The engine's
// collective steps -- the value-range MAX before init, the SUM of the init
// tables, the SUM of the int64 per-cluster partials every iteration -- run
// on the engine's stream (capturable in a CUDA graph).
struct RankComm;
void comm_destroy(RankComm* c);
void comm_sync_value_range(RankComm* c, Engine& e);
void comm_sum_centers(RankComm* c, Engine& e);
void comm_sum_partials(RankComm* c, Engine& e);

}  // namespace sslic_b200

// The C ABI's engine handle (include/sslic_b200.h).
struct sslic_engine {
  std::unique_ptr<sslic_b200::Engine> e;
  sslic_b200::RankComm* comm = nullptr;  // attached NCCL communicator (owned)
  ~sslic_engine() { sslic_b200::comm_destroy(comm); }
};

