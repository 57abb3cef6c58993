// Large transfers between PAGEABLE host memory and the device.
//
// A caller of the reference holds its image and label map in ordinary
// (pageable) memory -- std::vector storage behind NDImage / LabelMap
// (image.hpp:236-338). cudaMemcpy stages such memory through one driver
// buffer on one thread, 4-6 GB/s on this box; the 52 GB image and the 70 GB
// label map of config 5 spent 26 of the call's 40 s there. Here the transfer
// is cut into stripes, one host thread per stripe (up to 16): each thread moves its
// stripe through two pinned 8 MiB buffers on its own stream (memcpy into one
// buffer while the DMA drains the other), so the host-side copies run in
// parallel and the link stays busy. Pinned or small buffers keep the plain
// cudaMemcpyAsync.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "capi_internal.cuh"

namespace sslic_b200 {
namespace {

constexpr size_t kStageBytes = (size_t)8 << 20;   // per pinned buffer
constexpr size_t kLargeCopy = (size_t)32 << 20;   // below this: plain cudaMemcpyAsync
constexpr int kMaxThreads = 16;

// Process-wide pinned staging (2 buffers per worker), allocated on first use
// and kept (never freed: exit-order safe); one large copy at a time.
struct Staging {
  std::mutex mu;
  void* buf[kMaxThreads][2] = {};
  bool ok = false;
  bool tried = false;
  bool ensure() {
    if (tried) return ok;
    tried = true;
    for (int t = 0; t < kMaxThreads; ++t)
      for (int b = 0; b < 2; ++b)
        if (cudaHostAlloc(&buf[t][b], kStageBytes, cudaHostAllocPortable) != cudaSuccess) {
          cudaGetLastError();
          return ok = false;
        }
    return ok = true;
  }
};
Staging& staging() {
  static Staging* s = new Staging();
  return *s;
}

bool pageable(const void* p) {
  if (std::getenv("SSLIC_NO_STRIPED_COPY") != nullptr) return false;  // (A/B: the driver's staging)
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int worker_count(size_t bytes) {
  int t = (int)std::thread::hardware_concurrency();
  t = t < 1 ? 1 : std::min(t, kMaxThreads);  // (measured: D2H 151 ms at 8 threads, 119 ms at 16)
  if (const char* e = std::getenv("SSLIC_COPY_THREADS")) t = std::max(1, std::min(std::atoi(e), kMaxThreads));
  const size_t per = (size_t)4 * kStageBytes;  // at least a few chunks per worker
  return (int)std::max<size_t>(1, std::min<size_t>((size_t)t, bytes / per));
}

// One worker's stripe [off, off + len), double-buffered through its two
// pinned buffers on its own stream.
struct Worker {
  int device;
  void* stage[2];
  cudaStream_t s = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaError_t err = cudaSuccess;
  bool open(cudaEvent_t after) {
    if ((err = cudaSetDevice(device)) != cudaSuccess) return false;
    if ((err = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return false;
    for (auto& e : ev)
      if ((err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming)) != cudaSuccess) return false;
    // everything queued on the caller's stream so far (allocation, producer kernels)
    return (err = cudaStreamWaitEvent(s, after, 0)) == cudaSuccess;
  }
  void close() {
    if (s) cudaStreamSynchronize(s);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
  }
  void h2d(char* dev, const char* host, size_t len) {
    int b = 0;
    bool used[2] = {false, false};
    for (size_t o = 0; o < len && err == cudaSuccess; o += kStageBytes, b ^= 1) {
      const size_t n = std::min(kStageBytes, len - o);
      if (used[b] && (err = cudaEventSynchronize(ev[b])) != cudaSuccess) break;
      std::memcpy(stage[b], host + o, n);
      if ((err = cudaMemcpyAsync(dev + o, stage[b], n, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        break;
      err = cudaEventRecord(ev[b], s);
      used[b] = true;
    }
  }
  void d2h(char* host, const char* dev, size_t len) {
    // chunk i + 1 is in flight while chunk i is copied out of its buffer
    const size_t chunks = (len + kStageBytes - 1) / kStageBytes;
    auto issue = [&](size_t i) {
      const size_t o = i * kStageBytes, n = std::min(kStageBytes, len - o);
      const int b = (int)(i & 1);
      if ((err = cudaMemcpyAsync(stage[b], dev + o, n, cudaMemcpyDeviceToHost, s)) == cudaSuccess)
        err = cudaEventRecord(ev[b], s);
    };
    if (chunks) issue(0);
    for (size_t i = 0; i < chunks && err == cudaSuccess; ++i) {
      const int b = (int)(i & 1);
      if ((err = cudaEventSynchronize(ev[b])) != cudaSuccess) break;
      if (i + 1 < chunks) issue(i + 1);  // the other buffer is free (copied out last round)
      const size_t o = i * kStageBytes, n = std::min(kStageBytes, len - o);
      std::memcpy(host + o, stage[b], n);
    }
  }
};

void striped(bool to_device, void* dev, void* host, size_t bytes, int device, cudaStream_t s) {
  Staging& st = staging();
  std::lock_guard<std::mutex> lk(st.mu);
  if (!st.ensure()) {  // no pinned memory to be had: the driver's own staging
    SSLIC_CUDA_CHECK(to_device
                         ? cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s)
                         : cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
    if (!to_device) SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  cudaEvent_t after = nullptr;
  SSLIC_CUDA_CHECK(cudaEventCreateWithFlags(&after, cudaEventDisableTiming));
  SSLIC_CUDA_CHECK(cudaEventRecord(after, s));
  const int T = worker_count(bytes);
  std::vector<Worker> w(T);
  std::vector<std::thread> th;
  // stripes on 256-byte boundaries
  const size_t unit = 256, units = (bytes + unit - 1) / unit;
  for (int t = 0; t < T; ++t) {
    w[t].device = device;
    w[t].stage[0] = st.buf[t][0];
    w[t].stage[1] = st.buf[t][1];
    const size_t a = std::min(bytes, units * t / T * unit);
    const size_t b = std::min(bytes, units * (t + 1) / T * unit);
    th.emplace_back([&, t, a, b] {
      Worker& me = w[t];
      if (me.open(after)) {
        if (to_device) me.h2d(static_cast<char*>(dev) + a, static_cast<const char*>(host) + a, b - a);
        else me.d2h(static_cast<char*>(host) + a, static_cast<const char*>(dev) + a, b - a);
      }
      // H2D: the caller's stream must see the stripe before it goes on
      if (me.err == cudaSuccess && to_device && me.s) {
        cudaEvent_t done = nullptr;
        if ((me.err = cudaEventCreateWithFlags(&done, cudaEventDisableTiming)) == cudaSuccess) {
          me.err = cudaEventRecord(done, me.s);
          if (me.err == cudaSuccess) me.err = cudaStreamWaitEvent(s, done, 0);
          cudaEventDestroy(done);  // (released once the recorded work completes)
        }
      }
      me.close();
    });
  }
  for (auto& x : th) x.join();
  cudaEventDestroy(after);
  for (auto& x : w)
    if (x.err != cudaSuccess) {
      cudaGetLastError();
      throw Error(SSLIC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(x.err) +
                                   " (striped host copy)");
    }
}

}  // namespace

// Host -> device on stream `s`. Returns once the host buffer has been read
// (like cudaMemcpyAsync from pageable memory); the data is visible to work
// queued on `s` afterwards.
void copy_to_device(void* dev, const void* host, size_t bytes, int device, cudaStream_t s) {
  if (bytes < kLargeCopy || !pageable(host)) {
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  striped(true, dev, const_cast<void*>(host), bytes, device, s);
}

// Device -> host after everything queued on `s` so far. The host buffer is
// complete on return for pageable destinations; pinned ones follow stream
// order as with cudaMemcpyAsync (the caller synchronises `s`).
void copy_to_host(void* host, const void* dev, size_t bytes, int device, cudaStream_t s) {
  if (bytes < kLargeCopy || !pageable(host)) {
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s));
    return;
  }
  striped(false, const_cast<void*>(dev), host, bytes, device, s);
}

}  // namespace sslic_b200
