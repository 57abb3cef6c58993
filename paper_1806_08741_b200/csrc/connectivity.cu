// Connectivity enforcement (connectivity.hpp:125-273).
//
// Device part: face-connected component labelling of the label map by a
// lock-free union-find (atomicMin hooking, roots = smallest flat offset of
// each component), component sizes, and finalize_cluster_components
// (connectivity.hpp:125-173) as one thread per cluster: seed search, then
// "component of the seed is final if size > floor(prod S / 4)".
//
// Sweep part: sweep_relabel (connectivity.hpp:182-261) is a single-threaded
// raster recurrence whose fills see the labels written by earlier steps; it
// runs on the host over the device-computed marker map, exactly as the
// reference orders it (see DESIGN.md "Connectivity" for the status).
#include <cstring>
#include <vector>

#include "connectivity.cuh"

namespace sslic_b200 {

namespace {

__device__ __forceinline__ uint32_t find_root(const uint32_t* parent, uint32_t i) {
  uint32_t p = parent[i];
  while (p != i) {
    i = p;
    p = parent[i];
  }
  return i;
}

__device__ __forceinline__ void unite(uint32_t* parent, uint32_t a, uint32_t b) {
  for (;;) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a < b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMin(parent + a, b);
    if (old == a) return;
    a = old;
  }
}

__global__ void k_cc_init(uint32_t* parent, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) parent[i] = (uint32_t)i;
}

__global__ void k_cc_union(Geom g, const uint32_t* labels, uint32_t* parent, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t l = labels[i];
  int64_t rem = i;
  for (int a = 0; a < g.rank; ++a) {
    const int64_t c = rem % g.dims[a];
    rem /= g.dims[a];
    if (c + 1 < g.dims[a]) {
      const int64_t j = i + g.strides[a];
      if (labels[j] == l) unite(parent, (uint32_t)i, (uint32_t)j);
    }
  }
}

__global__ void k_cc_flatten(uint32_t* parent, unsigned* sizes, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t r = find_root(parent, (uint32_t)i);
  parent[i] = r;
  atomicAdd(sizes + r, 1u);
}

// finalize_cluster_components (connectivity.hpp:125-173), one thread per k.
__global__ void k_finalize(Geom g, const uint32_t* labels, const double* centers,
                           const uint32_t* root, const unsigned* sizes, int64_t min_size,
                           uint8_t* final_root) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= g.k) return;
  int64_t anchor[kMaxRank], aoff = 0;
  for (int a = 0; a < g.rank; ++a) {
    int64_t v = llround(centers[id * g.stride + g.channels + a]);
    v = v < 0 ? 0 : (v > g.dims[a] - 1 ? g.dims[a] - 1 : v);
    anchor[a] = v;
    aoff += v * g.strides[a];
  }
  int64_t seed = -1;
  if (labels[aoff] == (uint32_t)id) {
    seed = aoff;
  } else {
    int64_t lo[kMaxRank], hi[kMaxRank], cur[kMaxRank];
    bool empty = false;
    for (int a = 0; a < g.rank; ++a) {
      int64_t l = anchor[a] - g.grid[a] / 2, h = l + g.grid[a];
      l = l < 0 ? 0 : (l > g.dims[a] ? g.dims[a] : l);
      h = h < l ? l : (h > g.dims[a] ? g.dims[a] : h);
      lo[a] = l;
      hi[a] = h - 1;
      if (hi[a] < lo[a]) empty = true;
      cur[a] = lo[a];
    }
    while (!empty) {
      int64_t off = 0;
      for (int a = 0; a < g.rank; ++a) off += cur[a] * g.strides[a];
      if (labels[off] == (uint32_t)id) {
        seed = off;
        break;
      }
      int a = 0;
      for (; a < g.rank; ++a) {
        if (++cur[a] <= hi[a]) break;
        cur[a] = lo[a];
      }
      if (a == g.rank) break;
    }
  }
  if (seed < 0) return;
  const uint32_t r = root[seed];
  if ((int64_t)sizes[r] > min_size) final_root[r] = 1;
}

__global__ void k_markers(const uint32_t* root, const uint8_t* final_root, uint8_t* markers,
                          int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) markers[i] = final_root[root[i]];
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

// sweep_relabel (connectivity.hpp:182-261): raster order over non-final
// pixels; fills see earlier relabels.
uint32_t sweep_host(const Geom& g, std::vector<uint32_t>& labels, std::vector<uint8_t>& markers,
                    int64_t min_size, uint32_t k_start) {
  const int64_t n = (int64_t)labels.size();
  std::vector<uint8_t> visited(n, 0);
  std::vector<int64_t> comp, stack;
  uint32_t next_label = k_start;
  int64_t coord[kMaxRank];
  auto decode = [&](int64_t off) {
    for (int a = 0; a < g.rank; ++a) {
      coord[a] = off % g.dims[a];
      off /= g.dims[a];
    }
  };
  for (int64_t off = 0; off < n; ++off) {
    if (markers[off]) continue;
    const uint32_t label = labels[off];
    comp.clear();
    stack.clear();
    stack.push_back(off);
    visited[off] = 1;
    while (!stack.empty()) {
      const int64_t o = stack.back();
      stack.pop_back();
      comp.push_back(o);
      decode(o);
      for (int a = 0; a < g.rank; ++a) {
        if (coord[a] > 0) {
          const int64_t nb = o - g.strides[a];
          if (!visited[nb] && labels[nb] == label) {
            visited[nb] = 1;
            stack.push_back(nb);
          }
        }
        if (coord[a] + 1 < g.dims[a]) {
          const int64_t nb = o + g.strides[a];
          if (!visited[nb] && labels[nb] == label) {
            visited[nb] = 1;
            stack.push_back(nb);
          }
        }
      }
    }
    for (int64_t o : comp) visited[o] = 0;
    if ((int64_t)comp.size() > min_size) {
      for (int64_t o : comp) {
        labels[o] = next_label;
        markers[o] = 1;
      }
      ++next_label;
      continue;
    }
    int64_t best_before = -1, best_after = -1, best_pending = -1;
    uint32_t label_before = 0, label_after = 0, label_pending = 0;
    for (int64_t o : comp) {
      decode(o);
      for (int a = 0; a < g.rank; ++a) {
        for (int dir = -1; dir <= 1; dir += 2) {
          const int64_t c = coord[a] + dir;
          if (c < 0 || c >= g.dims[a]) continue;
          const int64_t adj = o + dir * g.strides[a];
          if (labels[adj] == label) continue;
          if (markers[adj]) {
            if (adj < off) {
              if (adj > best_before) {
                best_before = adj;
                label_before = labels[adj];
              }
            } else if (best_after < 0 || adj < best_after) {
              best_after = adj;
              label_after = labels[adj];
            }
          } else if (best_pending < 0 || adj < best_pending) {
            best_pending = adj;
            label_pending = labels[adj];
          }
        }
      }
    }
    if (best_before >= 0 || best_after >= 0) {
      const uint32_t target = best_before >= 0 ? label_before : label_after;
      for (int64_t o : comp) {
        labels[o] = target;
        markers[o] = 1;
      }
    } else if (best_pending >= 0) {
      for (int64_t o : comp) labels[o] = label_pending;
    } else {
      for (int64_t o : comp) {
        labels[o] = next_label;
        markers[o] = 1;
      }
      ++next_label;
    }
  }
  return next_label;
}

}  // namespace

uint32_t enforce_connectivity_device(const Geom& g, const uint32_t* labels_in,
                                     const double* centers, uint32_t* labels_out,
                                     cudaStream_t s) {
  int64_t n = 1;
  for (int a = 0; a < g.rank; ++a) n *= g.dims[a];
  if (n >= (int64_t)0xffffffffLL)
    throw Error(SSLIC_EINVAL, "enforce_connectivity: volumes >= 2^32 voxels are not supported yet");
  int64_t min_size = 1;
  for (int a = 0; a < g.rank; ++a) min_size *= g.grid[a];
  min_size /= 4;  // size_threshold (connectivity.hpp:34-38)

  uint32_t* parent = nullptr;
  unsigned* sizes = nullptr;
  uint8_t *final_root = nullptr, *markers = nullptr;
  SSLIC_CUDA_CHECK(cudaMallocAsync(&parent, n * sizeof(uint32_t), s));
  SSLIC_CUDA_CHECK(cudaMallocAsync(&sizes, n * sizeof(unsigned), s));
  SSLIC_CUDA_CHECK(cudaMallocAsync(&final_root, n, s));
  SSLIC_CUDA_CHECK(cudaMallocAsync(&markers, n, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(sizes, 0, n * sizeof(unsigned), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(final_root, 0, n, s));
  k_cc_init<<<nblk(n), 256, 0, s>>>(parent, n);
  k_cc_union<<<nblk(n), 256, 0, s>>>(g, labels_in, parent, n);
  k_cc_flatten<<<nblk(n), 256, 0, s>>>(parent, sizes, n);
  if (g.k > 0)
    k_finalize<<<nblk(g.k), 256, 0, s>>>(g, labels_in, centers, parent, sizes, min_size,
                                         final_root);
  k_markers<<<nblk(n), 256, 0, s>>>(parent, final_root, markers, n);
  SSLIC_CUDA_CHECK(cudaGetLastError());

  std::vector<uint32_t> h_labels(n);
  std::vector<uint8_t> h_markers(n);
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(h_labels.data(), labels_in, n * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, s));
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(h_markers.data(), markers, n, cudaMemcpyDeviceToHost, s));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
  const uint32_t next = sweep_host(g, h_labels, h_markers, min_size, (uint32_t)g.k);
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out, h_labels.data(), n * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, s));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFreeAsync(parent, s);
  cudaFreeAsync(sizes, s);
  cudaFreeAsync(final_root, s);
  cudaFreeAsync(markers, s);
  return next;
}

}  // namespace sslic_b200
