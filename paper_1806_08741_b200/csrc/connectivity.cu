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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
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
// pixels; fills see earlier relabels. Host, single-threaded by definition of
// the recurrence; fills carry coordinates (no div/mod per voxel). Any fill order gives the same component set,
// and the merge-target search is a max/min over it, so the visiting order
// does not affect the result.
struct Vox {
  int64_t off;
  int32_t c[3];
};

uint32_t sweep_host(const Geom& g, uint32_t* labels, uint8_t* markers, int64_t n,
                    int64_t min_size, uint32_t k_start) {
  const int rank = g.rank;
  int64_t dim[3] = {1, 1, 1}, str[3] = {0, 0, 0};
  for (int a = 0; a < rank; ++a) {
    dim[a] = g.dims[a];
    str[a] = g.strides[a];
  }
  // markers: bit 0 = final (the reference's MarkerMap), bit 1 = visited by
  // the current fill (one array: one page walk per neighbour instead of two)
  uint8_t* const mk = markers;
  std::vector<Vox> comp;
  comp.reserve(1 << 16);
  uint32_t next_label = k_start;
  int64_t off = 0;
  // raster coordinates of `off`, advanced incrementally (no 64-bit div/mod
  // per event unless the scan jumps more than a row)
  int64_t cx = 0, cy = 0, cz = 0, prev = 0;
  while (off < n) {
    // next unmarked voxel (short runs: a byte loop beats memchr's call cost)
    while (off < n && markers[off]) ++off;
    if (off >= n) break;
    {
      const int64_t d = off - prev;
      if (d < dim[0] - cx) {
        cx += d;
      } else {
        int64_t r = off;
        cx = r % dim[0];
        r /= dim[0];
        cy = r % dim[1];
        cz = r / dim[1];
      }
      prev = off;
    }
    const uint32_t label = labels[off];
    // one pass: the fill (same label, face-connected, marks ignored as in
    // scanline_fill) and, from its boundary, the merge candidates
    int64_t best_before = -1, best_after = -1, best_pending = -1;
    uint32_t label_before = 0, label_after = 0, label_pending = 0;
    comp.clear();
    {
      Vox v;
      v.off = off;
      v.c[0] = (int32_t)cx;
      v.c[1] = (int32_t)cy;
      v.c[2] = (int32_t)cz;
      comp.push_back(v);
      mk[off] |= 2;
    }
    // explicit face neighbours (predictable control flow, no inner axis loops)
    auto visit = [&](const Vox& v, int64_t adj, int a, int32_t c) {
      const uint32_t la = labels[adj];
      const uint8_t m = mk[adj];
      if (la == label) {
        if (!(m & 2)) {
          mk[adj] = m | 2;
          Vox w = v;
          w.off = adj;
          w.c[a] = c;
          comp.push_back(w);
        }
      } else if (m & 1) {
        if (adj < off) {
          if (adj > best_before) {
            best_before = adj;
            label_before = la;
          }
        } else if (best_after < 0 || adj < best_after) {
          best_after = adj;
          label_after = la;
        }
      } else if (best_pending < 0 || adj < best_pending) {
        best_pending = adj;
        label_pending = la;
      }
    };
    for (size_t head = 0; head < comp.size(); ++head) {
      const Vox v = comp[head];
      if (v.c[0] > 0) visit(v, v.off - 1, 0, v.c[0] - 1);
      if (v.c[0] + 1 < dim[0]) visit(v, v.off + 1, 0, v.c[0] + 1);
      if (rank > 1) {
        if (v.c[1] > 0) visit(v, v.off - str[1], 1, v.c[1] - 1);
        if (v.c[1] + 1 < dim[1]) visit(v, v.off + str[1], 1, v.c[1] + 1);
      }
      if (rank > 2) {
        if (v.c[2] > 0) visit(v, v.off - str[2], 2, v.c[2] - 1);
        if (v.c[2] + 1 < dim[2]) visit(v, v.off + str[2], 2, v.c[2] + 1);
      }
    }
    uint32_t target;
    uint8_t mark = 1;
    if ((int64_t)comp.size() > min_size) {
      target = next_label++;
    } else if (best_before >= 0 || best_after >= 0) {
      target = best_before >= 0 ? label_before : label_after;
    } else if (best_pending >= 0) {
      target = label_pending;  // adopt the pending label, stay unmarked
      mark = 0;
    } else {
      target = next_label++;
    }
    for (const Vox& v : comp) {
      labels[v.off] = target;
      mk[v.off] = (uint8_t)((mk[v.off] & 1) | mark);
    }
    ++off;
  }
  return next_label;
}

// The same recurrence over packed words: label | final << 31 | visited << 30
// (one array: each neighbour probe touches one cache line instead of two;
// used when every label, fresh ones included, stays below 2^30).
constexpr uint32_t kFin = 1u << 31, kVis = 1u << 30, kLab = kVis - 1u;
uint32_t sweep_host_packed(const Geom& g, uint32_t* w, int64_t n, int64_t min_size,
                           uint32_t k_start) {
  const int rank = g.rank;
  int64_t dim[3] = {1, 1, 1}, str[3] = {0, 0, 0};
  for (int a = 0; a < rank; ++a) {
    dim[a] = g.dims[a];
    str[a] = g.strides[a];
  }
  std::vector<Vox> comp;
  comp.reserve(1 << 16);
  uint32_t next_label = k_start;
  int64_t off = 0;
  int64_t cx = 0, cy = 0, cz = 0, prev = 0;
  while (off < n) {
    while (off < n && (w[off] & kFin)) ++off;
    if (off >= n) break;
    {
      const int64_t d = off - prev;
      if (d < dim[0] - cx) {
        cx += d;
      } else {
        int64_t r = off;
        cx = r % dim[0];
        r /= dim[0];
        cy = r % dim[1];
        cz = r / dim[1];
      }
      prev = off;
    }
    const uint32_t label = w[off] & kLab;
    int64_t best_before = -1, best_after = -1, best_pending = -1;
    uint32_t label_before = 0, label_after = 0, label_pending = 0;
    comp.clear();
    {
      Vox v;
      v.off = off;
      v.c[0] = (int32_t)cx;
      v.c[1] = (int32_t)cy;
      v.c[2] = (int32_t)cz;
      comp.push_back(v);
      w[off] |= kVis;
    }
    auto visit = [&](const Vox& v, int64_t adj, int a, int32_t c) {
      const uint32_t wa = w[adj];
      const uint32_t la = wa & kLab;
      if (la == label) {
        if (!(wa & kVis)) {
          w[adj] = wa | kVis;
          Vox u = v;
          u.off = adj;
          u.c[a] = c;
          comp.push_back(u);
        }
      } else if (wa & kFin) {
        if (adj < off) {
          if (adj > best_before) {
            best_before = adj;
            label_before = la;
          }
        } else if (best_after < 0 || adj < best_after) {
          best_after = adj;
          label_after = la;
        }
      } else if (best_pending < 0 || adj < best_pending) {
        best_pending = adj;
        label_pending = la;
      }
    };
    for (size_t head = 0; head < comp.size(); ++head) {
      const Vox v = comp[head];
      if (v.c[0] > 0) visit(v, v.off - 1, 0, v.c[0] - 1);
      if (v.c[0] + 1 < dim[0]) visit(v, v.off + 1, 0, v.c[0] + 1);
      if (rank > 1) {
        if (v.c[1] > 0) visit(v, v.off - str[1], 1, v.c[1] - 1);
        if (v.c[1] + 1 < dim[1]) visit(v, v.off + str[1], 1, v.c[1] + 1);
      }
      if (rank > 2) {
        if (v.c[2] > 0) visit(v, v.off - str[2], 2, v.c[2] - 1);
        if (v.c[2] + 1 < dim[2]) visit(v, v.off + str[2], 2, v.c[2] + 1);
      }
    }
    uint32_t target;
    uint32_t fin = kFin;
    if ((int64_t)comp.size() > min_size) {
      target = next_label++;
    } else if (best_before >= 0 || best_after >= 0) {
      target = best_before >= 0 ? label_before : label_after;
    } else if (best_pending >= 0) {
      target = label_pending;  // adopt the pending label, stay unmarked
      fin = 0;
    } else {
      target = next_label++;
    }
    for (const Vox& v : comp) w[v.off] = target | (w[v.off] & kFin) | fin;
    ++off;
  }
  return next_label;
}

__global__ void k_pack_flags(const uint32_t* labels, const uint8_t* markers, uint32_t* out,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = labels[i] | (markers[i] ? kFin : 0u);
}
__global__ void k_unpack_flags(const uint32_t* in, uint32_t* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] & kLab;
}
__global__ void k_max_label(const uint32_t* labels, int64_t n, unsigned* out) {
  uint32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, labels[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
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

  // packed path: every label below 2^30, fresh ones included (at most one
  // per component larger than min_size, plus one)
  bool packed = false;
  {
    const int64_t fresh = n / (min_size + 1) + 2;
    if ((int64_t)g.k + fresh < (int64_t)kVis) {
      SSLIC_CUDA_CHECK(cudaMemsetAsync(sizes, 0, sizeof(unsigned), s));
      k_max_label<<<148 * 8, 256, 0, s>>>(labels_in, n, sizes);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      unsigned mx = 0;
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(&mx, sizes, sizeof(mx), cudaMemcpyDeviceToHost, s));
      SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
      packed = mx < kVis && (int64_t)mx + fresh < (int64_t)kVis;
    }
  }
  if (packed) {  // (parent is free after k_markers)
    k_pack_flags<<<148 * 8, 256, 0, s>>>(labels_in, markers, parent, n);
    SSLIC_CUDA_CHECK(cudaGetLastError());
  }
  const auto tc0 = std::chrono::steady_clock::now();
  // host staging (labels + markers) for the sweep: 2 MB transparent huge
  // pages (the fills touch neighbouring planes megabytes apart; 4 KB pages
  // would make nearly every z-neighbour a TLB miss), then pinned for the copies
  const size_t host_bytes = ((size_t)n * (sizeof(uint32_t) + 1) + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1);
  uint8_t* host = nullptr;
  if (posix_memalign(reinterpret_cast<void**>(&host), 2u << 20, host_bytes) != 0)
    throw Error(SSLIC_ENOMEM, "enforce_connectivity: host staging");
  madvise(host, host_bytes, MADV_HUGEPAGE);
  const bool pinned = cudaHostRegister(host, host_bytes, cudaHostRegisterDefault) == cudaSuccess;
  if (!pinned) cudaGetLastError();
  uint32_t* h_labels = reinterpret_cast<uint32_t*>(host);
  uint8_t* h_markers = host + (size_t)n * sizeof(uint32_t);
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(h_labels, packed ? parent : labels_in,
                                   n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  if (!packed)
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(h_markers, markers, n, cudaMemcpyDeviceToHost, s));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
  const auto tc1 = std::chrono::steady_clock::now();
  uint32_t next = 0;
  try {
    next = packed ? sweep_host_packed(g, h_labels, n, min_size, (uint32_t)g.k)
                  : sweep_host(g, h_labels, h_markers, n, min_size, (uint32_t)g.k);
  } catch (...) {
    if (pinned) cudaHostUnregister(host);
    std::free(host);
    throw;
  }
  const auto tc2 = std::chrono::steady_clock::now();
  if (packed) {
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(parent, h_labels, n * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, s));
    k_unpack_flags<<<148 * 8, 256, 0, s>>>(parent, labels_out, n);
    SSLIC_CUDA_CHECK(cudaGetLastError());
  } else {
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out, h_labels, n * sizeof(uint32_t),
                                     cudaMemcpyHostToDevice, s));
  }
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
  if (pinned) cudaHostUnregister(host);
  std::free(host);
  if (std::getenv("SSLIC_TIMING")) {
    const auto tc3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[sslic] connectivity: device CCL+finalize+D2H %.1f ms, host sweep%s %.1f ms, H2D %.1f ms\n",
                 ms(tc0, tc1), packed ? " (packed)" : "", ms(tc1, tc2), ms(tc2, tc3));
  }
  cudaFreeAsync(parent, s);
  cudaFreeAsync(sizes, s);
  cudaFreeAsync(final_root, s);
  cudaFreeAsync(markers, s);
  return next;
}

}  // namespace sslic_b200
