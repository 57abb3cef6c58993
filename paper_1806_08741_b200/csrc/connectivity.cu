// Connectivity enforcement (connectivity.hpp:125-273), entirely on the device.
//
// 1. Face-connected component labelling of the label map: lock-free
//    union-find (atomicMin hooking; a component's root is its smallest flat
//    offset), then the components are numbered densely in root order, so a
//    node id orders components exactly like the raster sweep reaches them.
// 2. finalize_cluster_components (connectivity.hpp:125-173): one thread per
//    cluster (seed search, "final if size > floor(prod S / 4)").
// 3. sweep_relabel (connectivity.hpp:182-261) as a fixpoint over the
//    component graph instead of a raster recurrence:
//    * every non-final component C is an event at time root(C); its fill is C
//      itself unless an earlier merge gave a neighbour C's label;
//    * a small component merges into the component holding its largest
//      neighbour offset below root(C) (all such pixels are final by then), so
//      its final label is that component's final label (a static pointer);
//    * a fill can only grow through a neighbour that took label L = label(C)
//      by merging into the finalized component F_L; such a fill reaches F_L,
//      so it is fresh. This happens at most once per L, at the earliest such
//      event te(L); the fill also swallows the not-yet-swept L-fragments
//      adjacent to F_L's merged region ("absorbed");
//    * te(L) and the absorbed sets depend only on earlier events, so Jacobi
//      rounds (pointer jumping, one pass over the face edges) converge to the
//      unique fixpoint, which equals the sequential sweep's outcome;
//    * fresh ids are numbered by a prefix sum over events in root order.
//    A pending adoption (no finalized neighbour at all) can only start at
//    offset 0; the cascade it opens is emulated exactly by one device thread
//    until no pending pixel remains, then the fixpoint takes over. Label maps
//    holding ids >= k (never produced by run_slic) are swept entirely by that
//    device thread, because fresh ids could then collide with input labels.
#include <cub/device/device_scan.cuh>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "connectivity.cuh"

namespace sslic_b200 {

namespace {

constexpr uint32_t kNone = 0xffffffffu;

// node flags
constexpr uint8_t kFin = 1;     // finalized by finalize_cluster_components
constexpr uint8_t kFresh = 2;   // larger than min_size (or the whole image)
constexpr uint8_t kProc = 4;    // decided by the sequential prefix
constexpr uint8_t kFixed = 8;   // final label fixed by the prefix (flab)
constexpr uint8_t kAbs = 16;    // absorbed by the extension fill of its label

struct CG {
  int rank;
  uint32_t dims[kMaxRank];
  uint32_t strides[kMaxRank];
  uint32_t n;
};

__device__ __forceinline__ void decode(const CG& g, uint32_t p, uint32_t* c) {
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a < g.rank) {
      c[a] = p % g.dims[a];
      p /= g.dims[a];
    }
  }
}

// Calls f(q) for every face neighbour q of p.
template <class F>
__device__ __forceinline__ void for_neighbours(const CG& g, uint32_t p, F&& f) {
  uint32_t c[kMaxRank];
  decode(g, p, c);
#pragma unroll
  for (int a = 0; a < kMaxRank; ++a) {
    if (a < g.rank) {
      if (c[a] > 0) f(p - g.strides[a]);
      if (c[a] + 1 < g.dims[a]) f(p + g.strides[a]);
    }
  }
}

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

#define GRID_STRIDE(i, n)                                                     \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

__global__ void k_cc_init(uint32_t* parent, uint32_t n) {
  GRID_STRIDE(i, n) parent[i] = (uint32_t)i;
}

__global__ void k_cc_union(CG g, const uint32_t* labels, uint32_t* parent) {
  GRID_STRIDE(i, g.n) {
    const uint32_t p = (uint32_t)i, l = labels[p];
    uint32_t c[kMaxRank];
    decode(g, p, c);
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a)
      if (a < g.rank && c[a] + 1 < g.dims[a] && labels[p + g.strides[a]] == l)
        unite(parent, p, p + g.strides[a]);
  }
}

// parent -> root; idx[p] = 1 for roots (scanned into dense node ids)
__global__ void k_cc_flatten(uint32_t* parent, uint32_t* idx, uint32_t n) {
  GRID_STRIDE(i, n) {
    const uint32_t r = find_root(parent, (uint32_t)i);
    parent[i] = r;
    idx[i] = r == (uint32_t)i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) idx[n] = 0;
}

// parent[p] (root offset) -> node id, in place; node_off/size/label per node
__global__ void k_node_ids(uint32_t* nid, const uint32_t* idx, const uint32_t* labels,
                           uint32_t* node_off, uint32_t* size, uint32_t* nlab, uint32_t n) {
  GRID_STRIDE(i, n) {
    const uint32_t r = nid[i];
    const uint32_t id = idx[r];
    nid[i] = id;
    if (r == (uint32_t)i) {
      node_off[id] = r;
      nlab[id] = labels[r];
    }
    const unsigned same = __match_any_sync(__activemask(), id);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(same) - 1)) atomicAdd(size + id, __popc(same));
  }
}

// finalize_cluster_components (connectivity.hpp:125-173), one thread per k.
__global__ void k_finalize(Geom g, const uint32_t* labels, const double* centers,
                           const uint32_t* nid, const uint32_t* size, int64_t min_size,
                           uint8_t* flags, uint32_t* fcomp) {
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
  const uint32_t r = nid[seed];
  if ((int64_t)size[r] > min_size) {
    flags[r] = kFin;
    fcomp[id] = r;
  }
}

__global__ void k_max_label(const uint32_t* labels, uint32_t n, unsigned* out) {
  uint32_t m = 0;
  GRID_STRIDE(i, n) m = max(m, labels[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Largest neighbour offset below the component's root (the merge target of
// a small component: every pixel before the root is final when the sweep
// reaches it), and for the component at offset 0 the smallest finalized
// neighbour offset (best_after, connectivity.hpp:231-233).
__global__ void k_best_before(CG g, const uint32_t* nid, const uint32_t* node_off,
                              const uint8_t* flags, uint32_t* bb, uint32_t* ba0) {
  GRID_STRIDE(i, g.n) {
    const uint32_t p = (uint32_t)i, d = nid[p];
    uint32_t best = 0, after = kNone;
    if (!(flags[d] & kFin)) {
      const uint32_t r = node_off[d];
      for_neighbours(g, p, [&](uint32_t q) {
        if (q < r) best = max(best, q + 1);
        if (d == 0 && nid[q] != d && (flags[nid[q]] & kFin)) after = min(after, q);
      });
    }
    if (best) atomicMax(bb + d, best);
    if (after != kNone) atomicMin(ba0, after);
  }
}

// Static pointers and flags per node.
__global__ void k_pointers(uint32_t m, int64_t min_size, const uint32_t* nid,
                           const uint32_t* size, const uint32_t* bb, const uint32_t* ba0,
                           uint8_t* flags, uint32_t* ptr, unsigned* pending) {
  GRID_STRIDE(i, m) {
    uint8_t f = flags[i];
    uint32_t p = (uint32_t)i;
    if (!(f & kFin)) {
      if ((int64_t)size[i] > min_size || m == 1) {
        f |= kFresh;
      } else if (bb[i]) {
        p = nid[bb[i] - 1];
      } else if (*ba0 != kNone) {  // i == 0: merge ahead (best_after)
        p = nid[*ba0];
      } else {
        *pending = 1;  // pending adoption at offset 0
      }
    }
    flags[i] = f;
    ptr[i] = p;
  }
}

// ---- the exact sequential sweep on one device thread ------------------------
// connectivity.hpp:182-261 verbatim in behaviour, used (a) for the pending
// cascade at the start of the raster and (b) for label maps with ids >= k.
// cur: labels (in/out); mk: bit 0 final, bit 1 visited, bit 2 touched by an
// event; queue: n entries. Unless `full`, stops at the first offset > 0 where
// every touched pixel is final (no pending region left).
__global__ void k_sweep_serial(CG g, uint32_t* cur, uint8_t* mk,
                               uint32_t* queue, int64_t min_size, uint32_t next, int full,
                               uint32_t* result /* [0] = stop offset, [1] = next label */) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t pending = 0;
  uint32_t off = 0;
  while (off < g.n && (full || off == 0 || pending > 0)) {
    if (mk[off] & 1) {
      ++off;
      continue;
    }
    const uint32_t label = cur[off];
    uint32_t len = 0;
    queue[len++] = off;
    mk[off] |= 2;
    for (uint32_t head = 0; head < len; ++head) {
      for_neighbours(g, queue[head], [&](uint32_t q) {
        if (!(mk[q] & 2) && cur[q] == label) {
          mk[q] |= 2;
          queue[len++] = q;
        }
      });
    }
    int64_t bb = -1, ba = -1, bp = -1;
    uint32_t lb = 0, la = 0, lp = 0;
    for (uint32_t h = 0; h < len; ++h) {
      for_neighbours(g, queue[h], [&](uint32_t q) {
        const uint32_t lq = cur[q];
        if (lq == label) return;
        if (mk[q] & 1) {
          if (q < off) {
            if ((int64_t)q > bb) {
              bb = q;
              lb = lq;
            }
          } else if (ba < 0 || (int64_t)q < ba) {
            ba = q;
            la = lq;
          }
        } else if (bp < 0 || (int64_t)q < bp) {
          bp = q;
          lp = lq;
        }
      });
    }
    uint32_t target;
    uint8_t mark = 1;
    if ((int64_t)len > min_size) {
      target = next++;
    } else if (bb >= 0 || ba >= 0) {
      target = bb >= 0 ? lb : la;
    } else if (bp >= 0) {
      target = lp;  // adopt the pending label, stay unmarked
      mark = 0;
    } else {
      target = next++;
    }
    // pending = touched pixels that are not final yet (bit 2 = touched)
    for (uint32_t h = 0; h < len; ++h) {
      const uint32_t o = queue[h];
      const uint8_t w = mk[o];
      const bool was = (w & 4) && !(w & 1);
      cur[o] = target;
      mk[o] = (uint8_t)((w & 1) | mark | 4);
      pending += (int64_t)(!((w & 1) | mark)) - (int64_t)was;
    }
    ++off;
  }
  result[0] = off;
  result[1] = next;
}

__global__ void k_markers(const uint32_t* nid, const uint8_t* flags, uint8_t* mk, uint32_t n) {
  GRID_STRIDE(i, n) mk[i] = flags[nid[i]] & kFin;
}

// Components the prefix decided: pointer into F_label (merged into its
// region) or a fixed fresh label; a finalized component the prefix relabelled
// retires its label from the fixpoint.
__global__ void k_prefix_nodes(uint32_t m, const uint32_t* node_off, const uint32_t* nlab,
                               const uint32_t* cur, const uint8_t* mk, uint32_t k,
                               const uint32_t* fcomp, uint8_t* flags, uint32_t* ptr,
                               uint32_t* flab, uint8_t* factive, unsigned* err) {
  GRID_STRIDE(i, m) {
    const uint32_t r = node_off[i], lam = cur[r];
    uint8_t f = flags[i];
    if (f & kFin) {
      if (lam != nlab[i]) {
        flags[i] = f | kFixed;
        flab[i] = lam;
        factive[nlab[i]] = 0;
      }
    } else if (mk[r] & 1) {
      f |= kProc;
      if (lam >= k) {
        f |= kFixed;
        flab[i] = lam;
        ptr[i] = (uint32_t)i;
      } else if (fcomp[lam] != kNone) {
        ptr[i] = fcomp[lam];
      } else {
        *err = 1;
      }
      flags[i] = f;
    }
  }
}

// ---- fixpoint rounds ------------------------------------------------------
__global__ void k_round_ptr(uint32_t m, const uint8_t* flags, const uint32_t* ptr,
                            const uint32_t* nlab, const uint32_t* fcomp, const uint8_t* factive,
                            const uint32_t* te, uint32_t* T) {
  GRID_STRIDE(i, m) {
    const uint8_t f = flags[i];
    uint32_t t = ptr[i];
    if (!(f & (kFin | kProc))) {
      const uint32_t l = nlab[i];
      if (factive[l] && fcomp[l] != kNone && (te[l] == (uint32_t)i || (f & kAbs))) t = fcomp[l];
    }
    T[i] = t;
  }
}

// Pointer jumping towards the terminals (each thread chases a few hops).
__global__ void k_jump(uint32_t m, uint32_t* T, unsigned* changed) {
  bool ch = false;
  GRID_STRIDE(i, m) {
    uint32_t t = T[i];
#pragma unroll 1
    for (int h = 0; h < 8; ++h) {
      const uint32_t u = T[t];
      if (u == t) break;
      t = u;
      ch = true;
    }
    T[i] = t;
  }
  if (__any_sync(__activemask(), ch) && (threadIdx.x & 31) == 0) *changed = 1;
}

// One pass over the face edges: extension candidates (te_new) and absorbed
// components (against the previous round's te).
__global__ void k_edges(CG g, const uint32_t* nid, const uint8_t* flags, const uint32_t* nlab,
                        const uint32_t* fcomp, const uint8_t* factive, const uint32_t* T,
                        const uint32_t* te, uint32_t* te_new, uint8_t* absn) {
  GRID_STRIDE(i, g.n) {
    const uint32_t p = (uint32_t)i, d = nid[p];
    if (flags[d] & (kFin | kProc)) continue;
    const uint32_t l = nlab[d];
    if (!factive[l]) continue;
    const uint32_t f = fcomp[l];
    if (f == kNone) continue;
    const uint32_t t0 = te[l];
    bool cand = false, ab = false;
    for_neighbours(g, p, [&](uint32_t q) {
      const uint32_t x = nid[q];
      if (x == d || T[x] != f) return;
      const bool proc = flags[x] & kProc;
      if (x < d || proc) cand = true;
      if (t0 != kNone && d > t0 && (x < t0 || proc)) ab = true;
    });
    if (cand) atomicMin(te_new + l, d);
    if (ab) absn[d] = 1;
  }
}

__global__ void k_swap_te(uint32_t k, uint32_t* te, uint32_t* te_new, unsigned* changed) {
  GRID_STRIDE(i, k) {
    if (te[i] != te_new[i]) {
      te[i] = te_new[i];
      *changed = 1;
    }
    te_new[i] = kNone;
  }
}

__global__ void k_swap_abs(uint32_t m, uint8_t* flags, uint8_t* absn, unsigned* changed) {
  GRID_STRIDE(i, m) {
    const uint8_t f = flags[i];
    const bool a = absn[i] != 0, b = (f & kAbs) != 0;
    if (a != b) {
      flags[i] = a ? (f | kAbs) : (f & ~kAbs);
      *changed = 1;
    }
    absn[i] = 0;
  }
}

// ---- fresh ids and the output ---------------------------------------------
__device__ __forceinline__ bool is_ext(uint32_t i, uint8_t f, const uint32_t* nlab,
                                       const uint32_t* fcomp, const uint8_t* factive,
                                       const uint32_t* te) {
  if (f & (kFin | kProc)) return false;
  const uint32_t l = nlab[i];
  return factive[l] && fcomp[l] != kNone && te[l] == i;
}

__global__ void k_events(uint32_t m, const uint8_t* flags, const uint32_t* nlab,
                         const uint32_t* fcomp, const uint8_t* factive, const uint32_t* te,
                         uint32_t* ev) {
  GRID_STRIDE(i, m) {
    const uint8_t f = flags[i];
    ev[i] = is_ext((uint32_t)i, f, nlab, fcomp, factive, te) ||
            (!(f & (kFin | kProc)) && (f & kFresh) && !(f & kAbs));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ev[m] = 0;
}

__global__ void k_final_labels(uint32_t m, const uint8_t* flags, const uint32_t* nlab,
                               const uint32_t* fcomp, const uint8_t* factive,
                               const uint32_t* te, const uint32_t* rank, uint32_t next0,
                               uint32_t* flab) {
  GRID_STRIDE(i, m) {
    const uint8_t f = flags[i];
    if (f & kFixed) continue;
    if (f & kFin) {
      const uint32_t l = nlab[i];
      flab[i] = (factive[l] && te[l] != kNone) ? next0 + rank[te[l]] : l;
    } else if (!(f & kProc) && (f & kFresh) && !(f & kAbs) &&
               !is_ext((uint32_t)i, f, nlab, fcomp, factive, te)) {
      flab[i] = next0 + rank[i];
    }
  }
}

__global__ void k_output(const uint32_t* nid, const uint32_t* T, const uint32_t* flab,
                         uint32_t* out, uint32_t n) {
  GRID_STRIDE(i, n) out[i] = flab[T[nid[i]]];
}

// Stream-ordered device allocation owned for the scope of one call.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  Scratch(size_t bytes, cudaStream_t st) : s(st) {
    SSLIC_CUDA_CHECK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

inline unsigned blocks(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T h{};
  SSLIC_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

uint32_t enforce_connectivity_device(const Geom& g, const uint32_t* labels_in,
                                     const double* centers, uint32_t* labels_out,
                                     cudaStream_t s) {
  int64_t n64 = 1;
  for (int a = 0; a < g.rank; ++a) n64 *= g.dims[a];
  if (n64 >= (int64_t)0xffffffffLL)
    throw Error(SSLIC_EINVAL, "enforce_connectivity: volumes >= 2^32 voxels need the slab path");
  const uint32_t n = (uint32_t)n64;
  int64_t min_size = 1;
  for (int a = 0; a < g.rank; ++a) min_size *= g.grid[a];
  min_size /= 4;  // size_threshold (connectivity.hpp:34-38)
  const uint32_t k = (uint32_t)g.k;
  const bool timing = std::getenv("SSLIC_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();

  CG cg{};
  cg.rank = g.rank;
  cg.n = n;
  for (int a = 0; a < kMaxRank; ++a) {
    cg.dims[a] = a < g.rank ? (uint32_t)g.dims[a] : 1;
    cg.strides[a] = a < g.rank ? (uint32_t)g.strides[a] : 0;
  }
  // small control block: [0] max label, [1] pending, [2] changed, [3] err,
  // [4] ba0, [5..6] serial result
  Scratch ctl(8 * sizeof(unsigned), s);
  unsigned* c = ctl.as<unsigned>();
  SSLIC_CUDA_CHECK(cudaMemsetAsync(c, 0, 8 * sizeof(unsigned), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(c + 4, 0xff, sizeof(unsigned), s));

  Scratch nid_b((size_t)n * 4, s), idx_b(((size_t)n + 1) * 4, s);
  uint32_t* nid = nid_b.as<uint32_t>();
  uint32_t* idx = idx_b.as<uint32_t>();
  k_cc_init<<<blocks(n), 256, 0, s>>>(nid, n);
  k_cc_union<<<blocks(n), 256, 0, s>>>(cg, labels_in, nid);
  k_cc_flatten<<<blocks(n), 256, 0, s>>>(nid, idx, n);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, idx, idx, (int64_t)n + 1, s);
  Scratch tmp(tmp_bytes, s);
  SSLIC_CUDA_CHECK(
      cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, idx, idx, (int64_t)n + 1, s));
  k_max_label<<<148 * 8, 256, 0, s>>>(labels_in, n, c + 0);
  SSLIC_CUDA_CHECK(cudaGetLastError());
  const uint32_t m = read_scalar(idx + n, s);
  const unsigned max_label = read_scalar(c + 0, s);

  // per-node arrays
  Scratch node_off_b((size_t)m * 4, s), size_b((size_t)m * 4, s), nlab_b((size_t)m * 4, s),
      ptr_b((size_t)m * 4, s), T_b((size_t)m * 4, s), flab_b((size_t)m * 4, s),
      flags_b(m, s), absn_b(m, s);
  uint32_t *node_off = node_off_b.as<uint32_t>(), *size = size_b.as<uint32_t>(),
           *nlab = nlab_b.as<uint32_t>(), *ptr = ptr_b.as<uint32_t>(), *T = T_b.as<uint32_t>(),
           *flab = flab_b.as<uint32_t>();
  uint8_t *flags = flags_b.as<uint8_t>(), *absn = absn_b.as<uint8_t>();
  const size_t kk = k ? k : 1;
  Scratch fcomp_b(kk * 4, s), te_b(kk * 4, s), te_new_b(kk * 4, s), factive_b(kk, s);
  uint32_t *fcomp = fcomp_b.as<uint32_t>(), *te = te_b.as<uint32_t>(),
           *te_new = te_new_b.as<uint32_t>();
  uint8_t* factive = factive_b.as<uint8_t>();
  SSLIC_CUDA_CHECK(cudaMemsetAsync(size, 0, (size_t)m * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(flags, 0, m, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(absn, 0, m, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(flab, 0, (size_t)m * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(fcomp, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(te, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(te_new, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(factive, 1, kk, s));
  k_node_ids<<<blocks(n), 256, 0, s>>>(nid, idx, labels_in, node_off, size, nlab, n);
  if (g.k > 0)
    k_finalize<<<(unsigned)((g.k + 127) / 128), 128, 0, s>>>(g, labels_in, centers, nid, size,
                                                             min_size, flags, fcomp);
  SSLIC_CUDA_CHECK(cudaGetLastError());
  const bool full_serial = m > 0 && (uint64_t)max_label >= (uint64_t)k;

  uint32_t next = k;
  bool done = false;
  if (!full_serial) {
    // bb -> ptr (flab doubles as bb storage until the end)
    k_best_before<<<blocks(n), 256, 0, s>>>(cg, nid, node_off, flags, flab, c + 4);
    k_pointers<<<blocks(m), 256, 0, s>>>(m, min_size, nid, size, flab, c + 4, flags, ptr,
                                         c + 1);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(flab, 0, (size_t)m * 4, s));
    SSLIC_CUDA_CHECK(cudaGetLastError());
  }
  const bool serial = full_serial || read_scalar(c + 1, s) != 0;
  if (serial) {
    // exact sequential sweep on one device thread: the whole map (ids >= k)
    // or the pending cascade at the start of the raster
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out, labels_in, (size_t)n * 4,
                                     cudaMemcpyDeviceToDevice, s));
    Scratch mk_b(n, s);
    uint8_t* mk = mk_b.as<uint8_t>();
    k_markers<<<blocks(n), 256, 0, s>>>(nid, flags, mk, n);
    k_sweep_serial<<<1, 1, 0, s>>>(cg, labels_out, mk, idx, min_size, k,
                                   full_serial ? 1 : 0, c + 5);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    uint32_t res[2];
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(res, c + 5, sizeof(res), cudaMemcpyDeviceToHost, s));
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    next = res[1];
    if (res[0] >= n) {
      done = true;
    } else {
      k_prefix_nodes<<<blocks(m), 256, 0, s>>>(m, node_off, nlab, labels_out, mk, k, fcomp,
                                               flags, ptr, flab, factive, c + 3);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      if (read_scalar(c + 3, s) != 0)
        throw Error(SSLIC_ELOGIC, "enforce_connectivity: inconsistent prefix state");
    }
  }
  int rounds = 0, jumps = 0;
  if (!done) {
    for (;;) {
      ++rounds;
      k_round_ptr<<<blocks(m), 256, 0, s>>>(m, flags, ptr, nlab, fcomp, factive, te, T);
      for (;;) {
        ++jumps;
        SSLIC_CUDA_CHECK(cudaMemsetAsync(c + 2, 0, sizeof(unsigned), s));
        k_jump<<<blocks(m), 256, 0, s>>>(m, T, c + 2);
        SSLIC_CUDA_CHECK(cudaGetLastError());
        if (read_scalar(c + 2, s) == 0) break;
      }
      k_edges<<<blocks(n), 256, 0, s>>>(cg, nid, flags, nlab, fcomp, factive, T, te, te_new,
                                        absn);
      SSLIC_CUDA_CHECK(cudaMemsetAsync(c + 2, 0, sizeof(unsigned), s));
      k_swap_te<<<blocks(kk), 256, 0, s>>>(k, te, te_new, c + 2);
      k_swap_abs<<<blocks(m), 256, 0, s>>>(m, flags, absn, c + 2);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      if (read_scalar(c + 2, s) == 0) break;
    }
    // the last round left T consistent with the converged te / absorbed sets
    k_events<<<blocks(m), 256, 0, s>>>(m, flags, nlab, fcomp, factive, te, idx);
    SSLIC_CUDA_CHECK(
        cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, idx, idx, (int64_t)m + 1, s));
    k_final_labels<<<blocks(m), 256, 0, s>>>(m, flags, nlab, fcomp, factive, te, idx, next,
                                             flab);
    k_output<<<blocks(n), 256, 0, s>>>(nid, T, flab, labels_out, n);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    next += read_scalar(idx + m, s);
  }
  if (timing) {
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr,
                 "[sslic] connectivity: %u voxels, %u components, %s, %d rounds, %d jump "
                 "passes, %.2f ms\n",
                 n, m, full_serial ? "serial (ids >= k)" : (serial ? "serial prefix" : "no prefix"),
                 rounds, jumps, std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  return next;
}

}  // namespace sslic_b200
