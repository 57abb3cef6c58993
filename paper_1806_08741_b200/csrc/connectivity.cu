// Connectivity enforcement (connectivity.hpp:125-273), entirely on the device.
//
// 1. Face-connected component labelling of the label map, slab by slab along
//    the last axis (32-bit local offsets per slab): lock-free union-find
//    (atomicMin hooking; a component's root is its smallest flat offset) --
//    32x8x8 tiles in shared memory first, then the tile faces in global
//    memory with path halving (k_cc_tile, k_cc_seams) --
//    then the components are numbered densely in root order, so a node id
//    orders components exactly like the raster sweep reaches them. Volumes of
//    2^32 voxels or more take several slabs: their components are stitched
//    across the slab faces by a union-find over node ids (a set's smallest
//    node id is its smallest root offset) and renumbered densely, which gives
//    the same ids a whole-volume labelling would (SURVEY §2 "C2").
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
//      unique fixpoint, which equals the sequential sweep's outcome; the
//      edges that can matter are listed once (k_edge_list) and the rounds
//      walk that list;
//    * fresh ids are numbered by a prefix sum over events in root order.
//    A pending adoption (no finalized neighbour at all) can only start at
//    offset 0; the cascade it opens is emulated exactly by one device thread
//    until no pending pixel remains, then the fixpoint takes over. Label maps
//    holding ids >= k (never produced by run_slic) are swept entirely by that
//    device thread, because fresh ids could then collide with input labels.
//
// Voxel offsets are `Off` (uint32_t below 2^32 voxels, uint64_t above);
// component (node) ids are 32-bit. Per voxel the pass needs the label map and
// one node id (8 bytes); labels_out may alias labels_in. labels_out doubles
// as scratch (the edge list on a full device) until the final labels are
// written: after a failed call its content is undefined.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

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

// Geometry: the last axis is the slab axis; the in-plane extent is < 2^32.
template <class Off>
struct CG {
  int rank;
  Off dims[kMaxRank];
  Off strides[kMaxRank];
  Off n;
  Off plane;  // product of the in-plane extents (1 for rank 1)
};

template <class Off>
__device__ __forceinline__ void decode(const CG<Off>& g, Off p, Off* c) {
  const Off z = p / g.plane;
  uint32_t i = (uint32_t)(p - z * g.plane);
#pragma unroll
  for (int a = 0; a < kMaxRank - 1; ++a) {
    if (a < g.rank - 1) {
      const uint32_t d = (uint32_t)g.dims[a];
      c[a] = i % d;
      i /= d;
    }
  }
  c[g.rank - 1] = z;
}

// Calls f(q) for every face neighbour q of p.
template <class Off, class F>
__device__ __forceinline__ void for_neighbours(const CG<Off>& g, Off p, F&& f) {
  Off c[kMaxRank];
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

// find with path halving: a node that is not a root never becomes one again
// and only ever points at an ancestor, so the plain store of the grandparent
// is safe next to the hooking atomics (and keeps parent[i] <= i)
__device__ __forceinline__ uint32_t find_root_halving(uint32_t* parent, uint32_t i) {
  for (;;) {
    const uint32_t p = parent[i];
    if (p == i) return i;
    const uint32_t gp = parent[p];
    if (gp == p) return p;
    parent[i] = gp;
    i = gp;
  }
}

__device__ __forceinline__ void unite(uint32_t* parent, uint32_t a, uint32_t b) {
  for (;;) {
    a = find_root_halving(parent, a);
    b = find_root_halving(parent, b);
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

// grid-stride loop over [0, n) with a 64-bit counter (a 32-bit one would wrap
// past 2^32 near n); the body sees `i` as a T (the inner one-trip loop keeps
// `continue` meaning "next element")
#define GRID_STRIDE(T, i, n)                                                           \
  for (uint64_t i##_g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;               \
       i##_g < (uint64_t)(n); i##_g += (uint64_t)gridDim.x * blockDim.x)               \
    for (T i = (T)i##_g, i##_once = 1; i##_once; i##_once = 0)

// ---- slab CCL (32-bit local offsets) ------------------------------------------
__global__ void k_cc_init(uint32_t* parent, uint32_t n) {
  GRID_STRIDE(uint32_t, i, n) parent[i] = i;
}

__global__ void k_cc_union(CG<uint32_t> g, const uint32_t* labels, uint32_t* parent) {
  GRID_STRIDE(uint32_t, p, g.n) {
    const uint32_t l = labels[p];
    uint32_t c[kMaxRank];
    decode(g, p, c);
#pragma unroll
    for (int a = 0; a < kMaxRank; ++a)
      if (a < g.rank && c[a] + 1 < g.dims[a] && labels[p + g.strides[a]] == l)
        unite(parent, p, p + g.strides[a]);
  }
}

// ---- tiled CCL for ranks 2-3 (the whole-slab k_cc_union above stays for ranks 1 and 4)
// A CTA labels one 32x8x8 tile in shared memory (runs along x by ballot, then
// shared-memory atomicMin hooking along y and z) and writes each voxel's tile
// root as a slab offset; k_cc_seams then unites equal labels across the tile
// faces in global memory. A union is skipped when the pair one step back along
// another in-tile axis carries the same label on both sides: that pair (or,
// by induction, one further back) makes the same connection. Hooking always
// points the larger root at the smaller one and a tile's local order is the
// raster order, so a component's root is its smallest offset, as before.
constexpr uint32_t kTX = 32, kTY = 8, kTZ = 8, kTileVox = kTX * kTY * kTZ;

__device__ __forceinline__ void unite_tile(uint32_t* par, uint32_t a, uint32_t b) {
  for (;;) {
    uint32_t p = par[a];
    while (p != a) {
      a = p;
      p = par[a];
    }
    p = par[b];
    while (p != b) {
      b = p;
      p = par[b];
    }
    if (a == b) return;
    if (a < b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMin(par + a, b);
    if (old == a) return;
    a = old;
  }
}

__global__ void __launch_bounds__(256) k_cc_tile(uint32_t X, uint32_t Y, uint32_t Z, uint32_t ntx,
                                                 uint32_t nty, const uint32_t* __restrict__ labels,
                                                 uint32_t* __restrict__ parent) {
  __shared__ uint32_t lab[kTileVox];
  __shared__ uint32_t par[kTileVox];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t t = blockIdx.x;
  const uint32_t tx = t % ntx;
  t /= ntx;
  const uint32_t ty = t % nty, tz = t / nty;
  const uint32_t x0 = tx * kTX, y0 = ty * kTY, z0 = tz * kTZ;
  const uint32_t x = x0 + lane, y = y0 + w;
  const bool vxy = x < X && y < Y;
  const uint32_t nz = min(kTZ, Z - z0);
  const uint32_t pbase = x + X * (y + Y * z0), zs = X * Y;
  const uint32_t li0 = lane + kTX * w;
  // labels into shared memory; parents start at the head of the voxel's x-run
#pragma unroll
  for (uint32_t z = 0; z < kTZ; ++z) {
    const bool v = vxy && z < nz;
    const uint32_t l = v ? labels[pbase + z * zs] : 0u;
    const uint32_t left = __shfl_up_sync(0xffffffffu, l, 1);
    const unsigned same = __ballot_sync(0xffffffffu, v && lane > 0 && l == left);
    const unsigned heads = ~same & ((2u << lane) - 1u);  // bit 0 is always a head
    const uint32_t li = li0 + kTX * kTY * z;
    lab[li] = l;
    par[li] = li - lane + (31u - (uint32_t)__clz(heads));
  }
  __syncthreads();
  if (vxy) {
#pragma unroll
    for (uint32_t z = 0; z < kTZ; ++z) {
      if (z >= nz) break;
      const uint32_t li = li0 + kTX * kTY * z, l = lab[li];
      const bool back = lane > 0 && lab[li - 1] == l;
      if (w + 1 < kTY && y + 1 < Y) {
        const uint32_t lj = li + kTX;
        if (lab[lj] == l && !(back && lab[lj - 1] == l)) unite_tile(par, li, lj);
      }
      if (z + 1 < nz) {
        const uint32_t lj = li + kTX * kTY;
        if (lab[lj] == l && !(back && lab[lj - 1] == l)) unite_tile(par, li, lj);
      }
    }
  }
  __syncthreads();
  if (vxy) {
#pragma unroll
    for (uint32_t z = 0; z < kTZ; ++z) {
      if (z >= nz) break;
      uint32_t r = li0 + kTX * kTY * z, p = par[r];
      while (p != r) {
        r = p;
        p = par[r];
      }
      parent[pbase + z * zs] =
          (x0 + (r & (kTX - 1))) + X * ((y0 + ((r / kTX) & (kTY - 1))) + Y * (z0 + r / (kTX * kTY)));
    }
  }
}

// unions across the tile faces (the voxels with x % 32 == 31, y % 8 == 7 or
// z % 8 == 7 and their +1 neighbours)
__global__ void k_cc_seams(uint32_t X, uint32_t Y, uint32_t Z, const uint32_t* __restrict__ labels,
                           uint32_t* parent) {
  const uint32_t n = X * Y * Z, zs = X * Y;
  GRID_STRIDE(uint32_t, p, n) {
    const uint32_t z = p / zs, i = p - z * zs, y = i / X, x = i - y * X;
    const bool fx = (x & (kTX - 1)) == kTX - 1 && x + 1 < X;
    const bool fy = (y & (kTY - 1)) == kTY - 1 && y + 1 < Y;
    const bool fz = (z & (kTZ - 1)) == kTZ - 1 && z + 1 < Z;
    if (!(fx | fy | fz)) continue;
    const uint32_t l = labels[p];
    const bool backx = (x & (kTX - 1)) != 0 && labels[p - 1] == l;
    if (fx && labels[p + 1] == l) {
      const bool backy = (y & (kTY - 1)) != 0 && labels[p - X] == l && labels[p + 1 - X] == l;
      if (!backy) unite(parent, p, p + 1);
    }
    if (fy && labels[p + X] == l && !(backx && labels[p + X - 1] == l)) unite(parent, p, p + X);
    if (fz && labels[p + zs] == l && !(backx && labels[p + zs - 1] == l)) unite(parent, p, p + zs);
  }
}

// parent -> root; idx[p] = 1 for roots (scanned into dense node ids)
__global__ void k_cc_flatten(uint32_t* parent, uint32_t* idx, uint32_t n) {
  GRID_STRIDE(uint32_t, i, n) {
    const uint32_t r = find_root(parent, i);
    parent[i] = r;
    idx[i] = r == i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) idx[n] = 0;
}

// parent[p] (local root) -> global node id (base + dense local id), in place;
// node_off (global flat offset of the root), nlab and size per node
// component sizes are 32-bit; a component of 2^32 voxels or more sets *ovf
__device__ __forceinline__ void add_size(uint32_t* size, uint32_t id, uint32_t v, unsigned* ovf) {
  const uint32_t old = atomicAdd(size + id, v);
  if (old + v < old) *ovf = 1;
}

template <class Off>
__global__ void k_node_ids(uint32_t* nid, const uint32_t* idx, const uint32_t* labels,
                           Off* node_off, uint32_t* size, uint32_t* nlab, uint32_t n,
                           uint32_t base, Off off0, unsigned* ovf) {
  GRID_STRIDE(uint32_t, i, n) {
    const uint32_t r = nid[i];
    const uint32_t id = base + idx[r];
    nid[i] = id;
    if (r == i) {
      node_off[id] = off0 + (Off)r;
      nlab[id] = labels[r];
    }
    const unsigned same = __match_any_sync(__activemask(), id);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(same) - 1)) add_size(size, id, __popc(same), ovf);
  }
}

// ---- stitching across slab faces (node-level union-find) ---------------------
template <class Off>
__global__ void k_face_union(const uint32_t* labels, const uint32_t* nid, Off below, Off above,
                             uint32_t plane, uint32_t* parent) {
  GRID_STRIDE(uint32_t, i, plane) {
    const Off p = below + i, q = above + i;
    if (labels[p] == labels[q]) unite(parent, nid[p], nid[q]);
  }
}

__global__ void k_node_flatten(uint32_t* parent, uint32_t* flag, uint8_t* root, uint32_t m) {
  GRID_STRIDE(uint32_t, i, m) {
    const uint32_t r = find_root(parent, i);
    parent[i] = r;
    flag[i] = r == i;
    root[i] = r == i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flag[m] = 0;
}

// a merged set's size goes to its root entry (non-roots are only read)
__global__ void k_size_to_root(uint32_t m, const uint32_t* parent, uint32_t* size, unsigned* ovf) {
  GRID_STRIDE(uint32_t, i, m) {
    const uint32_t r = parent[i];
    if (r != i) add_size(size, r, size[i], ovf);
  }
}

template <class Off>
__global__ void k_nid_remap(uint32_t* nid, const uint32_t* parent, const uint32_t* fid, Off n) {
  GRID_STRIDE(Off, i, n) nid[i] = fid[parent[nid[i]]];
}

// finalize_cluster_components (connectivity.hpp:125-173), one thread per k.
template <class Off>
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

template <class Off>
__global__ void k_max_label(const uint32_t* labels, Off n, unsigned* out) {
  uint32_t m = 0;
  GRID_STRIDE(Off, i, n) m = max(m, labels[i]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Largest neighbour offset below the component's root (the merge target of
// a small component: every pixel before the root is final when the sweep
// reaches it), kept as the distance back from the root (< the plane stride,
// so 32 bits; 0xffffffff: none) and minimised; for the component at offset
// 0 the smallest finalized neighbour offset (best_after, connectivity.hpp:
// 231-233).
template <class Off>
__global__ void k_best_before(CG<Off> g, const uint32_t* nid, const Off* node_off,
                              const uint8_t* flags, uint32_t* back, unsigned long long* ba0) {
  GRID_STRIDE(Off, p, g.n) {
    const uint32_t d = nid[p];
    uint32_t best = kNone;
    unsigned long long after = ~0ull;
    if (!(flags[d] & kFin)) {
      const Off r = node_off[d];
      for_neighbours(g, p, [&](Off q) {
        if (q < r) best = min(best, (uint32_t)(r - q));
        if (d == 0 && nid[q] != d && (flags[nid[q]] & kFin)) after = min(after, (unsigned long long)q);
      });
    }
    if (best != kNone) atomicMin(back + d, best);
    if (after != ~0ull) atomicMin(ba0, after);
  }
}

// Static pointers and flags per node.
template <class Off>
__global__ void k_pointers(uint32_t m, int64_t min_size, const uint32_t* nid,
                           const uint32_t* size, const uint32_t* back,
                           const Off* node_off, const unsigned long long* ba0, uint8_t* flags,
                           uint32_t* ptr, unsigned* pending) {
  GRID_STRIDE(uint32_t, i, m) {
    uint8_t f = flags[i];
    uint32_t p = i;
    if (!(f & kFin)) {
      if ((int64_t)size[i] > min_size || m == 1) {
        f |= kFresh;
      } else if (back[i] != kNone) {
        p = nid[node_off[i] - (Off)back[i]];
      } else if (*ba0 != ~0ull) {  // i == 0: merge ahead (best_after)
        p = nid[(Off)*ba0];
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
// event; queue: qcap entries. Unless `full`, stops at the first offset > 0
// where every touched pixel is final (no pending region left).
template <class Off>
__global__ void k_sweep_serial(CG<Off> g, uint32_t* cur, uint8_t* mk, Off* queue, Off qcap,
                               int64_t min_size, uint32_t next, int full,
                               unsigned long long* result /* [0] stop, [1] next, [2] overflow */) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t pending = 0;
  Off off = 0;
  while (off < g.n && (full || off == 0 || pending > 0)) {
    if (mk[off] & 1) {
      ++off;
      continue;
    }
    const uint32_t label = cur[off];
    Off len = 0;
    queue[len++] = off;
    mk[off] |= 2;
    for (Off head = 0; head < len; ++head) {
      for_neighbours(g, queue[head], [&](Off q) {
        if (!(mk[q] & 2) && cur[q] == label) {
          mk[q] |= 2;
          if (len < qcap) queue[len] = q;
          ++len;
        }
      });
      if (len > qcap) {
        result[2] = 1;
        return;
      }
    }
    int64_t bb = -1, ba = -1, bp = -1;
    uint32_t lb = 0, la = 0, lp = 0;
    for (Off h = 0; h < len; ++h) {
      for_neighbours(g, queue[h], [&](Off q) {
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
    for (Off h = 0; h < len; ++h) {
      const Off o = queue[h];
      const uint8_t w = mk[o];
      const bool was = (w & 4) && !(w & 1);
      cur[o] = target;
      mk[o] = (uint8_t)((w & 1) | mark | 4);
      pending += (int64_t)(!((w & 1) | mark)) - (int64_t)was;
    }
    ++off;
  }
  result[0] = (unsigned long long)off;
  result[1] = next;
}

template <class Off>
__global__ void k_markers(const uint32_t* nid, const uint8_t* flags, uint8_t* mk, Off n) {
  GRID_STRIDE(Off, i, n) mk[i] = flags[nid[i]] & kFin;
}

// Components the prefix decided: pointer into F_label (merged into its
// region) or a fixed fresh label; a finalized component the prefix relabelled
// retires its label from the fixpoint.
template <class Off>
__global__ void k_prefix_nodes(uint32_t m, const Off* node_off, const uint32_t* nlab,
                               const uint32_t* cur, const uint8_t* mk, uint32_t k,
                               const uint32_t* fcomp, uint8_t* flags, uint32_t* ptr,
                               uint32_t* flab, uint8_t* factive, unsigned* err) {
  GRID_STRIDE(uint32_t, i, m) {
    const Off r = node_off[i];
    const uint32_t lam = cur[r];
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
        ptr[i] = i;
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
  GRID_STRIDE(uint32_t, i, m) {
    const uint8_t f = flags[i];
    uint32_t t = ptr[i];
    if (!(f & (kFin | kProc))) {
      const uint32_t l = nlab[i];
      if (factive[l] && fcomp[l] != kNone && (te[l] == i || (f & kAbs))) t = fcomp[l];
    }
    T[i] = t;
  }
}

// Pointer jumping towards the terminals (each thread chases a few hops).
__global__ void k_jump(uint32_t m, uint32_t* T, unsigned* changed) {
  bool ch = false;
  GRID_STRIDE(uint32_t, i, m) {
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
template <class Off>
__device__ __forceinline__ void edge_body(const CG<Off>& g, Off p, uint32_t d, uint32_t l,
                                          uint32_t f, const uint32_t* nid, const uint8_t* flags,
                                          const uint32_t* T, const uint32_t* te, uint32_t* te_new,
                                          uint8_t* absn) {
  const uint32_t t0 = te[l];
  bool cand = false, ab = false;
  for_neighbours(g, p, [&](Off q) {
    const uint32_t x = nid[q];
    if (x == d || T[x] != f) return;
    const bool proc = flags[x] & kProc;
    if (x < d || proc) cand = true;
    if (t0 != kNone && d > t0 && (x < t0 || proc)) ab = true;
  });
  if (cand) atomicMin(te_new + l, d);
  if (ab) absn[d] = 1;
}

template <class Off>
__global__ void k_edges(CG<Off> g, const uint32_t* nid, const uint8_t* flags,
                        const uint32_t* nlab, const uint32_t* fcomp, const uint8_t* factive,
                        const uint32_t* T, const uint32_t* te, uint32_t* te_new, uint8_t* absn) {
  GRID_STRIDE(Off, p, g.n) {
    const uint32_t d = nid[p];
    if (flags[d] & (kFin | kProc)) continue;
    const uint32_t l = nlab[d];
    if (!factive[l]) continue;
    const uint32_t f = fcomp[l];
    if (f == kNone) continue;
    edge_body(g, p, d, l, f, nid, flags, T, te, te_new, absn);
  }
}

// The rounds' edge pass as a list. Only a neighbour component x that is not
// final can satisfy T[x] == f for x != f (a final component's T is itself,
// always), and the voxels the pass skips are the same in every round, so the
// candidate edges (d, x, label of d | kProc(x) << 31) are listed once, in any
// order (the pass only takes minima and sets flags), and every round walks
// the list with ONE gather (T[x]) per edge instead of the node ids and flags
// of six neighbours per voxel. *count may pass cap; the caller then keeps the
// whole-map pass.
template <class Off>
__global__ void k_edge_list(CG<Off> g, const uint32_t* nid, const uint8_t* flags,
                            const uint32_t* nlab, const uint32_t* fcomp, const uint8_t* factive,
                            uint32_t* ed, uint32_t* ex, uint32_t* el, unsigned long long cap,
                            unsigned long long* count) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
       base < (uint64_t)g.n; base += warps * 32) {
    const uint64_t p = base + lane;
    bool act = false;
    uint32_t d = 0, l = 0, f = 0;
    if (p < (uint64_t)g.n) {
      d = nid[p];
      if (!(flags[d] & (kFin | kProc))) {
        l = nlab[d];
        f = fcomp[l];
        act = factive[l] && f != kNone;
      }
    }
    if (!__any_sync(0xffffffffu, act)) continue;
    // the qualifying neighbour components, one register per face (static
    // slots: the loops are unrolled), so the neighbours are gathered once
    uint32_t xs[2 * kMaxRank];
    unsigned vm = 0;
    if (act) {
      Off c[kMaxRank];
      decode(g, (Off)p, c);
#pragma unroll
      for (int a = 0; a < kMaxRank; ++a) {
        if (a < g.rank) {
          if (c[a] > 0) {
            const uint32_t x = nid[(Off)p - g.strides[a]];
            const uint8_t fx = x != d ? flags[x] : kFin;
            xs[2 * a] = x | 0u;
            if (x != d && (!(fx & kFin) || x == f)) vm |= (1u | (fx & kProc ? 2u : 0u)) << (4 * a);
          }
          if (c[a] + 1 < g.dims[a]) {
            const uint32_t x = nid[(Off)p + g.strides[a]];
            const uint8_t fx = x != d ? flags[x] : kFin;
            xs[2 * a + 1] = x;
            if (x != d && (!(fx & kFin) || x == f)) vm |= (4u | (fx & kProc ? 8u : 0u)) << (4 * a);
          }
        }
      }
    }
    // bits 0/2 of each nibble: slot 2a / 2a+1 holds an edge; bits 1/3: x is kProc
    const unsigned cnt = __popc(vm & 0x5555u);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (unsigned)o) incl += v;
    }
    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(count, (unsigned long long)total);
    pos = __shfl_sync(0xffffffffu, pos, 0) + (incl - cnt);
    if (cnt && pos + cnt <= cap) {
#pragma unroll
      for (int j = 0; j < 2 * kMaxRank; ++j) {
        if (vm >> (2 * j) & 1u) {
          ed[pos] = d;
          ex[pos] = xs[j];
          el[pos] = l | (vm >> (2 * j + 1) & 1u ? 0x80000000u : 0u);
          ++pos;
        }
      }
    }
  }
}

__global__ void k_edges_list(const uint32_t* ed, const uint32_t* ex, const uint32_t* el,
                             unsigned long long count, const uint32_t* fcomp, const uint32_t* T,
                             const uint32_t* te, uint32_t* te_new, uint8_t* absn) {
  GRID_STRIDE(uint64_t, i, count) {
    const uint32_t x = ex[i], lp = el[i], l = lp & 0x7fffffffu;
    if (T[x] != fcomp[l]) continue;
    const uint32_t d = ed[i], t0 = te[l];
    const bool proc = lp >> 31;
    if (x < d || proc) atomicMin(te_new + l, d);
    if (t0 != kNone && d > t0 && (x < t0 || proc)) absn[d] = 1;
  }
}

__global__ void k_swap_te(uint32_t k, uint32_t* te, uint32_t* te_new, unsigned* changed) {
  GRID_STRIDE(uint32_t, i, k) {
    if (te[i] != te_new[i]) {
      te[i] = te_new[i];
      *changed = 1;
    }
    te_new[i] = kNone;
  }
}

__global__ void k_swap_abs(uint32_t m, uint8_t* flags, uint8_t* absn, unsigned* changed) {
  GRID_STRIDE(uint32_t, i, m) {
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
  GRID_STRIDE(uint32_t, i, m) {
    const uint8_t f = flags[i];
    ev[i] = is_ext(i, f, nlab, fcomp, factive, te) ||
            (!(f & (kFin | kProc)) && (f & kFresh) && !(f & kAbs));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ev[m] = 0;
}

__global__ void k_final_labels(uint32_t m, const uint8_t* flags, const uint32_t* nlab,
                               const uint32_t* fcomp, const uint8_t* factive,
                               const uint32_t* te, const uint32_t* rank, uint32_t next0,
                               uint32_t* flab) {
  GRID_STRIDE(uint32_t, i, m) {
    const uint8_t f = flags[i];
    if (f & kFixed) continue;
    if (f & kFin) {
      const uint32_t l = nlab[i];
      flab[i] = (factive[l] && te[l] != kNone) ? next0 + rank[te[l]] : l;
    } else if (!(f & kProc) && (f & kFresh) && !(f & kAbs) &&
               !is_ext(i, f, nlab, fcomp, factive, te)) {
      flab[i] = next0 + rank[i];
    }
  }
}

template <class Off>
__global__ void k_output(const uint32_t* nid, const uint32_t* T, const uint32_t* flab,
                         uint32_t* out, Off n) {
  GRID_STRIDE(Off, i, n) out[i] = flab[T[nid[i]]];
}

// k_output fused with the output files' by-products: the max label and the
// contour bitmask, from the neighbours' OUTPUT labels (flab[T[nid[q]]], so no
// second pass over the written map is needed).
template <class Off>
__global__ void k_output_fused(CG<Off> g, const uint32_t* nid, const uint32_t* T,
                               const uint32_t* flab, uint32_t* out, unsigned* max_label,
                               uint32_t* boundary) {
  uint32_t mx = 0;
  GRID_STRIDE(Off, i, g.n) {
    const uint32_t L = flab[T[nid[i]]];
    out[i] = L;
    mx = max(mx, L);
    if (boundary) {
      bool b = false;
      for_neighbours(g, i, [&](Off q) { b |= flab[T[nid[q]]] != L; });
      // lanes of this warp-iteration: consecutive i from a 32-aligned base
      const uint64_t base = (uint64_t)i - (threadIdx.x & 31);
      const uint64_t left = (uint64_t)g.n - base;
      const unsigned act = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
      const unsigned bits = __ballot_sync(act, b);
      if ((threadIdx.x & 31) == 0 && bits) boundary[i / 32] = bits;  // i is 32-aligned here
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);  // every lane leaves the loop and gets here
  if ((threadIdx.x & 31) == 0 && max_label) atomicMax(max_label, mx);
}

// the same by-products of a final label map
template <class Off>
__global__ void k_label_outputs(CG<Off> g, const uint32_t* labels, unsigned* max_label,
                                uint32_t* boundary) {
  uint32_t mx = 0;
  GRID_STRIDE(Off, i, g.n) {
    const uint32_t L = labels[i];
    mx = max(mx, L);
    if (boundary) {
      bool b = false;
      for_neighbours(g, i, [&](Off q) { b |= labels[q] != L; });
      // lanes of this warp-iteration: consecutive i from a 32-aligned base
      const uint64_t base = (uint64_t)i - (threadIdx.x & 31);
      const uint64_t left = (uint64_t)g.n - base;
      const unsigned act = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
      const unsigned bits = __ballot_sync(act, b);
      if ((threadIdx.x & 31) == 0 && bits) boundary[i / 32] = bits;
    }
  }
  mx = __reduce_max_sync(0xffffffffu, mx);  // every lane leaves the loop and gets here
  if ((threadIdx.x & 31) == 0 && max_label) atomicMax(max_label, mx);
}

// Stream-ordered device allocation owned for the scope of one call.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s;
  Scratch() : s(nullptr) {}
  Scratch(size_t bytes, cudaStream_t st) : s(st) {
    SSLIC_CUDA_CHECK(cudaMallocAsync(&p, bytes ? bytes : 1, st));
  }
  // optional buffers: false (and no sticky error) when the memory is not there
  bool try_alloc(size_t bytes, cudaStream_t st) {
    release();
    s = st;
    if (cudaMallocAsync(&p, bytes ? bytes : 1, st) != cudaSuccess) {
      p = nullptr;
      (void)cudaGetLastError();
      return false;
    }
    return true;
  }
  ~Scratch() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
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

template <class Off>
CG<Off> make_cg(const Geom& g, int64_t z0, int64_t z1) {
  CG<Off> c{};
  c.rank = g.rank;
  int64_t plane = 1;
  for (int a = 0; a < kMaxRank; ++a) {
    c.dims[a] = a < g.rank ? (Off)g.dims[a] : 1;
    c.strides[a] = a < g.rank ? (Off)g.strides[a] : 0;
  }
  for (int a = 0; a + 1 < g.rank; ++a) plane *= g.dims[a];
  c.dims[g.rank - 1] = (Off)(z1 - z0);
  c.plane = (Off)plane;
  c.n = (Off)(plane * (z1 - z0));
  return c;
}

// Planes per CCL slab: the whole image below 2^31 voxels (one slab), else
// slabs of at most 2^30 voxels (32-bit local offsets and a 4 GB scan
// buffer). SSLIC_CC_SLAB_PLANES forces a slab height (tests of the
// stitching on small volumes).
int64_t slab_planes(const Geom& g, int64_t plane, int64_t last) {
  if (const char* e = std::getenv("SSLIC_CC_SLAB_PLANES")) {
    const int64_t v = std::atoll(e);
    if (v > 0) return std::min(v, last);
  }
  if (plane * last < ((int64_t)1 << 31)) return last;
  const int64_t p = ((int64_t)1 << 30) / plane;
  if (p < 1) throw Error(SSLIC_EINVAL, "enforce_connectivity: one plane holds >= 2^30 voxels");
  return std::min(p, last);
}

template <class Off>
uint32_t connectivity_impl(const Geom& g, const uint32_t* labels_in, const double* centers,
                           uint32_t* labels_out, cudaStream_t s, LabelOutputs outs) {
  int64_t n64 = 1;
  for (int a = 0; a < g.rank; ++a) n64 *= g.dims[a];
  const Off n = (Off)n64;
  int64_t min_size = 1;
  for (int a = 0; a < g.rank; ++a) min_size *= g.grid[a];
  min_size /= 4;  // size_threshold (connectivity.hpp:34-38)
  const uint32_t k = (uint32_t)g.k;
  const bool timing = std::getenv("SSLIC_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  double ph[5] = {0, 0, 0, 0, 0};  // CCL, node ids + stitching, finalize + pointers, list, rounds
  auto stamp = [&](int i) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    ph[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  const int last_axis = g.rank - 1;
  const int64_t last = g.dims[last_axis];
  int64_t plane = 1;
  for (int a = 0; a < last_axis; ++a) plane *= g.dims[a];
  const CG<Off> cg = make_cg<Off>(g, 0, last);

  // small control block: [0] max label, [1] pending, [2] changed, [3] err
  Scratch ctl(8 * sizeof(unsigned), s);
  unsigned* c = ctl.as<unsigned>();
  SSLIC_CUDA_CHECK(cudaMemsetAsync(c, 0, 8 * sizeof(unsigned), s));
  // [0] best_after of node 0, [1..3] serial, [4] listed edge-pass voxels
  Scratch ull(5 * sizeof(unsigned long long), s);
  unsigned long long* cu = ull.as<unsigned long long>();
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cu, 0, 5 * sizeof(unsigned long long), s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(cu, 0xff, sizeof(unsigned long long), s));
  k_max_label<Off><<<148 * 8, 256, 0, s>>>(labels_in, n, c + 0);

  // ---- 1. CCL per slab, node ids in raster order ----
  const int64_t sp = slab_planes(g, plane, last);
  const int nslabs = (int)((last + sp - 1) / sp);
  const int64_t slab_max = sp * plane;
  Scratch nid_b((size_t)n64 * 4, s), idx_b(((size_t)slab_max + 1) * 4, s);
  uint32_t* nid = nid_b.as<uint32_t>();
  uint32_t* idx = idx_b.as<uint32_t>();
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, idx, idx, slab_max + 1, s);
  std::vector<uint32_t> slab_m(nslabs);
  // tiled shared-memory CCL for ranks 2-3 with rows of at least half a tile
  // (a 1-D image would fill 1/64 of each tile; SSLIC_CC_NO_TILES=1: the
  // whole-slab union-find, kept for ranks 1 and 4 and for the equality test)
  const bool tiled = g.rank >= 2 && g.rank <= 3 && g.dims[0] >= 16 &&
                     std::getenv("SSLIC_CC_NO_TILES") == nullptr;
  // -> nid[slab] = local roots, idx = root flags; `again`: the roots are
  // still in nid from the first pass (only idx was reused), so just the flags
  auto slab_ccl = [&](int si, bool again = false) {
    const int64_t z0 = si * sp, z1 = std::min(last, z0 + sp);
    const CG<uint32_t> sg = make_cg<uint32_t>(g, z0, z1);
    uint32_t* par = nid + z0 * plane;
    const uint32_t* lab = labels_in + z0 * plane;
    if (again) {
    } else if (tiled) {
      const uint32_t X = sg.dims[0], Y = g.rank > 1 ? sg.dims[1] : 1, Z = g.rank > 2 ? sg.dims[2] : 1;
      const uint32_t ntx = (X + kTX - 1) / kTX, nty = (Y + kTY - 1) / kTY, ntz = (Z + kTZ - 1) / kTZ;
      k_cc_tile<<<ntx * nty * ntz, 256, 0, s>>>(X, Y, Z, ntx, nty, lab, par);
      k_cc_seams<<<blocks(sg.n), 256, 0, s>>>(X, Y, Z, lab, par);
    } else {
      k_cc_init<<<blocks(sg.n), 256, 0, s>>>(par, sg.n);
      k_cc_union<<<blocks(sg.n), 256, 0, s>>>(sg, lab, par);
    }
    k_cc_flatten<<<blocks(sg.n), 256, 0, s>>>(par, idx, sg.n);
    return sg.n;
  };
  uint64_t m_total = 0;
  {
    Scratch tmp(tmp_bytes, s);
    for (int si = 0; si < nslabs; ++si) {
      const uint32_t ns = slab_ccl(si);
      SSLIC_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, idx, idx, (int64_t)ns + 1, s));
      slab_m[si] = read_scalar(idx + ns, s);
      m_total += slab_m[si];
    }
  }
  stamp(0);
  if (m_total >= kNone) throw Error(SSLIC_EINVAL, "enforce_connectivity: >= 2^32 components");
  uint32_t m = (uint32_t)m_total;
  const unsigned max_label = read_scalar(c + 0, s);
  // per-node arrays (node_off / nlab / size are compacted in place after
  // stitching; ptr / T / flags double as the stitching scratch)
  Scratch node_off_b((size_t)m * sizeof(Off), s), nlab_b((size_t)m * 4, s),
      size_b(((size_t)m + 1) * 4, s);
  Scratch ptr_b((size_t)m * 4, s), T_b(((size_t)m + 1) * 4, s), flab_b((size_t)m * 4, s),
      flags_b(m, s), absn_b(m, s);
  SSLIC_CUDA_CHECK(cudaMemsetAsync(size_b.p, 0, (size_t)m * 4, s));
  {
    Scratch tmp(tmp_bytes, s);
    uint32_t base = 0;
    for (int si = 0; si < nslabs; ++si) {
      const int64_t z0 = si * sp;
      uint32_t ns;
      if (nslabs > 1) {  // the first pass's root flags were overwritten by the next slab's
        ns = slab_ccl(si, true);
        SSLIC_CUDA_CHECK(
            cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, idx, idx, (int64_t)ns + 1, s));
      } else {
        ns = (uint32_t)(plane * last);
      }
      k_node_ids<Off><<<blocks(ns), 256, 0, s>>>(nid + z0 * plane, idx, labels_in + z0 * plane,
                                                node_off_b.as<Off>(), size_b.as<uint32_t>(),
                                                nlab_b.as<uint32_t>(), ns, base,
                                                (Off)(z0 * plane), c + 4);
      base += slab_m[si];
    }
  }
  idx_b.release();
  if (nslabs > 1) {
    // stitch the slab faces: union of the node ids of face-adjacent voxels
    // with equal labels; the smallest node id of a set holds its root offset
    uint32_t* par = ptr_b.as<uint32_t>();
    uint32_t* fid = T_b.as<uint32_t>();
    uint8_t* isroot = flags_b.as<uint8_t>();
    k_cc_init<<<blocks(m), 256, 0, s>>>(par, m);
    for (int si = 1; si < nslabs; ++si) {
      const int64_t zb = si * sp;
      k_face_union<Off><<<blocks(plane), 256, 0, s>>>(labels_in, nid, (Off)((zb - 1) * plane),
                                                      (Off)(zb * plane), (uint32_t)plane, par);
    }
    k_node_flatten<<<blocks(m), 256, 0, s>>>(par, fid, isroot, m);
    {
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, fid, fid, (int64_t)m + 1, s);
      Scratch tmp(tb, s);
      SSLIC_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, fid, fid, (int64_t)m + 1, s));
    }
    const uint32_t mf = read_scalar(fid + m, s);
    k_nid_remap<Off><<<blocks(n64), 256, 0, s>>>(nid, par, fid, n);
    k_size_to_root<<<blocks(m), 256, 0, s>>>(m, par, size_b.as<uint32_t>(), c + 4);
    // keep the root entries, in place, in node order (= final id order)
    {
      Scratch nsel_b(sizeof(long long), s);
      long long* nsel = nsel_b.as<long long>();
      size_t tb = 0, t2 = 0, t3 = 0;
      cub::DeviceSelect::Flagged(nullptr, tb, node_off_b.as<Off>(), isroot, nsel, (int64_t)m, s);
      cub::DeviceSelect::Flagged(nullptr, t2, nlab_b.as<uint32_t>(), isroot, nsel, (int64_t)m, s);
      cub::DeviceSelect::Flagged(nullptr, t3, size_b.as<uint32_t>(), isroot, nsel, (int64_t)m, s);
      Scratch tmp(std::max(tb, std::max(t2, t3)), s);
      size_t tbb = std::max(tb, std::max(t2, t3));
      SSLIC_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp.p, tbb, node_off_b.as<Off>(), isroot, nsel,
                                                  (int64_t)m, s));
      tbb = std::max(tb, std::max(t2, t3));
      SSLIC_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp.p, tbb, nlab_b.as<uint32_t>(), isroot,
                                                  nsel, (int64_t)m, s));
      tbb = std::max(tb, std::max(t2, t3));
      SSLIC_CUDA_CHECK(cub::DeviceSelect::Flagged(tmp.p, tbb, size_b.as<uint32_t>(), isroot,
                                                  nsel, (int64_t)m, s));
    }
    SSLIC_CUDA_CHECK(cudaGetLastError());
    m = mf;
  }
  if (read_scalar(c + 4, s) != 0)
    throw Error(SSLIC_EINVAL, "enforce_connectivity: a component holds >= 2^32 voxels");
  stamp(1);
  const Off* node_off = node_off_b.as<Off>();
  const uint32_t* nlab = nlab_b.as<uint32_t>();
  uint32_t* size = size_b.as<uint32_t>();

  // ---- 2. finalize; 3. static pointers ----
  uint32_t *ptr = ptr_b.as<uint32_t>(), *T = T_b.as<uint32_t>(), *flab = flab_b.as<uint32_t>();
  uint8_t *flags = flags_b.as<uint8_t>(), *absn = absn_b.as<uint8_t>();
  const size_t kk = k ? k : 1;
  Scratch fcomp_b(kk * 4, s), te_b(kk * 4, s), te_new_b(kk * 4, s), factive_b(kk, s);
  uint32_t *fcomp = fcomp_b.as<uint32_t>(), *te = te_b.as<uint32_t>(),
           *te_new = te_new_b.as<uint32_t>();
  uint8_t* factive = factive_b.as<uint8_t>();
  SSLIC_CUDA_CHECK(cudaMemsetAsync(flags, 0, m, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(absn, 0, m, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(fcomp, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(te, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(te_new, 0xff, kk * 4, s));
  SSLIC_CUDA_CHECK(cudaMemsetAsync(factive, 1, kk, s));
  if (g.k > 0)
    k_finalize<Off><<<(unsigned)((g.k + 127) / 128), 128, 0, s>>>(g, labels_in, centers, nid, size,
                                                                   min_size, flags, fcomp);
  SSLIC_CUDA_CHECK(cudaGetLastError());
  const bool full_serial = m > 0 && (uint64_t)max_label >= (uint64_t)k;

  uint32_t next = k;
  bool done = false;
  if (!full_serial) {
    // distance back to the merge target -> ptr (flab doubles as its storage)
    SSLIC_CUDA_CHECK(cudaMemsetAsync(flab, 0xff, (size_t)m * 4, s));
    k_best_before<Off><<<blocks(n64), 256, 0, s>>>(cg, nid, node_off, flags, flab, cu + 0);
    k_pointers<Off><<<blocks(m), 256, 0, s>>>(m, min_size, nid, size, flab, node_off, cu + 0,
                                              flags, ptr, c + 1);
    SSLIC_CUDA_CHECK(cudaMemsetAsync(flab, 0, (size_t)m * 4, s));
    SSLIC_CUDA_CHECK(cudaGetLastError());
  }
  const bool serial = full_serial || read_scalar(c + 1, s) != 0;
  if (serial) {
    // exact sequential sweep on one device thread: the whole map (ids >= k)
    // or the pending cascade at the start of the raster
    if (full_serial && sizeof(Off) > 4)
      throw Error(SSLIC_EINVAL,
                  "enforce_connectivity: label ids >= k on >= 2^32 voxels (serial sweep) "
                  "are not supported");
    if (labels_out != labels_in)
      SSLIC_CUDA_CHECK(cudaMemcpyAsync(labels_out, labels_in, (size_t)n64 * 4,
                                       cudaMemcpyDeviceToDevice, s));
    Scratch mk_b((size_t)n64, s);
    uint8_t* mk = mk_b.as<uint8_t>();
    const Off qcap = (Off)std::min<int64_t>(n64, (int64_t)1 << 28);
    Scratch q_b((size_t)qcap * sizeof(Off), s);
    k_markers<Off><<<blocks(n64), 256, 0, s>>>(nid, flags, mk, n);
    k_sweep_serial<Off><<<1, 1, 0, s>>>(cg, labels_out, mk, q_b.as<Off>(), qcap, min_size, k,
                                        full_serial ? 1 : 0, cu + 1);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    unsigned long long res[3];
    SSLIC_CUDA_CHECK(cudaMemcpyAsync(res, cu + 1, sizeof(res), cudaMemcpyDeviceToHost, s));
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    if (res[2]) throw Error(SSLIC_ENOMEM, "enforce_connectivity: serial fill exceeds its queue");
    next = (uint32_t)res[1];
    if (res[0] >= (unsigned long long)n64) {
      done = true;
    } else {
      k_prefix_nodes<Off><<<blocks(m), 256, 0, s>>>(m, node_off, nlab, labels_out, mk, k, fcomp,
                                                    flags, ptr, flab, factive, c + 3);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      if (read_scalar(c + 3, s) != 0)
        throw Error(SSLIC_ELOGIC, "enforce_connectivity: inconsistent prefix state");
    }
  }
  stamp(2);
  int rounds = 0, jumps = 0;
  // List of the edge pass's candidate edges (12 bytes each). It lives in a
  // buffer of its own when the device has room for one edge per voxel beyond
  // a 4 GB reserve; otherwise in the OUTPUT map, which nothing reads between
  // here and k_output (which rewrites all of it, also when it aliases the
  // input): room for one edge per three voxels. If the edges outnumber the
  // room (or labels need 32 bits), every round scans the map.
  size_t mem_free = 0, mem_total = 0;
  SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));  // (the pool returns what was freed so far)
  if (cudaMemGetInfo(&mem_free, &mem_total) != cudaSuccess) mem_free = 0;
  const unsigned long long reserve = 4ull << 30;
  unsigned long long list_cap = (unsigned long long)n64 + 64;
  unsigned long long n_edges = 0;
  Scratch elist_b;
  uint32_t* ed = nullptr;
  bool use_list = !done && k < 0x80000000u && std::getenv("SSLIC_CC_NO_LIST") == nullptr;
  if (use_list) {
    if (std::getenv("SSLIC_CC_LIST_IN_OUTPUT") == nullptr && mem_free > reserve &&
        (mem_free - reserve) / 12 >= list_cap && elist_b.try_alloc((size_t)list_cap * 12, s)) {
      ed = elist_b.as<uint32_t>();
    } else {
      ed = labels_out;
      list_cap = (unsigned long long)n64 / 3;
    }
  }
  uint32_t* ex = ed + list_cap;
  uint32_t* el = ex + list_cap;
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
      if (rounds == 1 && use_list) {
        // (first round: list the candidate edges)
        k_edge_list<Off><<<blocks(n64), 256, 0, s>>>(cg, nid, flags, nlab, fcomp, factive, ed, ex,
                                                     el, list_cap, cu + 4);
        SSLIC_CUDA_CHECK(cudaGetLastError());
        n_edges = read_scalar(cu + 4, s);
        stamp(3);
        if (n_edges > list_cap) use_list = false;
      }
      if (use_list)
        k_edges_list<<<blocks((int64_t)n_edges), 256, 0, s>>>(ed, ex, el, n_edges, fcomp, T, te,
                                                              te_new, absn);
      else
        k_edges<Off><<<blocks(n64), 256, 0, s>>>(cg, nid, flags, nlab, fcomp, factive, T, te,
                                                 te_new, absn);
      SSLIC_CUDA_CHECK(cudaMemsetAsync(c + 2, 0, sizeof(unsigned), s));
      k_swap_te<<<blocks(kk), 256, 0, s>>>(k, te, te_new, c + 2);
      k_swap_abs<<<blocks(m), 256, 0, s>>>(m, flags, absn, c + 2);
      SSLIC_CUDA_CHECK(cudaGetLastError());
      if (read_scalar(c + 2, s) == 0) break;
    }
    // the last round left T consistent with the converged te / absorbed sets;
    // the event flags and their ranks reuse the (now dead) size array
    stamp(4);
    uint32_t* ev = size;  // m + 1 entries
    k_events<<<blocks(m), 256, 0, s>>>(m, flags, nlab, fcomp, factive, te, ev);
    {
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, ev, ev, (int64_t)m + 1, s);
      Scratch tmp(tb, s);
      SSLIC_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, ev, ev, (int64_t)m + 1, s));
    }
    k_final_labels<<<blocks(m), 256, 0, s>>>(m, flags, nlab, fcomp, factive, te, ev, next, flab);
    if (outs.max_label || outs.boundary)
      k_output_fused<Off><<<blocks(n64), 256, 0, s>>>(cg, nid, T, flab, labels_out,
                                                      outs.max_label, outs.boundary);
    else
      k_output<Off><<<blocks(n64), 256, 0, s>>>(nid, T, flab, labels_out, n);
    SSLIC_CUDA_CHECK(cudaGetLastError());
    next += read_scalar(ev + m, s);
  } else if (outs.max_label || outs.boundary) {  // the serial sweep wrote the map
    k_label_outputs<Off><<<blocks(n64), 256, 0, s>>>(cg, labels_out, outs.max_label,
                                                     outs.boundary);
    SSLIC_CUDA_CHECK(cudaGetLastError());
  }
  if (timing) {
    SSLIC_CUDA_CHECK(cudaStreamSynchronize(s));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr,
                 "[sslic] connectivity: %lld voxels, %u components, %d CCL slab(s), %s, %d "
                 "rounds (%s, %llu edges), %d jump passes, %.2f ms (ms from start: CCL %.1f, "
                 "node ids %.1f, pointers %.1f, edge list %.1f, rounds %.1f)\n",
                 (long long)n64, m, nslabs,
                 full_serial ? "serial (ids >= k)" : (serial ? "serial prefix" : "no prefix"),
                 rounds, use_list ? "edge list" : "map scans", n_edges, jumps,
                 std::chrono::duration<double, std::milli>(t1 - t0).count(), ph[0], ph[1], ph[2],
                 ph[3], ph[4]);
  }
  return next;
}

}  // namespace

uint32_t enforce_connectivity_device(const Geom& g, const uint32_t* labels_in,
                                     const double* centers, uint32_t* labels_out,
                                     cudaStream_t s, LabelOutputs outs) {
  int64_t n = 1;
  for (int a = 0; a < g.rank; ++a) n *= g.dims[a];
  // (SSLIC_CC_FORCE64=1: the 64-bit offset path on a small volume, for tests)
  if (n < ((int64_t)1 << 32) - 1 && std::getenv("SSLIC_CC_FORCE64") == nullptr)
    return connectivity_impl<uint32_t>(g, labels_in, centers, labels_out, s, outs);
  return connectivity_impl<uint64_t>(g, labels_in, centers, labels_out, s, outs);
}

void label_outputs_device(const Geom& g, const uint32_t* labels, LabelOutputs outs,
                          cudaStream_t s) {
  int64_t n = 1;
  for (int a = 0; a < g.rank; ++a) n *= g.dims[a];
  const int64_t last = g.dims[g.rank - 1];
  if (n < ((int64_t)1 << 32) - 1)
    k_label_outputs<uint32_t><<<blocks(n), 256, 0, s>>>(make_cg<uint32_t>(g, 0, last), labels,
                                                        outs.max_label, outs.boundary);
  else
    k_label_outputs<uint64_t><<<blocks(n), 256, 0, s>>>(make_cg<uint64_t>(g, 0, last), labels,
                                                        outs.max_label, outs.boundary);
  SSLIC_CUDA_CHECK(cudaGetLastError());
}

}  // namespace sslic_b200
