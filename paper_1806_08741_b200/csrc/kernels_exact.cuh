// Exact, general kernels of the SSLIC hot path (any rank 1..4, any channel
// count, any dtype). These are the bit-exact building blocks:
//   * init/perturb          (slic.hpp:206-267, color.hpp:71-102)
//   * anchor-cell binning   (candidate search structure for assignment)
//   * assign+accumulate     (slic.hpp:275-346), pixel-centric, fp64 exact
//   * update                (slic.hpp:352-372)
// The tuned fast-path assignment kernel lives in kernels_fast.cuh and falls
// back to these routines' arithmetic for every near-tie.
#pragma once

#include "common.cuh"

namespace sslic_b200 {

// ---------------------------------------------------------------------------
// K1: init_centers + perturb_centers, one thread per cluster.
// ---------------------------------------------------------------------------
static __device__ inline double gradient_sq_at(const Geom& g, const void* img, const int64_t* coord) {
  // color.hpp:71-102: axes in order, channels in order; h = 2 central,
  // h = 1 one-sided at borders; axes of extent 1 skipped.
  int64_t base = 0;
  for (int a = 0; a < g.rank; ++a) base += coord[a] * g.strides[a];
  double acc = 0.0;
  for (int a = 0; a < g.rank; ++a) {
    if (g.dims[a] == 1) continue;
    int64_t lo = base, hi = base;
    double h = 2.0;
    if (coord[a] == 0) {
      hi += g.strides[a];
      h = 1.0;
    } else if (coord[a] == g.dims[a] - 1) {
      lo -= g.strides[a];
      h = 1.0;
    } else {
      hi += g.strides[a];
      lo -= g.strides[a];
    }
    const int64_t ih = data_index(g, hi), il = data_index(g, lo);
    for (int c = 0; c < g.channels; ++c) {
      const double d =
          __ddiv_rn(__dsub_rn(load_value(img, g.dtype, ih + c), load_value(img, g.dtype, il + c)), h);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  return acc;
}

// (z0 <= z1: only the clusters whose initial centre lies in planes [z0, z1)
// are written, the others are left as they are -- the pipelined start of
// run_slic perturbs the clusters chunk by chunk as the image arrives)
static __global__ void k_init_perturb(Geom g, const void* img, double* centers, int perturb,
                                      int64_t z0 = 0, int64_t z1 = -1) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= g.k) return;
  if (z0 <= z1) {
    const int last = g.rank - 1;
    const int64_t zc = id / (g.k / g.cells[last]);
    int64_t z = zc * g.grid[last] + g.grid[last] / 2;
    if (z > g.dims[last] - 1) z = g.dims[last] - 1;
    if (z < z0 || z >= z1) return;
  }
  double* ctr = centers + id * g.stride;
  int64_t coord[kMaxRank];
  int64_t rem = id;
  for (int a = 0; a < g.rank; ++a) {  // row-major cell enumeration (slic.hpp:220)
    const int64_t cell = rem % g.cells[a];
    rem /= g.cells[a];
    int64_t x = cell * g.grid[a] + g.grid[a] / 2;
    if (x > g.dims[a] - 1) x = g.dims[a] - 1;
    coord[a] = x;
  }
  const int last = g.rank - 1;
  if (coord[last] < g.slab_begin || coord[last] >= g.slab_end) {
    for (int i = 0; i < g.stride; ++i) ctr[i] = 0.0;  // owned by another slab
    return;
  }
  int64_t best[kMaxRank];
  for (int a = 0; a < g.rank; ++a) best[a] = coord[a];
  if (perturb) {
    // slic.hpp:236-267: clamped 3^n hood, row-major, first strict minimum.
    int64_t lo[kMaxRank], hi[kMaxRank], cur[kMaxRank];
    for (int a = 0; a < g.rank; ++a) {
      lo[a] = coord[a] - 1 < 0 ? 0 : coord[a] - 1;
      hi[a] = coord[a] + 1 > g.dims[a] - 1 ? g.dims[a] - 1 : coord[a] + 1;
      cur[a] = lo[a];
    }
    bool first = true;
    double best_g = 0.0;
    for (;;) {
      const double gv = gradient_sq_at(g, img, cur);
      if (first || gv < best_g) {
        first = false;
        best_g = gv;
        for (int a = 0; a < g.rank; ++a) best[a] = cur[a];
      }
      int a = 0;
      for (; a < g.rank; ++a) {
        if (++cur[a] <= hi[a]) break;
        cur[a] = lo[a];
      }
      if (a == g.rank) break;
    }
  }
  int64_t off = 0;
  for (int a = 0; a < g.rank; ++a) off += best[a] * g.strides[a];
  const int64_t di = data_index(g, off);
  for (int c = 0; c < g.channels; ++c) ctr[c] = load_value(img, g.dtype, di + c);
  for (int a = 0; a < g.rank; ++a) ctr[g.channels + a] = (double)best[a];
}

// Perturbation of a caller-given table (sslic_perturb_centers): same hood
// rule around llround(centre).
static __global__ void k_perturb_table(Geom g, const void* img, double* centers) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= g.k) return;
  double* ctr = centers + id * g.stride;
  int64_t lo[kMaxRank], hi[kMaxRank], cur[kMaxRank], best[kMaxRank];
  bool empty = false;
  for (int a = 0; a < g.rank; ++a) {
    const int64_t anchor = anchor_of(ctr[g.channels + a]);
    int64_t l = anchor - 1, h = anchor + 2;  // clamp_region (image.hpp:158-167)
    l = l < 0 ? 0 : (l > g.dims[a] ? g.dims[a] : l);
    h = h < l ? l : (h > g.dims[a] ? g.dims[a] : h);
    lo[a] = l;
    hi[a] = h - 1;
    if (hi[a] < lo[a]) empty = true;
    cur[a] = lo[a];
  }
  if (empty) return;  // the reference would read an unset coordinate; keep the centre
  bool first = true;
  double best_g = 0.0;
  for (;;) {
    const double gv = gradient_sq_at(g, img, cur);
    if (first || gv < best_g) {
      first = false;
      best_g = gv;
      for (int a = 0; a < g.rank; ++a) best[a] = cur[a];
    }
    int a = 0;
    for (; a < g.rank; ++a) {
      if (++cur[a] <= hi[a]) break;
      cur[a] = lo[a];
    }
    if (a == g.rank) break;
  }
  int64_t off = 0;
  for (int a = 0; a < g.rank; ++a) off += best[a] * g.strides[a];
  const int64_t di = data_index(g, off);
  for (int c = 0; c < g.channels; ++c) ctr[c] = load_value(img, g.dtype, di + c);
  for (int a = 0; a < g.rank; ++a) ctr[g.channels + a] = (double)best[a];
}

static __global__ void k_gradient_points(Geom g, const void* img, const int64_t* coords, int64_t n,
                                  double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = gradient_sq_at(g, img, coords + i * g.rank);
}

static __global__ void k_distance_points(Geom g, int64_t n, const double* centers, const double* pixels,
                                  const int64_t* coords, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = exact_distance(centers + i * g.stride, pixels + i * g.channels, coords + i * g.rank, g);
}

// ---------------------------------------------------------------------------
// Anchor-cell binning: cluster k's window [anchor-S, anchor+S] covers voxel x
// only if anchor's cell (anchor / S, clamped into the grid) is within one cell
// of x's cell, so the candidates of a voxel are exactly the clusters binned in
// its 3^rank cell neighbourhood — under any drift.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t clamp_cell(int64_t a, int s, int cells) {
  int64_t c = a >= 0 ? a / s : -1;
  return c < 0 ? 0 : (c >= cells ? cells - 1 : c);
}

static __global__ void k_anchors(Geom g, const double* centers, int* anchors, int* cell_of,
                          int* cell_count) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= g.k) return;
  int64_t cell = 0, mul = 1;
  for (int a = 0; a < g.rank; ++a) {
    const int64_t an = anchor_of(centers[id * g.stride + g.channels + a]);
    anchors[id * kMaxRank + a] = (int)an;
    cell += clamp_cell(an, g.grid[a], g.cells[a]) * mul;
    mul *= g.cells[a];
  }
  for (int a = g.rank; a < kMaxRank; ++a) anchors[id * kMaxRank + a] = 0;
  cell_of[id] = (int)cell;
  atomicAdd(cell_count + cell, 1);
}

// Identity anchor-cell bins (cluster k in cell k, one per cell): the bins
// commit() builds at iteration 0 whenever perturbation cannot move an anchor
// out of its initial cell (Engine::pipeline_ok).
static __global__ void k_identity_bins(int64_t ncells, int* cell_start, int* items) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncells) return;
  cell_start[c] = (int)c;
  if (c < ncells) items[c] = (int)c;
}

// Anchors and the hi/lo fp32 split (padded rows of s2 float2) of the clusters
// whose initial centre lies in planes [z0, z1) (pipelined start).
static __global__ void k_anchors_split_range(Geom g, const double* centers, int* anchors,
                                             float2* split, int s2, int64_t z0, int64_t z1) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= g.k) return;
  const int last = g.rank - 1;
  const int64_t zc = id / (g.k / g.cells[last]);
  int64_t z = zc * g.grid[last] + g.grid[last] / 2;
  if (z > g.dims[last] - 1) z = g.dims[last] - 1;
  if (z < z0 || z >= z1) return;
  for (int a = 0; a < kMaxRank; ++a)
    anchors[id * kMaxRank + a] =
        a < g.rank ? (int)anchor_of(centers[id * g.stride + g.channels + a]) : 0;
  for (int i = 0; i < s2; ++i) {
    if (i >= g.stride) {
      split[id * s2 + i] = make_float2(0.f, 0.f);
      continue;
    }
    const double v = centers[id * g.stride + i];
    const float h = __double2float_rn(v);
    split[id * s2 + i] = make_float2(h, __double2float_rn(v - (double)h));
  }
}

static __global__ void k_bin_fill(int64_t k, const int* cell_of, const int* cell_start, int* cursor,
                           int* items) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= k) return;
  const int c = cell_of[id];
  const int pos = atomicAdd(cursor + c, 1);
  items[cell_start[c] + pos] = (int)id;
}

// Ascending cluster ids in items[b, e): insertion sort for the usual one or
// two clusters per cell, heapsort (O(n log n)) for crowded cells.
__device__ __forceinline__ void sort_cell(int* items, int b, int e) {
  if (e - b > 32) {
    int* a = items + b;
    const int n = e - b;
    auto sift = [&](int root, int end) {
      for (;;) {
        int child = 2 * root + 1;
        if (child >= end) return;
        if (child + 1 < end && a[child + 1] > a[child]) ++child;
        if (a[root] >= a[child]) return;
        const int t = a[root];
        a[root] = a[child];
        a[child] = t;
        root = child;
      }
    };
    for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
    for (int end = n - 1; end > 0; --end) {
      const int t = a[0];
      a[0] = a[end];
      a[end] = t;
      sift(0, end);
    }
    return;
  }
  for (int i = b + 1; i < e; ++i) {
    const int v = items[i];
    int j = i - 1;
    while (j >= b && items[j] > v) {
      items[j + 1] = items[j];
      --j;
    }
    items[j + 1] = v;
  }
}

// Deterministic order inside each cell (ascending cluster id).
static __global__ void k_bin_sort(int64_t ncells, const int* cell_start, int* items) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int b = cell_start[c], e = cell_start[c + 1];
  if (e - b > 32) {  // crowded cell (degenerate tables): heapsort, O(n log n) worst case
    int* a = items + b;
    const int n = e - b;
    auto sift = [&](int root, int end) {
      for (;;) {
        int child = 2 * root + 1;
        if (child >= end) return;
        if (child + 1 < end && a[child + 1] > a[child]) ++child;
        if (a[root] >= a[child]) return;
        const int t = a[root];
        a[root] = a[child];
        a[child] = t;
        root = child;
      }
    };
    for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
    for (int end = n - 1; end > 0; --end) {
      const int t = a[0];
      a[0] = a[end];
      a[end] = t;
      sift(0, end);
    }
    return;
  }
  for (int i = b + 1; i < e; ++i) {  // typical cells hold one or two clusters
    const int v = items[i];
    int j = i - 1;
    while (j >= b && items[j] > v) {
      items[j + 1] = items[j];
      --j;
    }
    items[j + 1] = v;
  }
}

// ---------------------------------------------------------------------------
// Label words. Tag mode packs (iteration tag, label) into one uint32 so no
// per-voxel distance buffer is needed: d_old is recomputed exactly from the
// centre table of the iteration that set the label.
// ---------------------------------------------------------------------------


// Warp-aggregated accumulation of one voxel's joint vector into the
// per-cluster int64 accumulator acc[label*(stride+1) + ...] (ClusterAccumulatorMap,
// slic.hpp:108-149). Integer sums are exact and associative, so the result is
// independent of the order and of the slab/GPU decomposition.
static __device__ inline void count_undefined(bool undef, unsigned long long* undefined_count) {
  const unsigned full = __activemask();
  const unsigned undef_mask = __ballot_sync(full, undef);
  if (undef_mask && (threadIdx.x & 31) == __ffs(undef_mask) - 1)
    atomicAdd(undefined_count, (unsigned long long)__popc(undef_mask));
}

// sign = +1 adds the voxel's joint vector to cluster `label`, -1 removes it
// (delta accumulation: exact because the sums are integers).
static __device__ inline void warp_accumulate(const Geom& g, int shift, uint32_t label, bool valid,
                                              int sign, const void* img, int64_t di,
                                              const int64_t* coord, unsigned long long* acc) {
  const unsigned full = __activemask();
  const int lane = threadIdx.x & 31;
  valid = valid && label != kUndefined;
  unsigned todo = __ballot_sync(full, valid);
  while (todo) {
    const int leader = __ffs(todo) - 1;
    const uint32_t lab = __shfl_sync(full, label, leader);
    const bool mine = valid && label == lab;
    const unsigned grp = __ballot_sync(full, mine);
    unsigned long long* dst = acc + (uint64_t)lab * (g.stride + 1);
    for (int i = 0; i <= g.stride; ++i) {
      long long v = 0;
      if (mine) {
        if (i < g.channels) v = to_fixed(load_value(img, g.dtype, di + i), shift);
        else if (i < g.stride) v = coord[i - g.channels];
        else v = 1;
        v *= sign;
      }
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(full, v, o);
      if (lane == leader && v != 0) atomicAdd(dst + i, (unsigned long long)v);
    }
    todo &= ~grp;
  }
}

// ---------------------------------------------------------------------------
// K2 (exact): one thread per voxel of the slab, candidates from the 3^rank
// anchor-cell neighbourhood, lexicographic (D, k) minimum (equivalent to the
// reference's ascending-k strict-< scan, slic.hpp:285-297), strict < against
// the carried-over distance. DIST=true keeps an explicit fp64 DistanceMap
// (the compat path); DIST=false recomputes d_old from the history table.
// ACC: fuse accumulate_region.
// ---------------------------------------------------------------------------
template <bool DIST, bool ACC>
static __global__ void __launch_bounds__(256) k_assign_exact(
    Geom g, const void* img, const double* centers, const double* history, const int* anchors,
    const int* cell_start, const int* items, uint32_t* labels, double* dists, LabelCodec codec,
    uint32_t tag_now, int shift, unsigned long long* acc, unsigned long long* undefined_count,
    unsigned long long* eval_count) {
  const int64_t nslab = (g.slab_end - g.slab_begin) * g.plane;
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = li < nslab;
  const int64_t off = li + g.slab_begin * g.plane;
  int64_t coord[kMaxRank] = {0, 0, 0, 0};
  int64_t di = 0;
  uint32_t word = kUndefined;
  uint32_t out_label = kUndefined, old_label = kUndefined;
  unsigned evals = 0;
  if (valid) {
    int64_t rem = off;
    for (int a = 0; a < g.rank; ++a) {
      coord[a] = rem % g.dims[a];
      rem /= g.dims[a];
    }
    di = data_index(g, off);
    double pix[8];
    const int cached = g.channels < 8 ? g.channels : 8;
    for (int c = 0; c < cached; ++c) pix[c] = load_value(img, g.dtype, di + c);

    // Candidate scan over the clamped 3^rank cell neighbourhood.
    int64_t clo[kMaxRank], chi[kMaxRank], cc[kMaxRank];
    for (int a = 0; a < kMaxRank; ++a) {
      if (a < g.rank) {
        const int64_t xc = coord[a] / g.grid[a];
        clo[a] = xc > 0 ? xc - 1 : 0;
        chi[a] = xc + 1 < g.cells[a] ? xc + 1 : g.cells[a] - 1;
      } else {
        clo[a] = chi[a] = 0;
      }
      cc[a] = clo[a];
    }
    double best_d = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    uint32_t best_k = kUndefined;
    for (;;) {
      int64_t cell = 0, mul = 1;
      for (int a = 0; a < g.rank; ++a) {
        cell += cc[a] * mul;
        mul *= g.cells[a];
      }
      for (int it = cell_start[cell]; it < cell_start[cell + 1]; ++it) {
        const int kid = items[it];
        bool covered = true;
        for (int a = 0; a < g.rank; ++a) {
          const int64_t dx = coord[a] - anchors[kid * kMaxRank + a];
          if (dx < -g.grid[a] || dx > g.grid[a]) covered = false;
        }
        if (!covered) continue;
        ++evals;
        const double* ctr = centers + (int64_t)kid * g.stride;
        double color = 0.0;
        for (int c = 0; c < g.channels; ++c) {
          const double p = c < 8 ? pix[c] : load_value(img, g.dtype, di + c);
          const double d = __dsub_rn(ctr[c], p);
          color = __dadd_rn(color, __dmul_rn(d, d));
        }
        double spatial = 0.0;
        for (int a = 0; a < g.rank; ++a) {
          const double d =
              __ddiv_rn(__dsub_rn(ctr[g.channels + a], (double)coord[a]), (double)g.grid[a]);
          spatial = __dadd_rn(spatial, __dmul_rn(d, d));
        }
        const double dist = __dadd_rn(color, __dmul_rn(g.m_sq, spatial));
        if (dist < best_d || (dist == best_d && (uint32_t)kid < best_k)) {
          best_d = dist;
          best_k = (uint32_t)kid;
        }
      }
      int a = 0;
      for (; a < g.rank; ++a) {
        if (++cc[a] <= chi[a]) break;
        cc[a] = clo[a];
      }
      if (a == g.rank) break;
    }

    word = labels[li];
    old_label = codec.label(word);
    double d_old;
    if (DIST) {
      d_old = dists[li];
    } else if (word == kUndefined) {
      d_old = __longlong_as_double(0x7ff0000000000000LL);
    } else {
      const double* hc =
          history + ((int64_t)codec.tag(word) * g.k + codec.label(word)) * g.stride;
      double color = 0.0;
      for (int c = 0; c < g.channels; ++c) {
        const double p = c < 8 ? pix[c] : load_value(img, g.dtype, di + c);
        const double d = __dsub_rn(hc[c], p);
        color = __dadd_rn(color, __dmul_rn(d, d));
      }
      double spatial = 0.0;
      for (int a = 0; a < g.rank; ++a) {
        const double d =
            __ddiv_rn(__dsub_rn(hc[g.channels + a], (double)coord[a]), (double)g.grid[a]);
        spatial = __dadd_rn(spatial, __dmul_rn(d, d));
      }
      d_old = __dadd_rn(color, __dmul_rn(g.m_sq, spatial));
    }
    if (best_d < d_old) {  // strict (slic.hpp:297)
      word = codec.pack(best_k, tag_now);
      labels[li] = word;
      if (DIST) dists[li] = best_d;
    }
    out_label = codec.label(word);
  }
  if (ACC) {
    // delta accumulation into the persistent integer sums: only voxels whose
    // label value changed contribute (+ new cluster, - old cluster).
    count_undefined(valid && out_label == kUndefined, undefined_count);
    const bool changed = valid && out_label != old_label;
    warp_accumulate(g, shift, out_label, changed, +1, img, di, coord, acc);
    warp_accumulate(g, shift, old_label, changed, -1, img, di, coord, acc);
  }
  if (eval_count) {
    unsigned s = evals;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(eval_count, (unsigned long long)s);
  }
}

// accumulate_region only (sslic_accumulate and the exact update path).
static __global__ void __launch_bounds__(256) k_accumulate(Geom g, const void* img,
                                                    const uint32_t* labels, LabelCodec codec,
                                                    int shift, unsigned long long* acc,
                                                    unsigned long long* undefined_count,
                                                    unsigned long long* out_of_range) {
  const int64_t nslab = (g.slab_end - g.slab_begin) * g.plane;
  const int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool valid = li < nslab;
  const int64_t off = li + g.slab_begin * g.plane;
  int64_t coord[kMaxRank] = {0, 0, 0, 0};
  uint32_t lab = kUndefined;
  int64_t di = 0;
  bool ok = valid;
  if (valid) {
    int64_t rem = off;
    for (int a = 0; a < g.rank; ++a) {
      coord[a] = rem % g.dims[a];
      rem /= g.dims[a];
    }
    di = data_index(g, off);
    lab = codec.label(labels[li]);
    if (lab != kUndefined && (int64_t)lab >= g.k) {
      atomicAdd(out_of_range, 1ull);
      ok = false;
    }
  }
  count_undefined(ok && lab == kUndefined, undefined_count);
  warp_accumulate(g, shift, lab, ok, +1, img, di, coord, acc);
}

// ---------------------------------------------------------------------------
// K3: reduce_and_update (slic.hpp:352-372). One thread per cluster; the
// per-cluster squared displacement is reduced in a fixed tree order
// (deterministic; the reference's sequential (k, i) order is not reproduced
// bit-for-bit).
// ---------------------------------------------------------------------------
static __global__ void k_update(Geom g, int shift, const unsigned long long* delta,
                                unsigned long long* sums, const double* old_c, double* new_c,
                                double* block_partials, int* chg, int next_table) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double part = 0.0;
  if (id < g.k) {
    // persistent exact integer sums += this iteration's (allreduced) deltas
    long long* a = reinterpret_cast<long long*>(sums) + id * (g.stride + 1);
    const long long* dl = reinterpret_cast<const long long*>(delta) + id * (g.stride + 1);
    for (int i = 0; i <= g.stride; ++i) a[i] += dl[i];
    const long long cnt = a[g.stride];
    const double* o = old_c + id * g.stride;
    double* n = new_c + id * g.stride;
    bool changed = false;
    if (cnt == 0) {
      for (int i = 0; i < g.stride; ++i) n[i] = o[i];
    } else {
      const double dc = (double)cnt;
      for (int i = 0; i < g.stride; ++i) {
        const double s = i < g.channels ? ldexp((double)a[i], -shift) : (double)a[i];
        const double v = __ddiv_rn(s, dc);
        const double d = __dsub_rn(v, o[i]);
        part = __dadd_rn(part, __dmul_rn(d, d));
        changed |= __double_as_longlong(v) != __double_as_longlong(o[i]);
        n[i] = v;
      }
    }
    // chg[k]: first table index from which centre k is bitwise unchanged
    if (chg && changed) chg[id] = next_table;
  }
  __shared__ double red[256];
  red[threadIdx.x] = part;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) block_partials[blockIdx.x] = red[0];
}

// One cluster of the fused update (k_update_fused, k_update_bins_small):
// sums += deltas (deltas re-zeroed), the new centre (count > 0) or the old
// one, chg, the hi/lo fp32 split row, the anchors; adds (new-old)^2 to *part
// and returns the anchor cell.
__device__ __forceinline__ int update_cluster(const Geom& g, int shift, unsigned long long* delta,
                                              unsigned long long* sums, const double* old_c,
                                              double* new_c, int* chg, int next_table,
                                              float2* split_out, int split_stride, int* anchors,
                                              int64_t id, double* part) {
  long long* a = reinterpret_cast<long long*>(sums) + id * (g.stride + 1);
  long long* dl = reinterpret_cast<long long*>(delta) + id * (g.stride + 1);
  for (int i = 0; i <= g.stride; ++i) {
    a[i] += dl[i];
    dl[i] = 0;
  }
  const long long cnt = a[g.stride];
  const double* o = old_c + id * g.stride;
  double* n = new_c + id * g.stride;
  bool changed = false;
  float2* sp = split_out + id * split_stride;
  for (int i = 0; i < g.stride; ++i) {
    double v = o[i];
    if (cnt != 0) {
      const double s = i < g.channels ? ldexp((double)a[i], -shift) : (double)a[i];
      v = __ddiv_rn(s, (double)cnt);
      const double d = __dsub_rn(v, o[i]);
      *part = __dadd_rn(*part, __dmul_rn(d, d));
      changed |= __double_as_longlong(v) != __double_as_longlong(o[i]);
    }
    n[i] = v;
    const float h = __double2float_rn(v);
    sp[i] = make_float2(h, __double2float_rn(v - (double)h));
  }
  for (int i = g.stride; i < split_stride; ++i) sp[i] = make_float2(0.f, 0.f);
  if (changed) chg[id] = next_table;
  int64_t cell = 0, mul = 1;
  for (int ax = 0; ax < g.rank; ++ax) {
    const int64_t an = anchor_of(n[g.channels + ax]);
    anchors[id * kMaxRank + ax] = (int)an;
    cell += clamp_cell(an, g.grid[ax], g.cells[ax]) * mul;
    mul *= g.cells[ax];
  }
  for (int ax = g.rank; ax < kMaxRank; ++ax) anchors[id * kMaxRank + ax] = 0;
  return (int)cell;
}

// Fused update for the tag-mode loop (one launch instead of update +
// residual + anchors + hi/lo split): sums += deltas and the deltas are
// zeroed for the next iteration; new centre (count > 0) or unchanged; chg;
// the new table's hi/lo fp32 split row; anchors + anchor-cell counts for the
// bins; the residual by a last-block reduction (fixed order: deterministic).
// cell_count must be zero on entry (k_bin_sort_reset leaves it so).
static __global__ void k_update_fused(Geom g, int shift, unsigned long long* delta,
                                      unsigned long long* sums, const double* old_c,
                                      double* new_c, double* block_partials, int* chg,
                                      int next_table, float2* split_out, int split_stride,
                                      int* anchors, int* cell_of, int* cell_count,
                                      unsigned* done, double* residual_out,
                                      const unsigned long long* undefined_count,
                                      unsigned* undefined_seen) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id == 0 && *undefined_count) *undefined_seen = 1u;  // latched for run_slic
  double part = 0.0;
  if (id < g.k) {
    const int cell = update_cluster(g, shift, delta, sums, old_c, new_c, chg, next_table,
                                    split_out, split_stride, anchors, id, &part);
    cell_of[id] = cell;
    atomicAdd(cell_count + cell, 1);
  }
  __shared__ double red[256];
  __shared__ bool last;
  red[threadIdx.x] = part;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    block_partials[blockIdx.x] = red[0];
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
    t = __dadd_rn(t, *((volatile double*)block_partials + i));
  red[threadIdx.x] = t;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *residual_out = sqrt(red[0]);
    *done = 0;  // ready for the next launch
  }
}

// k_bin_sort that also re-zeroes the cell counters and fill cursors for the
// next k_update_fused / k_bin_fill.
static __global__ void k_bin_sort_reset(int64_t ncells, const int* cell_start, int* items,
                                        int* cell_count, int* cursor) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncells) return;
  cell_count[c] = 0;
  if (c == ncells) return;
  cursor[c] = 0;
  const int b = cell_start[c], e = cell_start[c + 1];
  if (e - b > 32) {  // crowded cell (degenerate tables): heapsort, O(n log n) worst case
    int* a = items + b;
    const int n = e - b;
    auto sift = [&](int root, int end) {
      for (;;) {
        int child = 2 * root + 1;
        if (child >= end) return;
        if (child + 1 < end && a[child + 1] > a[child]) ++child;
        if (a[root] >= a[child]) return;
        const int t = a[root];
        a[root] = a[child];
        a[child] = t;
        root = child;
      }
    };
    for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
    for (int end = n - 1; end > 0; --end) {
      const int t = a[0];
      a[0] = a[end];
      a[end] = t;
      sift(0, end);
    }
    return;
  }
  for (int i = b + 1; i < e; ++i) {  // typical cells hold one or two clusters
    const int v = items[i];
    int j = i - 1;
    while (j >= b && items[j] > v) {
      items[j + 1] = items[j];
      --j;
    }
    items[j + 1] = v;
  }
}

static __global__ void k_residual_final(const double* block_partials, int nblocks, double* residual_out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) s = __dadd_rn(s, block_partials[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + st]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *residual_out = sqrt(red[0]);
}

static __global__ void k_f64_to_f32(const double* in, float* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = __double2float_rn(in[i]);
}

static __global__ void k_fill_f64(double* p, int64_t n, double v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// Strip iteration tags: plain LabelMap values.
static __global__ void k_unpack_labels(int64_t n, const uint32_t* words, LabelCodec codec,
                                uint32_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = codec.label(words[i]);
}

// max |v| over the stored image values (fixed-point scale selection).
static __global__ void k_absmax(const void* img, int dtype, int64_t n, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(load_value(img, dtype, i)));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Algorithmic evaluation count sum_k |W_k ∩ slab| (window clamped to the
// image and to the slab), for the roofline's E.
static __global__ void k_window_volume(Geom g, const int* anchors, unsigned long long* out) {
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  unsigned long long vol = 0;
  if (id < g.k) {
    vol = 1;
    for (int a = 0; a < g.rank; ++a) {
      int64_t lo = (int64_t)anchors[id * kMaxRank + a] - g.grid[a];
      int64_t hi = (int64_t)anchors[id * kMaxRank + a] + g.grid[a] + 1;
      int64_t blo = 0, bhi = g.dims[a];
      if (a == g.rank - 1) {
        blo = g.slab_begin;
        bhi = g.slab_end;
      }
      lo = lo < blo ? blo : lo;
      hi = hi > bhi ? bhi : hi;
      vol *= (unsigned long long)(hi > lo ? hi - lo : 0);
    }
  }
  for (int o = 16; o > 0; o >>= 1) vol += __shfl_xor_sync(0xffffffffu, vol, o);
  if ((threadIdx.x & 31) == 0 && vol) atomicAdd(out, vol);
}

}  // namespace sslic_b200
