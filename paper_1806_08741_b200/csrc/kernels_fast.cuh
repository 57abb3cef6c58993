// K2 fast path: fused assign + delta-accumulate for rank 2/3, 1..4 channels,
// u8/u16/f32 volumes (configs 1-5). See DESIGN.md "K2".
//
// Work decomposition: one CTA per cell-aligned region (R_a = f_a * S_a voxels
// per axis). The region's candidate clusters are exactly those binned in the
// anchor cells within one cell of the region (any drift). Each
// candidate is staged once in shared memory as one record
//   [ sx[RXp] | sy[RY] | sz[RZ] | (c_hi, c_lo) per channel ]
// where s_a[x] = m^2 ((c_a - x)/S_a)^2 or +inf outside the cluster's window,
// which folds the window test into the arithmetic. Each warp sweeps 8x4x4
// voxel boxes (8x16 in 2D), each lane 4 consecutive voxels along x, against
// the candidates covering its box, two candidates per step with paired
// fp32x2 arithmetic and 3-input integer min/max.
//
// Exactness: the bulk distance evaluations run in fp32 (hi/lo split centre
// intensities, FMA allowed) with a rigorous error bound; the per-voxel argmin
// is decided in fp32 only when the runner-up is provably farther, and the
// carried-over comparison D* < d_old (slic.hpp:297) only when provably
// decided. Every other voxel is re-decided with the exact fp64 arithmetic of
// squared_distance_raw (slic.hpp:156-171) and the lexicographic (D, k) rule,
// so labels are bit-identical to the reference.
//
// Accumulation: the per-cluster sums are exact integers, so the kernel only
// emits DELTAS for voxels whose label value changed (+ new cluster, - old
// cluster); the engine keeps the running sums (k_update). Deltas are
// warp-aggregated per label (u32 reductions; f32 intensities as 2^-shift
// fixed point in three lanes), summed in CTA shared-memory int64 slots per
// candidate, and flushed with one global atomic per (cluster, component).
#pragma once

#include <cuda.h>  // CUtensorMap (TMA descriptors; built on the host, kernels_fast_main.cuh)

#include "common.cuh"
#include "kernels_exact.cuh"

namespace sslic_b200 {

constexpr int kFastThreads = 128;
constexpr int kFastMaxCand = 64;
constexpr int kFastMaxR = 64;  // max region extent per axis (spatial table width)
constexpr float kInf = __builtin_huge_valf();

struct FastParams {
  Geom g;
  const void* img;        // the sweep's image: native u8/u16/f32, or an f32 copy of f64 data
  const void* img_exact;  // the caller's image in g.dtype (fp64 re-decisions, f64 deltas)
  float pix_err;          // f64 inputs: bound of |v - fl32(v)| (scaled); 0 otherwise
  const double* centers;  // current table (fp64)
  const double* history;  // all tables, history[t * k * stride]
  const float2* hist32;   // hi/lo fp32 split of every table
  const int* chg;         // first table index from which centre k is unchanged
  const int* anchors;     // current anchors (kMaxRank per cluster)
  const int* cell_start;
  const int* items;
  uint32_t* labels;
  LabelCodec codec;
  uint32_t tag_now;
  int shift;
  unsigned long long* acc;       // int64 deltas
  unsigned long long* counters;  // [0] undefined, [5] fp64 re-decided, [6] crowded, [7] changed
  unsigned long long* eval_count;
  int R[3];           // region extent per axis (R[2] = 1 in 2D)
  int nreg[3];        // regions per axis (z counts only the slab)
  int64_t reg_z0;     // first global z plane of region row 0
  float margin;       // relative fp32 decision margin
  float abs_margin;   // absolute term (hi/lo split residue)
  float inv_grid[3];  // fl32(1/S_a) (d_old filter; its rounding is in the margin)
  double inv_grid64[3];
  const float2* cur32;      // hi/lo split of the current table (padded rows)
  float key_scale;          // 2^-k: fp32 distances are computed on scaled operands
  float key_scale2;         // 2^-2k
  const int* region_cand;   // per region: [count, ids...] (k_region_cand)
  int* region_cand_out;     // same buffer, written by k_region_cand
  int aligned4;       // dims[0] % 4 == 0: 4-voxel runs are vector-aligned
  int max_cand;       // regions with more candidates take the exact crowded path
  int skip_full;      // k_assign_fast: full regions were done by k_assign_lean
  int first;          // every label word of the slab is undefined (iteration 0 after a reset)
  float vmax;         // value range of the image (max |v|; dtype max for u8/u16)
  // TMA descriptors of the label words (dims0 x dims1 x slab planes, u32) and
  // the image (dims0*C x dims1 x data planes) for 8x4x4 box loads
  alignas(64) CUtensorMap tmap_words;
  alignas(64) CUtensorMap tmap_img;
};

// A region not clipped by the volume or the slab (k_assign_lean's domain).
__device__ __forceinline__ bool region_full(const FastParams& P, const int64_t* org, int RX,
                                            int RY, int RZ) {
  return org[0] + RX <= P.g.dims[0] && org[1] + RY <= P.g.dims[1] &&
         org[2] >= P.g.slab_begin && org[2] + RZ <= P.g.slab_end;
}

#ifndef SSLIC_BOX3_X  // (build-time override for layout experiments)
#define SSLIC_BOX3_X 8
#define SSLIC_BOX3_Y 4
#define SSLIC_BOX3_Z 4
#endif
template <int RANK>
struct BoxShape;
template <>
struct BoxShape<2> {
  static constexpr int X = 8, Y = 16, Z = 1;
};
template <>
struct BoxShape<3> {
  static constexpr int X = SSLIC_BOX3_X, Y = SSLIC_BOX3_Y, Z = SSLIC_BOX3_Z;
  static_assert(X * Y * Z == 128 && X % 4 == 0, "a warp box is 32 lanes x 4 voxels along x");
};

struct alignas(16) FastSmem {
  unsigned long long tma_bar[kFastThreads / 32][2];  // per warp, per box buffer (TMA loads)
  int n_cand;
  unsigned stats[3];  // k_assign_lean diagnostics (P.eval_count): fp64 re-decisions, label changes, evaluations
  int id[kFastMaxCand];
  short anc[kFastMaxCand][3];  // region-local anchors
  alignas(8) uint32_t wl[kFastThreads / 32][kFastMaxCand + 8];  // record offsets (floats)
  unsigned short htab[2 * kFastMaxCand];                               // cluster id -> slot
  float cpl[kFastMaxCand][3];        // centre coordinates relative to the region origin
  unsigned long long bmask[3][16];   // per axis and box index: candidates whose window overlaps
};

// 32-bit words of one lane's prefetched pixel run (4 voxels x C channels),
// 0 when the run exceeds one 16-byte cp.async (then pixels load directly)
__host__ __device__ constexpr int pf_pix_words(int C, int esize) {
  return 4 * C * esize <= 16 ? C * esize : 0;
}
__host__ __device__ constexpr int dtype_size(int dt) {
  return dt == SSLIC_U8 ? 1 : dt == SSLIC_U16 ? 2 : dt == SSLIC_F32 ? 4 : 8;
}

constexpr int kSlotHash = 2 * kFastMaxCand;
constexpr int kRegionCandStride = kFastMaxCand + 1;  // [count, ids...] per region
// float2 entries per hi/lo history row, padded to a 16-byte multiple
__host__ __device__ constexpr int hist32_stride(int stride) { return (stride + 1) & ~1; }
// Up to this many delta contributions per warp box, lanes add their own
// contributions (per-lane path); above it, a box dominated by one label is
// warp-aggregated per label. Measured per channel count: with native 32-bit
// shared atomics, 128 is faster for 1 and 4 channels (config 3 iteration 0
// 16.9 -> 16.6 ms, config 4 4.46 -> 4.15 ms), while the RGB configs, whose
// iteration 0 has many one-label boxes, keep 24 (config 2 iteration 0:
// 0.17 ms at 24, 0.41 ms at 128; config 5: 355 vs 372 ms).
__host__ __device__ constexpr unsigned sparse_deltas(int C) { return C == 3 ? 24u : 128u; }
__device__ __forceinline__ int slot_hash(uint32_t id) { return (int)((id * 0x9E3779B1u) >> 25); }
// Slot of cluster `id` in the region's candidate list, -1 if absent.
__device__ __forceinline__ int slot_of(const FastSmem& sm, uint32_t id) {
  int h = slot_hash(id);
  for (;;) {
    const int s = sm.htab[h];
    if (s == 0xffff) return -1;
    if ((uint32_t)sm.id[s] == id) return s;
    h = (h + 1) & (kSlotHash - 1);
  }
}

// x[i & 3] through predicated selects (inline PTX: a select chain written in
// C++ is turned into an indexed local-memory array by the compiler)
__device__ __forceinline__ uint32_t sel4(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                                         int i) {
  uint32_t r;
  asm("{\n\t.reg .pred p0, p1;\n\t.reg .b32 t0, t1;\n\t"
      "and.b32 t0, %5, 1;\n\tsetp.ne.b32 p0, t0, 0;\n\t"
      "and.b32 t1, %5, 2;\n\tsetp.ne.b32 p1, t1, 0;\n\t"
      "selp.b32 t0, %2, %1, p0;\n\tselp.b32 t1, %4, %3, p0;\n\t"
      "selp.b32 %0, t1, t0, p1;\n\t}"
      : "=r"(r)
      : "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(i));
  return r;
}
// (a[i & 3] for the 8 delta bits: i < 4 -> a, else b)
__device__ __forceinline__ uint32_t sel8(const uint32_t (&a)[4], const uint32_t (&b)[4], int i) {
  const uint32_t x = sel4(a[0], a[1], a[2], a[3], i), y = sel4(b[0], b[1], b[2], b[3], i);
  return i < 4 ? x : y;
}

// ---- fp32x2 (sm_100a paired FP32) --------------------------------------------
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// Keys: every fp32 distance is pre-scaled by 2^-2k (exact) so that real
// distances are < 2^-67 and any sum with uncovered-axis sentinels (2^-66
// each, at most 3) stays < 2^-63, i.e. below bit pattern 2^29. Then
// key = bits * 8 + j orders by (D, j) lexicographically with no mantissa
// lost, and is one IMAD (FMA pipe); keys >= kSentKey mean "not covered".
__device__ __forceinline__ uint32_t fkey(float d, uint32_t j) {
  return __float_as_uint(d) * 8u + j;
}
__device__ __forceinline__ float kval(uint32_t key) { return __uint_as_float(key >> 3); }
constexpr uint32_t kSentKey = 0x1E800000u * 8u;        // fkey(2^-66, 0)
constexpr float kSentinel = 1.3552527156068805e-20f;   // 2^-66
__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) {
  return min(min(a, b), c);
}

// Upper bound, over every voxel of a box, of the (scaled) fp32 distance to
// candidate j -- +inf unless j's window covers the whole box, so that every
// voxel of the box really evaluates j. A box that holds undefined voxels
// (d_old = +inf, slic.hpp:285-297 on a fresh DistanceMap) has no finite
// "largest carried-over distance" to prune against; the smallest such bound
// UB_r takes its place: a candidate k with LB_k > UB_r has D_k(v) > D_r(v) at
// every voxel, so the strict-minimum scan never picks k (iteration 0: the 3^n
// covering candidates drop to the ones that can win). crec = the record's
// (c_hi, c_lo) pairs; b0/b1 = the box's inclusive region-local extent.
template <int RANK, int C>
__device__ __forceinline__ float box_upper_bound(const FastSmem& sm, const float* crec, int j,
                                                 bool overlaps, const float* pmin,
                                                 const float* pmax, const int* b0, const int* b1,
                                                 const int* grid, const float* inv_grid,
                                                 float msq_scaled) {
  bool all = overlaps;
  float sl = 0.f;
#pragma unroll
  for (int a = 0; a < RANK; ++a) {
    const int an = sm.anc[j][a];
    all &= (an - grid[a] <= b0[a]) & (an + grid[a] >= b1[a]);
    const float cpl = sm.cpl[j][a];
    const float t = (fmaxf(cpl - (float)b0[a], (float)b1[a] - cpl) + 1e-3f) * inv_grid[a];
    sl = fmaf(t, t, sl);
  }
  float ub = sl * msq_scaled;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float ch = crec[2 * c], cl = fabsf(crec[2 * c + 1]);
    const float t = fmaxf(pmax[c] - ch, ch - pmin[c]) + cl;
    ub = fmaf(t, t, ub);
  }
  return all ? ub : kInf;
}

// Exact per-voxel decision over the region's candidate list (fp64, the
// reference arithmetic). full: lexicographic (D, k) argmin over all covering
// candidates; else only the fp32-certain winner jstar is re-evaluated.
static __device__ __noinline__ uint32_t exact_region_voxel(const FastParams& P, const FastSmem& sm,
                                                    int64_t x, int64_t y, int64_t z, int64_t di,
                                                    uint32_t word, bool full, int jstar,
                                                    const int64_t* org) {
  // sm.anc holds region-local anchors (relative to org)
  const Geom& g = P.g;
  const int64_t coord[kMaxRank] = {x, y, z, 0};
  double pix[4];
  for (int c = 0; c < g.channels; ++c) pix[c] = load_value(P.img_exact, g.dtype, di + c);
  double best_d = kInf;
  uint32_t best_k = kUndefined;
  if (full) {
    for (int j = 0; j < sm.n_cand; ++j) {
      bool covered = true;
      for (int a = 0; a < g.rank; ++a) {
        const int64_t dx = coord[a] - (org[a] + sm.anc[j][a]);
        if (dx < -g.grid[a] || dx > g.grid[a]) covered = false;
      }
      if (!covered) continue;
      const uint32_t kid = (uint32_t)sm.id[j];
      const double d = exact_distance(P.centers + (int64_t)kid * g.stride, pix, coord, g);
      if (d < best_d || (d == best_d && kid < best_k)) {
        best_d = d;
        best_k = kid;
      }
    }
  } else {
    best_k = (uint32_t)sm.id[jstar];
    best_d = exact_distance(P.centers + (int64_t)best_k * g.stride, pix, coord, g);
  }
  double d_old = kInf;
  if (word != kUndefined)
    d_old = exact_distance(
        P.history + ((int64_t)P.codec.tag(word) * g.k + P.codec.label(word)) * g.stride, pix,
        coord, g);
  if (best_k != kUndefined && best_d < d_old) return P.codec.pack(best_k, P.tag_now);
  return word;
}

// Crowded region (more than kFastMaxCand candidates): generic exact scan.
template <int RANK, int C>
__device__ __noinline__ void crowded_region(const FastParams& P, const int64_t* org,
                                            const int64_t* hi, int64_t zlo, int64_t zhi) {
  const Geom& g = P.g;
  const int RX = P.R[0], RY = P.R[1], RZ = P.R[2];
  const int64_t nvox = (int64_t)RX * RY * (RANK == 3 ? RZ : 1);
  for (int64_t base = 0; base < nvox; base += kFastThreads) {
    const int64_t i = base + threadIdx.x;
    int64_t coord[kMaxRank] = {0, 0, 0, 0};
    coord[0] = org[0] + i % RX;
    coord[1] = org[1] + (i / RX) % RY;
    coord[2] = RANK == 3 ? org[2] + i / ((int64_t)RX * RY) : 0;
    const bool valid = i < nvox && coord[0] <= hi[0] && coord[1] <= hi[1] &&
                       (RANK == 2 || (coord[2] >= zlo && coord[2] <= zhi));
    uint32_t lab = kUndefined, old = kUndefined;
    int64_t di = 0;
    if (valid) {
      const int64_t off = coord[0] + coord[1] * g.strides[1] + coord[2] * g.strides[2];
      const int64_t li = off - g.slab_begin * g.plane;
      di = data_index(g, off);
      uint32_t word = P.labels[li];
      old = P.codec.label(word);
      double pix[4];
      for (int c = 0; c < C; ++c) pix[c] = load_value(P.img_exact, g.dtype, di + c);
      double best_d = kInf;
      uint32_t best_k = kUndefined;
      int64_t clo[3], chi[3], cc[3];
      for (int a = 0; a < 3; ++a) {
        if (a < RANK) {
          const int64_t xc = coord[a] / g.grid[a];
          clo[a] = xc > 0 ? xc - 1 : 0;
          chi[a] = xc + 1 < g.cells[a] ? xc + 1 : g.cells[a] - 1;
        } else {
          clo[a] = chi[a] = 0;
        }
        cc[a] = clo[a];
      }
      for (;;) {
        const int64_t cell = (cc[2] * g.cells[1] + cc[1]) * g.cells[0] + cc[0];
        for (int it = P.cell_start[cell]; it < P.cell_start[cell + 1]; ++it) {
          const int kid = P.items[it];
          bool covered = true;
          for (int a = 0; a < RANK; ++a) {
            const int64_t dx = coord[a] - P.anchors[kid * kMaxRank + a];
            if (dx < -g.grid[a] || dx > g.grid[a]) covered = false;
          }
          if (!covered) continue;
          const double d = exact_distance(P.centers + (int64_t)kid * g.stride, pix, coord, g);
          if (d < best_d || (d == best_d && (uint32_t)kid < best_k)) {
            best_d = d;
            best_k = (uint32_t)kid;
          }
        }
        int a = 0;
        for (; a < RANK; ++a) {
          if (++cc[a] <= chi[a]) break;
          cc[a] = clo[a];
        }
        if (a == RANK) break;
      }
      double d_old = kInf;
      if (word != kUndefined)
        d_old = exact_distance(
            P.history + ((int64_t)P.codec.tag(word) * g.k + P.codec.label(word)) * g.stride, pix,
            coord, g);
      if (best_d < d_old) {
        word = P.codec.pack(best_k, P.tag_now);
        P.labels[li] = word;
      }
      lab = P.codec.label(word);
    }
    count_undefined(valid && lab == kUndefined, P.counters);
    const bool changed = valid && lab != old;
    warp_accumulate(g, P.shift, lab, changed, +1, P.img_exact, di, coord, P.acc);
    warp_accumulate(g, P.shift, old, changed, -1, P.img_exact, di, coord, P.acc);
  }
}

}  // namespace sslic_b200
