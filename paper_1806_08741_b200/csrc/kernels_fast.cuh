// K2 fast path: fused assign + delta-accumulate for rank 2/3, 1..4 channels,
// u8/u16/f32 volumes (configs 1-5). See DESIGN.md "K2".
//
// Work decomposition: one CTA per cell-aligned region (R_a = f_a * S_a voxels
// per axis). The region's candidate clusters are exactly those binned in the
// anchor cells within one cell of the region (any drift). Each
// candidate is staged once in shared memory as one record
//   [ (c_hi, c_hi, c_lo, c_lo) per channel | sx[RXp] | (sy,sy)[RY] | (sz,sz)[RZ] ]
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

#include "common.cuh"
#include "kernels_exact.cuh"

namespace sslic_b200 {

constexpr int kFastThreads = 128;
constexpr int kFastMaxCand = 64;
constexpr int kFastMaxR = 64;  // max region extent per axis (spatial table width)
constexpr float kInf = __builtin_huge_valf();

struct FastParams {
  Geom g;
  const void* img;
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
};

template <int RANK>
struct BoxShape {
  static constexpr int X = 8, Y = RANK == 3 ? 4 : 16, Z = RANK == 3 ? 4 : 1;
};

struct alignas(16) FastSmem {
  int n_cand;
  int overflow;
  int rs;  // record stride in floats
  int pad;
  int id[kFastMaxCand];
  int anc[kFastMaxCand][3];
  unsigned short wl[kFastThreads / 32][kFastMaxCand + 2];   // record offsets (floats)
  unsigned char wj[kFastThreads / 32][kFastMaxCand + 2];    // candidate slots
};

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

__device__ __forceinline__ uint32_t fkey(float d, uint32_t j) {
  return (__float_as_uint(d) & ~7u) | j;
}
__device__ __forceinline__ float kval(uint32_t key) { return __uint_as_float(key & ~7u); }
__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) {
  return min(min(a, b), c);
}

// Exact per-voxel decision over the region's candidate list (fp64, the
// reference arithmetic). full: lexicographic (D, k) argmin over all covering
// candidates; else only the fp32-certain winner jstar is re-evaluated.
static __device__ __noinline__ uint32_t exact_region_voxel(const FastParams& P, const FastSmem& sm,
                                                    int64_t x, int64_t y, int64_t z, int64_t di,
                                                    uint32_t word, bool full, int jstar) {
  const Geom& g = P.g;
  const int64_t coord[kMaxRank] = {x, y, z, 0};
  double pix[4];
  for (int c = 0; c < g.channels; ++c) pix[c] = load_value(P.img, g.dtype, di + c);
  double best_d = kInf;
  uint32_t best_k = kUndefined;
  if (full) {
    for (int j = 0; j < sm.n_cand; ++j) {
      bool covered = true;
      for (int a = 0; a < g.rank; ++a) {
        const int64_t dx = coord[a] - sm.anc[j][a];
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
      for (int c = 0; c < C; ++c) pix[c] = load_value(P.img, g.dtype, di + c);
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
    warp_accumulate(g, P.shift, lab, changed, +1, P.img, di, coord, P.acc);
    warp_accumulate(g, P.shift, old, changed, -1, P.img, di, coord, P.acc);
  }
}

template <int RANK, int C, typename T>
__global__ void __launch_bounds__(kFastThreads) k_assign_fast(FastParams P) {
  using Box = BoxShape<RANK>;
  constexpr int kStride = C + RANK;
  constexpr int kComp = kStride + 1;
  constexpr int kHdr = 4 * C;  // (hi, hi, lo, lo) per channel
  const Geom& g = P.g;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(smem_raw);
  const int RX = P.R[0], RY = P.R[1], RZ = RANK == 3 ? P.R[2] : 1;
  const int RXp = (RX + 3) & ~3;
  const int RS = (kHdr + RXp + 2 * RY + (RANK == 3 ? 2 * RZ : 0) + 3) & ~3;
  float* rec = reinterpret_cast<float*>(smem_raw + sizeof(FastSmem));  // [cand+1][RS]
  unsigned long long* accs =
      reinterpret_cast<unsigned long long*>(rec + (size_t)(kFastMaxCand + 1) * RS);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- region ----
  int64_t rb = blockIdx.x;
  const int rxi = (int)(rb % P.nreg[0]);
  rb /= P.nreg[0];
  const int ryi = (int)(rb % P.nreg[1]);
  rb /= P.nreg[1];
  const int rzi = (int)rb;
  const int64_t org[3] = {(int64_t)rxi * RX, (int64_t)ryi * RY,
                          RANK == 3 ? P.reg_z0 + (int64_t)rzi * RZ : 0};
  const int64_t hi[3] = {min(org[0] + RX, g.dims[0]) - 1, min(org[1] + RY, g.dims[1]) - 1,
                         RANK == 3 ? min(org[2] + RZ, g.dims[2]) - 1 : 0};
  const int64_t zlo = RANK == 3 ? max(org[2], g.slab_begin) : 0;
  const int64_t zhi = RANK == 3 ? min(hi[2], g.slab_end - 1) : 0;

  // ---- gather candidates (warp 0) ----
  if (warp == 0) {
    int clo[3], chi[3], nc = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (a < RANK) {
        const int64_t lo_a = a == 2 ? zlo : org[a];
        const int64_t hi_a = a == 2 ? zhi : hi[a];
        const int64_t l = lo_a - g.grid[a];
        clo[a] = l < 0 ? 0 : (int)(l / g.grid[a]);
        const int64_t h = (hi_a + g.grid[a]) / g.grid[a];
        chi[a] = h > g.cells[a] - 1 ? g.cells[a] - 1 : (int)h;
      } else {
        clo[a] = chi[a] = 0;
      }
      nc *= chi[a] - clo[a] + 1;
    }
    int total = 0;
    for (int base = 0; base < nc; base += 32) {
      const int i = base + lane;
      int cnt = 0, cstart = 0;
      if (i < nc) {
        const int nx = chi[0] - clo[0] + 1, ny = chi[1] - clo[1] + 1;
        const int cx = clo[0] + i % nx, cy = clo[1] + (i / nx) % ny, cz = clo[2] + i / (nx * ny);
        const int64_t cell = ((int64_t)cz * g.cells[1] + cy) * g.cells[0] + cx;
        cstart = P.cell_start[cell];
        cnt = P.cell_start[cell + 1] - cstart;
      }
      int incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int excl = total + incl - cnt;
      for (int q = 0; q < cnt; ++q)
        if (excl + q < kFastMaxCand) sm.id[excl + q] = P.items[cstart + q];
      total += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) {
      sm.n_cand = total < kFastMaxCand ? total : kFastMaxCand;
      sm.overflow = total > kFastMaxCand;
    }
  }
  __syncthreads();
  const int n = sm.n_cand;
  if (sm.overflow) {
    if (tid == 0) atomicAdd(P.counters + 6, 1ull);
    crowded_region<RANK, C>(P, org, hi, zlo, zhi);
    return;
  }

  // ---- stage candidate records (+ one all-inf padding record at slot n) ----
  for (int j = tid; j <= n; j += kFastThreads) {
    float* r = rec + (size_t)j * RS;
    if (j < n) {
      const int kid = sm.id[j];
      const double* ctr = P.centers + (int64_t)kid * g.stride;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float h = __double2float_rn(ctr[c]);
        const float l = __double2float_rn(ctr[c] - (double)h);
        r[4 * c] = h;
        r[4 * c + 1] = h;
        r[4 * c + 2] = l;
        r[4 * c + 3] = l;
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) sm.anc[j][a] = a < RANK ? P.anchors[kid * kMaxRank + a] : 0;
    } else {
#pragma unroll
      for (int c = 0; c < 4 * C; ++c) r[c] = 0.f;
    }
  }
  for (int i = tid; i < n * kComp; i += kFastThreads) accs[i] = 0ull;
  __syncthreads();
  {
    const int per = RX + RY + (RANK == 3 ? RZ : 0);
    for (int e = tid; e < (n + 1) * per; e += kFastThreads) {
      const int j = e / per;
      int r = e - j * per, a = 0;
      if (r >= RX) {
        r -= RX;
        a = 1;
        if (r >= RY) {
          r -= RY;
          a = 2;
        }
      }
      float v = kInf;
      if (j < n) {
        const int64_t x = (a == 0 ? org[0] : (a == 1 ? org[1] : org[2])) + r;
        const int kid = sm.id[j];
        const int an = a == 0 ? sm.anc[j][0] : (a == 1 ? sm.anc[j][1] : sm.anc[j][2]);
        const int s = g.grid[a];
        const int64_t dx = x - an;
        if (dx >= -s && dx <= s) {
          const double t = (P.centers[(int64_t)kid * g.stride + C + a] - (double)x) / (double)s;
          v = __double2float_rn(g.m_sq * (t * t));
        }
      }
      float* rj = rec + (size_t)j * RS + kHdr;
      if (a == 0) {
        rj[r] = v;
      } else if (a == 1) {
        rj[RXp + 2 * r] = v;
        rj[RXp + 2 * r + 1] = v;
      } else {
        rj[RXp + 2 * RY + 2 * r] = v;
        rj[RXp + 2 * RY + 2 * r + 1] = v;
      }
    }
  }
  __syncthreads();

  // ---- per-warp sweep over the region's boxes ----
  const int nbx = (RX + Box::X - 1) / Box::X, nby = (RY + Box::Y - 1) / Box::Y;
  const int nbz = RANK == 3 ? (RZ + Box::Z - 1) / Box::Z : 1;
  const int nbox = nbx * nby * nbz;
  const int xq = lane & 1;
  const int yq = RANK == 3 ? (lane >> 1) & 3 : lane >> 1;
  const int zq = RANK == 3 ? lane >> 3 : 0;
  const float M = P.margin;
  const float A = P.abs_margin;
  const float fscale = ldexpf(1.0f, P.shift);
  unsigned n_changed = 0, n_redecided = 0, n_evals = 0;

  for (int b = warp; b < nbox; b += kFastThreads / 32) {
    const int bx = b % nbx, by = (b / nbx) % nby, bz = b / (nbx * nby);
    const int lx0 = bx * Box::X + 4 * xq, ly = by * Box::Y + yq, lz = bz * Box::Z + zq;
    const int64_t gx0 = org[0] + lx0, gy = org[1] + ly, gz = org[2] + lz;
    const int64_t blo[3] = {org[0] + bx * Box::X, org[1] + by * Box::Y,
                            RANK == 3 ? max(org[2] + bz * Box::Z, zlo) : 0};
    const int64_t bhi[3] = {min(org[0] + bx * Box::X + Box::X - 1, hi[0]),
                            min(org[1] + by * Box::Y + Box::Y - 1, hi[1]),
                            RANK == 3 ? min(org[2] + bz * Box::Z + Box::Z - 1, zhi) : 0};
    if (blo[0] > bhi[0] || blo[1] > bhi[1] || blo[2] > bhi[2]) continue;  // uniform
    bool row_ok = gy <= hi[1] && ly < RY;
    if (RANK == 3) row_ok = row_ok && gz >= zlo && gz <= zhi && lz < RZ;
    bool valid[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) valid[v] = row_ok && lx0 + v < RX && gx0 + v <= hi[0];

    // candidates covering this box -> compact warp list (padded to even)
    __syncwarp();
    int nl;
    {
      bool cov[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        bool c = j < n;
        if (c) {
#pragma unroll
          for (int a = 0; a < RANK; ++a) {
            const int64_t an = sm.anc[j][a];
            if (an + g.grid[a] < blo[a] || an - g.grid[a] > bhi[a]) c = false;
          }
        }
        cov[h] = c;
      }
      const unsigned m0 = __ballot_sync(0xffffffffu, cov[0]);
      const unsigned m1 = __ballot_sync(0xffffffffu, cov[1]);
      const unsigned lt = (1u << lane) - 1u;
      if (cov[0]) {
        const int pos = __popc(m0 & lt);
        sm.wl[warp][pos] = (unsigned short)(lane * RS);
        sm.wj[warp][pos] = (unsigned char)lane;
      }
      if (cov[1]) {
        const int pos = __popc(m0) + __popc(m1 & lt);
        sm.wl[warp][pos] = (unsigned short)((lane + 32) * RS);
        sm.wj[warp][pos] = (unsigned char)(lane + 32);
      }
      nl = __popc(m0) + __popc(m1);
      if (lane == 0 && (nl & 1)) {
        sm.wl[warp][nl] = (unsigned short)(n * RS);  // all-inf padding record
        sm.wj[warp][nl] = (unsigned char)n;
      }
      __syncwarp();
    }
    const int nlp = (nl + 1) & ~1;
#pragma unroll
    for (int v = 0; v < 4; ++v) n_evals += valid[v] ? nl : 0;

    // pixels (paired per channel) and label words
    const int64_t off0 = gx0 + gy * g.strides[1] + (RANK == 3 ? gz * g.strides[2] : 0);
    const int64_t li0 = off0 - g.slab_begin * g.plane;
    const int64_t di0 = data_index(g, off0);
    float p[4][C];
    uint32_t word[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      word[v] = kUndefined;
#pragma unroll
      for (int c = 0; c < C; ++c) p[v][c] = 0.f;
      if (valid[v]) {
        word[v] = P.labels[li0 + v];
#pragma unroll
        for (int c = 0; c < C; ++c) p[v][c] = (float)static_cast<const T*>(P.img)[di0 + v * C + c];
      }
    }
    f2 p01[C], p23[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      p01[c] = pk2(p[0][c], p[1][c]);
      p23[c] = pk2(p[2][c], p[3][c]);
    }
    const int ox = kHdr + (lx0 < RXp ? lx0 : 0);
    const int oy = kHdr + RXp + 2 * (ly < RY ? ly : 0);
    const int oz = kHdr + RXp + 2 * RY + 2 * (lz < RZ ? lz : 0);

    // fp32 argmin with runner-up: keys = value with 3 low bits = index in group
    uint32_t best[4], second[4];
    int grp[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      best[v] = second[v] = 0xffffffffu;
      grp[v] = 0;
    }
    for (int g0 = 0; g0 < nlp; g0 += 8) {
      uint32_t before[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) before[v] = best[v];
      const int g1 = min(g0 + 8, nlp);
      for (int jj = g0; jj < g1; jj += 2) {
        uint32_t key[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float* r = rec + sm.wl[warp][jj + h];
          const ulonglong2 sxv = *reinterpret_cast<const ulonglong2*>(r + ox);
          f2 syz = *reinterpret_cast<const f2*>(r + oy);
          if (RANK == 3) syz = add2(syz, *reinterpret_cast<const f2*>(r + oz));
          f2 a01 = add2(sxv.x, syz), a23 = add2(sxv.y, syz);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const ulonglong2 hl = *reinterpret_cast<const ulonglong2*>(r + 4 * c);
            const f2 d01 = add2(sub2(hl.x, p01[c]), hl.y);
            const f2 d23 = add2(sub2(hl.x, p23[c]), hl.y);
            a01 = fma2(d01, d01, a01);
            a23 = fma2(d23, d23, a23);
          }
          float f0, f1, f2v, f3;
          up2(a01, f0, f1);
          up2(a23, f2v, f3);
          const uint32_t jl = (uint32_t)((jj + h) & 7);
          key[h][0] = fkey(f0, jl);
          key[h][1] = fkey(f1, jl);
          key[h][2] = fkey(f2v, jl);
          key[h][3] = fkey(f3, jl);
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t lo = min(key[0][v], key[1][v]);
          const uint32_t hk = max(key[0][v], key[1][v]);
          const uint32_t t = max(best[v], lo);
          best[v] = min(best[v], lo);
          second[v] = min3u(second[v], hk, t);
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (best[v] != before[v]) grp[v] = g0;
    }

    // ---- decisions ----
    uint32_t newl[4], oldl[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      oldl[v] = newl[v] = P.codec.label(word[v]);
      if (!valid[v]) continue;
      uint32_t w = word[v];
      const bool has_best = best[v] < 0x7f800000u;
      if (!has_best) continue;  // no window covers the voxel: keep the old label
      const int jstar = sm.wj[warp][grp[v] + (best[v] & 7u)];
      const float bv = kval(best[v]);
      const bool amb_cand = second[v] < 0x7f800000u && kval(second[v]) <= bv * (1.0f + M) + A;
      int decided = 0;  // 1 = update, 2 = keep, 0 = exact re-decision
      if (!amb_cand) {
        if (w == kUndefined) {
          decided = 1;
        } else {
          const uint32_t L = P.codec.label(w), Tg = P.codec.tag(w);
          if ((uint32_t)sm.id[jstar] == L && __ldg(P.chg + L) <= (int)Tg) {
            decided = 2;  // same centre as when the label was set: D* == d_old
          } else {
            const float2* hc = P.hist32 + ((int64_t)Tg * g.k + L) * kStride;
            float sp = 0.f;
#pragma unroll
            for (int a = 0; a < RANK; ++a) {
              const float2 cc = __ldg(hc + C + a);
              const float x = (float)(a == 0 ? gx0 + v : (a == 1 ? gy : gz));
              const float t = ((cc.x - x) + cc.y) / (float)g.grid[a];
              sp = fmaf(t, t, sp);
            }
            float dold = sp * (float)g.m_sq;
#pragma unroll
            for (int c = 0; c < C; ++c) {
              const float2 cc = __ldg(hc + c);
              const float d = (cc.x - p[v][c]) + cc.y;
              dold = fmaf(d, d, dold);
            }
            if (bv * (1.0f + M) + A < dold) decided = 1;
            else if (bv > dold * (1.0f + M) + A) decided = 2;
          }
        }
      }
      if (decided == 1) {
        w = P.codec.pack((uint32_t)sm.id[jstar], P.tag_now);
      } else if (decided == 0) {
        ++n_redecided;
        w = exact_region_voxel(P, sm, gx0 + v, gy, gz, di0 + v * C, w, amb_cand, jstar);
      }
      if (w != word[v]) P.labels[li0 + v] = w;
      newl[v] = P.codec.label(w);
    }

    // ---- delta accumulation: +new / -old for voxels whose label changed ----
    unsigned pending = 0;  // bit v: +new[v]; bit 4+v: -old[v]
    bool undef_any = false;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if (!valid[v]) continue;
      if (newl[v] == kUndefined) undef_any = true;
      if (newl[v] != oldl[v]) {
        pending |= 1u << v;
        if (oldl[v] != kUndefined) pending |= 1u << (4 + v);
        ++n_changed;
      }
    }
    if (__any_sync(0xffffffffu, undef_any)) {
      unsigned u = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) u += valid[v] && newl[v] == kUndefined;
      const unsigned tu = __reduce_add_sync(0xffffffffu, u);
      if (lane == 0) atomicAdd(P.counters, (unsigned long long)tu);  // slic.hpp:330-331
    }
    for (;;) {
      const unsigned any = __ballot_sync(0xffffffffu, pending != 0);
      if (!any) break;
      const int leader = __ffs(any) - 1;
      uint32_t mylab = 0;
      if (pending) {
        const int bit = __ffs(pending) - 1;
#pragma unroll
        for (int v = 0; v < 8; ++v)
          if (v == bit) mylab = v < 4 ? newl[v] : oldl[v - 4];
      }
      const uint32_t L = __shfl_sync(0xffffffffu, mylab, leader);
      int cnt = 0, sxr = 0, syr = 0, szr = 0;
      int64_t sv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) sv[c] = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int v = q & 3;
        const uint32_t lq = q < 4 ? newl[v] : oldl[v];
        if ((pending >> q & 1) && lq == L) {
          pending &= ~(1u << q);
          const int sgn = q < 4 ? 1 : -1;
          cnt += sgn;
          sxr += sgn * (lx0 + v);
          syr += sgn * ly;
          szr += sgn * lz;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            if (sizeof(T) < 4) sv[c] += sgn * (int64_t)p[v][c];
            else sv[c] += sgn * __float2ll_rn(p[v][c] * fscale);  // exact: |v| 2^s < 2^40
          }
        }
      }
      const int tc = (int)__reduce_add_sync(0xffffffffu, (uint32_t)cnt);
      const int tx = (int)__reduce_add_sync(0xffffffffu, (uint32_t)sxr);
      const int ty = (int)__reduce_add_sync(0xffffffffu, (uint32_t)syr);
      const int tz = RANK == 3 ? (int)__reduce_add_sync(0xffffffffu, (uint32_t)szr) : 0;
      long long tvs[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (sizeof(T) < 4) {
          tvs[c] = (int)__reduce_add_sync(0xffffffffu, (uint32_t)sv[c]);
        } else {
          const uint64_t u = (uint64_t)sv[c];
          const int32_t h = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(sv[c] >> 32));
          const uint32_t l1 = __reduce_add_sync(0xffffffffu, (uint32_t)(u & 0xffffu));
          const uint32_t l2 = __reduce_add_sync(0xffffffffu, (uint32_t)((u >> 16) & 0xffffu));
          tvs[c] = (long long)h * 4294967296LL + (long long)l2 * 65536LL + (long long)l1;
        }
      }
      if (lane == leader) {
        int S = -1;
        for (int j = 0; j < n; ++j)
          if ((uint32_t)sm.id[j] == L) {
            S = j;
            break;
          }
        if (S >= 0) {
          unsigned long long* a = accs + S * kComp;
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (tvs[c]) atomicAdd(a + c, (unsigned long long)tvs[c]);
          if (tx) atomicAdd(a + C, (unsigned long long)(long long)tx);
          if (ty) atomicAdd(a + C + 1, (unsigned long long)(long long)ty);
          if (RANK == 3 && tz) atomicAdd(a + C + 2, (unsigned long long)(long long)tz);
          if (tc) atomicAdd(a + kStride, (unsigned long long)(long long)tc);
        } else {
          // label outside the region's candidates: global, absolute coordinates
          unsigned long long* a = P.acc + (uint64_t)L * kComp;
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (tvs[c]) atomicAdd(a + c, (unsigned long long)tvs[c]);
          atomicAdd(a + C, (unsigned long long)(tx + (long long)tc * org[0]));
          atomicAdd(a + C + 1, (unsigned long long)(ty + (long long)tc * org[1]));
          if (RANK == 3) atomicAdd(a + C + 2, (unsigned long long)(tz + (long long)tc * org[2]));
          if (tc) atomicAdd(a + kStride, (unsigned long long)(long long)tc);
        }
      }
    }
  }
  if (P.eval_count) {
    const unsigned a = __reduce_add_sync(0xffffffffu, n_redecided);
    const unsigned c = __reduce_add_sync(0xffffffffu, n_changed);
    const unsigned e = __reduce_add_sync(0xffffffffu, n_evals);
    if (lane == 0) {
      atomicAdd(P.counters + 5, (unsigned long long)a);
      atomicAdd(P.counters + 7, (unsigned long long)c);
      atomicAdd(P.eval_count, (unsigned long long)e);
    }
  }
  __syncthreads();
  // ---- flush CTA slots (one global atomic per non-zero component) ----
  for (int e = tid; e < n * kComp; e += kFastThreads) {
    const int j = e / kComp, i = e - j * kComp;
    long long v = (long long)accs[e];
    if (i >= C && i < kStride) v += (long long)accs[j * kComp + kStride] * org[i - C];
    if (v) atomicAdd(P.acc + (uint64_t)sm.id[j] * kComp + i, (unsigned long long)v);
  }
}

// Evaluation count of the fast path (bench statistics): candidates per box x
// voxels is recorded by the host from the window volumes; this kernel only
// needs the counters above.

// hi/lo fp32 split of one centre table (for the fp32 d_old filter).
static __global__ void k_split32(const double* c, float2* out, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float h = __double2float_rn(c[i]);
  out[i] = make_float2(h, __double2float_rn(c[i] - (double)h));
}

inline bool fast_path_supported(const Geom& g) {
  if (g.rank != 2 && g.rank != 3) return false;
  if (g.channels < 1 || g.channels > 4) return false;
  if (g.dtype != SSLIC_U8 && g.dtype != SSLIC_U16 && g.dtype != SSLIC_F32) return false;
  for (int a = 0; a < g.rank; ++a)
    if (g.grid[a] > kFastMaxR) return false;
  if (g.k >= (int64_t)1 << 30) return false;
  return true;
}

// Region extent per axis: a multiple of S, at least 16 voxels (and <= 64).
inline int region_extent(int s) {
  int f = (16 + s - 1) / s;
  int r = f * s;
  while (r > kFastMaxR && f > 1) r = --f * s;
  return r;
}

inline size_t fast_smem_bytes(const Geom& g, const int* R) {
  const int RXp = (R[0] + 3) & ~3;
  const int RS = (4 * g.channels + RXp + 2 * R[1] + (g.rank == 3 ? 2 * R[2] : 0) + 3) & ~3;
  size_t b = sizeof(FastSmem);
  b += (size_t)(kFastMaxCand + 1) * RS * sizeof(float);
  b += (size_t)kFastMaxCand * (g.stride + 1) * sizeof(unsigned long long);
  return b;
}

template <int RANK, int C, typename T>
void launch_fast_t(const FastParams& P, size_t smem, int64_t nblocks, cudaStream_t s) {
  auto kern = k_assign_fast<RANK, C, T>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  kern<<<(unsigned)nblocks, kFastThreads, smem, s>>>(P);
}

template <int RANK, int C>
void launch_fast_c(const FastParams& P, size_t smem, int64_t nb, cudaStream_t s) {
  switch (P.g.dtype) {
    case SSLIC_U8: launch_fast_t<RANK, C, uint8_t>(P, smem, nb, s); break;
    case SSLIC_U16: launch_fast_t<RANK, C, uint16_t>(P, smem, nb, s); break;
    default: launch_fast_t<RANK, C, float>(P, smem, nb, s); break;
  }
}

template <int RANK>
void launch_fast_r(const FastParams& P, size_t smem, int64_t nb, cudaStream_t s) {
  switch (P.g.channels) {
    case 1: launch_fast_c<RANK, 1>(P, smem, nb, s); break;
    case 2: launch_fast_c<RANK, 2>(P, smem, nb, s); break;
    case 3: launch_fast_c<RANK, 3>(P, smem, nb, s); break;
    default: launch_fast_c<RANK, 4>(P, smem, nb, s); break;
  }
}

// Relative fp32 decision margin: each fp32
// distance is within (C + 10) u of the fp64 one (u = 2^-24) and keys are
// truncated by < 8 ulp (2^-20 relative); 2x for the two sides, 1.5x slack.
inline float fast_margin(int channels) {
  const double u = 1.0 / 16777216.0;
  return (float)(1.5 * (2.0 * (channels + 10) * u + 1.0 / 1048576.0));
}

inline void launch_fast_assign(FastParams P, cudaStream_t s) {
  const Geom& g = P.g;
  for (int a = 0; a < 3; ++a) P.R[a] = a < g.rank ? region_extent(g.grid[a]) : 1;
  P.nreg[0] = (int)((g.dims[0] + P.R[0] - 1) / P.R[0]);
  P.nreg[1] = (int)((g.dims[1] + P.R[1] - 1) / P.R[1]);
  if (g.rank == 3) {
    const int64_t z0 = g.slab_begin / P.R[2] * P.R[2];
    P.reg_z0 = z0;
    P.nreg[2] = (int)((g.slab_end - z0 + P.R[2] - 1) / P.R[2]);
  } else {
    P.reg_z0 = 0;
    P.nreg[2] = 1;
  }
  P.margin = fast_margin(g.channels);
  const int64_t nb = (int64_t)P.nreg[0] * P.nreg[1] * P.nreg[2];
  const size_t smem = fast_smem_bytes(g, P.R);
  if (g.rank == 3) launch_fast_r<3>(P, smem, nb, s);
  else launch_fast_r<2>(P, smem, nb, s);
}

}  // namespace sslic_b200
