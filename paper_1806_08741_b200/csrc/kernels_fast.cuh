// K2 fast path: fused assign + accumulate for rank 2/3, 1..4 channels,
// u8/u16/f32 volumes (configs 1-5). See DESIGN.md "K2".
//
// Work decomposition: one CTA per cell-aligned region (R_a = f_a * S_a voxels
// per axis). The region's candidate clusters are exactly those binned in the
// anchor cells within one cell of the region (any drift); they
// are staged once in shared memory together with per-axis spatial tables
// sx[j][x] = m^2 ((c_x - x)/S_x)^2 (or +inf outside cluster j's window, which
// folds the window test into the arithmetic). Each warp sweeps 8x4x4 voxel
// boxes (16x... in 2D), each lane 4 consecutive voxels along x, against the
// candidates covering its box.
//
// Exactness: the bulk distance evaluations run in fp32 (hi/lo split centre
// intensities, FMA allowed) with a rigorous error bound; the per-voxel argmin
// is decided in fp32 only when the runner-up is provably farther, and the
// carried-over comparison D* < d_old (slic.hpp:297) only when provably
// decided. Every other voxel is re-decided with the exact fp64 arithmetic of
// squared_distance_raw (slic.hpp:156-171) and the lexicographic (D, k) rule,
// so labels are bit-identical to the reference.
//
// Accumulation: warp-level aggregation of equal labels (u32 reductions; f32
// intensities as 2^-shift fixed point split in three 16/32-bit lanes), CTA
// shared-memory int64 slots per candidate, one global int64 atomic per
// (cluster, component) per CTA at the end. Stale labels outside the region's
// candidates go straight to global atomics.
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
  unsigned long long* acc;
  unsigned long long* counters;  // [0] undefined, [5] ambiguous (stats), [6] overflow blocks
  unsigned long long* eval_count;
  int R[3];           // region extent per axis (3D; R[2] = 1 in 2D)
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
  int id[kFastMaxCand];
  int anc[kFastMaxCand][3];
  unsigned char wl[kFastThreads / 32][kFastMaxCand];
};

__device__ __forceinline__ uint32_t fkey(float d, uint32_t j) {
  return (__float_as_uint(d) & ~7u) | j;
}
__device__ __forceinline__ float kval(uint32_t key) { return __uint_as_float(key & ~7u); }

template <typename T>
__device__ __forceinline__ float to_f(T v) { return (float)v; }

// Exact per-voxel decision over the region's candidate list (fp64, the
// reference arithmetic). Returns the new label word and the winner's slot.
__device__ inline uint32_t exact_region_voxel(const FastParams& P, const FastSmem& sm,
                                              const int64_t* coord, int64_t di, uint32_t word,
                                              bool full, int jstar, int* slot_out) {
  const Geom& g = P.g;
  double pix[4];
  for (int c = 0; c < g.channels; ++c) pix[c] = load_value(P.img, g.dtype, di + c);
  double best_d = kInf;
  uint32_t best_k = kUndefined;
  int best_j = -1;
  auto dist_of = [&](const double* ctr) {
    double color = 0.0;
    for (int c = 0; c < g.channels; ++c) {
      const double d = __dsub_rn(ctr[c], pix[c]);
      color = __dadd_rn(color, __dmul_rn(d, d));
    }
    double spatial = 0.0;
    for (int a = 0; a < g.rank; ++a) {
      const double d =
          __ddiv_rn(__dsub_rn(ctr[g.channels + a], (double)coord[a]), (double)g.grid[a]);
      spatial = __dadd_rn(spatial, __dmul_rn(d, d));
    }
    return __dadd_rn(color, __dmul_rn(g.m_sq, spatial));
  };
  if (full) {
    for (int j = 0; j < sm.n_cand; ++j) {
      bool covered = true;
      for (int a = 0; a < g.rank; ++a) {
        const int64_t dx = coord[a] - sm.anc[j][a];
        if (dx < -g.grid[a] || dx > g.grid[a]) covered = false;
      }
      if (!covered) continue;
      const uint32_t kid = (uint32_t)sm.id[j];
      const double d = dist_of(P.centers + (int64_t)kid * g.stride);
      if (d < best_d || (d == best_d && kid < best_k)) {
        best_d = d;
        best_k = kid;
        best_j = j;
      }
    }
  } else {
    best_j = jstar;
    best_k = (uint32_t)sm.id[jstar];
    best_d = dist_of(P.centers + (int64_t)best_k * g.stride);
  }
  double d_old = kInf;
  if (word != kUndefined)
    d_old = dist_of(P.history +
                    ((int64_t)P.codec.tag(word) * g.k + P.codec.label(word)) * g.stride);
  if (best_j >= 0 && best_d < d_old) {
    *slot_out = best_j;
    return P.codec.pack(best_k, P.tag_now);
  }
  *slot_out = -2;  // unchanged: caller resolves the slot of the old label
  return word;
}

template <int RANK, int C, typename T>
__global__ void __launch_bounds__(kFastThreads) k_assign_fast(FastParams P) {
  using Box = BoxShape<RANK>;
  constexpr int kStride = C + RANK;
  constexpr int kComp = kStride + 1;
  const Geom& g = P.g;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(smem_raw);
  const int RX = P.R[0], RY = P.R[1], RZ = P.R[2];
  const int RXp = (RX + 3) & ~3;
  float* cvh = reinterpret_cast<float*>(smem_raw + sizeof(FastSmem));  // [cand][C]
  float* cvl = cvh + kFastMaxCand * C;
  float* sx = cvl + kFastMaxCand * C;                                   // [cand][RXp]
  float* sy = sx + kFastMaxCand * RXp;                                  // [cand][RY]
  float* sz = sy + kFastMaxCand * RY;                                   // [cand][RZ]
  unsigned long long* accs =
      reinterpret_cast<unsigned long long*>(sz + kFastMaxCand * (RANK == 3 ? RZ : 1));
  // accs may be misaligned for 8-byte access: align up
  accs = reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(accs) + 7) & ~uintptr_t(7));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- region ----
  int64_t rb = blockIdx.x;
  const int rxi = (int)(rb % P.nreg[0]);
  rb /= P.nreg[0];
  const int ryi = (int)(rb % P.nreg[1]);
  rb /= P.nreg[1];
  const int rzi = (int)rb;
  int64_t org[3] = {(int64_t)rxi * RX, (int64_t)ryi * RY,
                    RANK == 3 ? P.reg_z0 + (int64_t)rzi * RZ : 0};
  int64_t hi[3];  // inclusive last coordinate of the region inside the image
  hi[0] = min(org[0] + RX, g.dims[0]) - 1;
  hi[1] = min(org[1] + RY, g.dims[1]) - 1;
  hi[2] = RANK == 3 ? min(org[2] + RZ, g.dims[2]) - 1 : 0;
  const int64_t zlo = RANK == 3 ? max(org[2], g.slab_begin) : 0;
  const int64_t zhi = RANK == 3 ? min(hi[2], g.slab_end - 1) : 0;

  // ---- gather candidates (warp 0) ----
  if (warp == 0) {
    int clo[3], chi[3], nc = 1;
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
    // Crowded region (heavy drift): exact generic per-voxel scan.
    if (tid == 0) atomicAdd(P.counters + 6, 1ull);
    const int64_t nvox = (int64_t)RX * RY * (RANK == 3 ? RZ : 1);
    for (int64_t base = 0; base < nvox; base += kFastThreads) {
      const int64_t i = base + tid;
      int64_t coord[kMaxRank] = {0, 0, 0, 0};
      coord[0] = org[0] + i % RX;
      coord[1] = org[1] + (i / RX) % RY;
      coord[2] = RANK == 3 ? org[2] + i / ((int64_t)RX * RY) : 0;
      const bool valid = i < nvox && coord[0] <= hi[0] && coord[1] <= hi[1] &&
                         (RANK == 2 || (coord[2] >= zlo && coord[2] <= zhi));
      uint32_t lab = kUndefined;
      int64_t di = 0;
      if (valid) {
        const int64_t off = coord[0] + coord[1] * g.strides[1] + coord[2] * g.strides[2];
        const int64_t li = off - g.slab_begin * g.plane;
        di = data_index(g, off);
        uint32_t word = P.labels[li];
        // generic candidate scan over the 3^rank anchor-cell hood
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
              P.history + ((int64_t)P.codec.tag(word) * g.k + P.codec.label(word)) * g.stride,
              pix, coord, g);
        if (best_d < d_old) {
          word = P.codec.pack(best_k, P.tag_now);
          P.labels[li] = word;
        }
        lab = P.codec.label(word);
      }
      warp_accumulate(g, P.shift, lab, valid, P.img, di, coord, P.acc, P.counters);
    }
    return;
  }

  // ---- stage candidates: centres (hi/lo fp32), anchors, spatial tables ----
  for (int j = tid; j < n; j += kFastThreads) {
    const int kid = sm.id[j];
    const double* ctr = P.centers + (int64_t)kid * g.stride;
    for (int c = 0; c < C; ++c) {
      const float h = __double2float_rn(ctr[c]);
      cvh[j * C + c] = h;
      cvl[j * C + c] = __double2float_rn(ctr[c] - (double)h);
    }
    for (int a = 0; a < 3; ++a) sm.anc[j][a] = a < RANK ? P.anchors[kid * kMaxRank + a] : 0;
  }
  for (int j = 0; j < n; ++j)
    for (int i = tid; i < kComp; i += kFastThreads) accs[j * kComp + i] = 0ull;
  __syncthreads();
  {
    const int RZt = RANK == 3 ? RZ : 0;
    const int per = RX + RY + RZt;
    for (int e = tid; e < n * per; e += kFastThreads) {
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
      const int64_t x = org[a] + r;
      const int kid = sm.id[j];
      const double cpos = P.centers[(int64_t)kid * g.stride + C + a];
      const int64_t dx = x - sm.anc[j][a];
      float v = kInf;
      if (dx >= -g.grid[a] && dx <= g.grid[a]) {
        const double t = (cpos - (double)x) / (double)g.grid[a];
        v = __double2float_rn(g.m_sq * (t * t));
      }
      if (a == 0) sx[j * RXp + r] = v;
      else if (a == 1) sy[j * RY + r] = v;
      else sz[j * RZ + r] = v;
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

  for (int b = warp; b < nbox; b += kFastThreads / 32) {
    const int bx = b % nbx, by = (b / nbx) % nby, bz = b / (nbx * nby);
    const int lx0 = bx * Box::X + 4 * xq, ly = by * Box::Y + yq, lz = bz * Box::Z + zq;
    const int64_t gx0 = org[0] + lx0, gy = org[1] + ly, gz = org[2] + lz;
    // box bounds (global, clipped) for the warp's candidate culling
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

    // candidates covering this box -> compact warp list
    unsigned m0, m1;
    __syncwarp();  // previous box's readers of wl are done
    {
      bool c0 = false, c1 = false;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        bool cov = j < n;
        if (cov) {
          for (int a = 0; a < RANK; ++a) {
            const int64_t an = sm.anc[j][a];
            if (an + g.grid[a] < blo[a] || an - g.grid[a] > bhi[a]) cov = false;
          }
        }
        if (h == 0) c0 = cov;
        else c1 = cov;
      }
      m0 = __ballot_sync(0xffffffffu, c0);
      m1 = __ballot_sync(0xffffffffu, c1);
      const unsigned lt = (1u << lane) - 1u;
      if (c0) sm.wl[warp][__popc(m0 & lt)] = (unsigned char)lane;
      if (c1) sm.wl[warp][__popc(m0) + __popc(m1 & lt)] = (unsigned char)(lane + 32);
      __syncwarp();
    }
    const int nl = __popc(m0) + __popc(m1);

    // pixels and label words
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
        for (int c = 0; c < C; ++c)
          p[v][c] = to_f(static_cast<const T*>(P.img)[di0 + v * C + c]);
      }
    }

    // fp32 argmin with runner-up (keys: value with 3 low bits = index in group)
    uint32_t best[4], second[4];
    int grp[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      best[v] = second[v] = 0xffffffffu;
      grp[v] = 0;
    }
    for (int g0 = 0; g0 < nl; g0 += 8) {
      uint32_t before[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) before[v] = best[v];
      const int g1 = min(g0 + 8, nl);
      for (int jj = g0; jj < g1; ++jj) {
        const int j = sm.wl[warp][jj];
        float syz = sy[j * RY + (ly < RY ? ly : 0)];
        if (RANK == 3) syz += sz[j * RZ + (lz < RZ ? lz : 0)];
        const float4 s4 = *reinterpret_cast<const float4*>(sx + j * RXp + (lx0 < RXp ? lx0 : 0));
        const float sxv[4] = {s4.x, s4.y, s4.z, s4.w};
        float ch[C], cl[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          ch[c] = cvh[j * C + c];
          cl[c] = cvl[j * C + c];
        }
        const uint32_t jl = (uint32_t)(jj & 7);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          float acc = sxv[v] + syz;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const float d = (ch[c] - p[v][c]) + cl[c];
            acc = fmaf(d, d, acc);
          }
          const uint32_t key = fkey(acc, jl);
          const uint32_t t = max(best[v], key);
          best[v] = min(best[v], key);
          second[v] = min(second[v], t);
        }
      }
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (best[v] != before[v]) grp[v] = g0;
    }

    // decisions
    uint32_t lab_out[4];
    int slot[4];
    unsigned amb_count = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      lab_out[v] = kUndefined;
      slot[v] = -1;
      if (!valid[v]) continue;
      const int64_t li = li0 + v;
      uint32_t w = word[v];
      const bool has_best = best[v] < 0x7f800000u;
      const int jstar = has_best ? sm.wl[warp][grp[v] + (best[v] & 7u)] : -1;
      const float bv = kval(best[v]);
      const bool amb_cand = has_best && second[v] < 0x7f800000u &&
                            kval(second[v]) <= bv * (1.0f + M) + A;
      int decided = 0;  // 1 = update, 2 = keep, 0 = exact needed
      if (!has_best) {
        decided = 2;
      } else if (!amb_cand) {
        if (w == kUndefined) {
          decided = 1;
        } else {
          const uint32_t L = P.codec.label(w), Tg = P.codec.tag(w);
          if ((uint32_t)sm.id[jstar] == L && P.chg[L] <= (int)Tg) {
            decided = 2;  // same centre as when the label was set: D* == d_old
          } else {
            const float2* hc = P.hist32 + ((int64_t)Tg * g.k + L) * kStride;
            float dold = 0.f;
#pragma unroll
            for (int a = 0; a < RANK; ++a) {
              const float2 cc = hc[C + a];
              const float x = (float)(a == 0 ? gx0 + v : (a == 1 ? gy : gz));
              const float t = ((cc.x - x) + cc.y) / (float)g.grid[a];
              dold = fmaf(t, t, dold);
            }
            dold *= (float)g.m_sq;
#pragma unroll
            for (int c = 0; c < C; ++c) {
              const float2 cc = hc[c];
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
        P.labels[li] = w;
        slot[v] = jstar;
      } else if (decided == 0) {
        ++amb_count;
        int64_t coord[kMaxRank] = {gx0 + v, gy, gz, 0};
        int s;
        const uint32_t nw =
            exact_region_voxel(P, sm, coord, data_index(g, off0 + v), w, amb_cand, jstar, &s);
        if (nw != w) {
          w = nw;
          P.labels[li] = w;
          slot[v] = s;
        }
      }
      lab_out[v] = P.codec.label(w);
      if (slot[v] < 0 && lab_out[v] != kUndefined) {
        if (jstar >= 0 && (uint32_t)sm.id[jstar] == lab_out[v]) {
          slot[v] = jstar;
        } else {
          slot[v] = -1;
          for (int j = 0; j < n; ++j)
            if ((uint32_t)sm.id[j] == lab_out[v]) {
              slot[v] = j;
              break;
            }
        }
      }
    }
    if (P.eval_count) {
      const unsigned a = __reduce_add_sync(0xffffffffu, amb_count);
      unsigned nv = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) nv += valid[v];
      const unsigned tv = __reduce_add_sync(0xffffffffu, nv);
      if (lane == 0) {
        atomicAdd(P.eval_count, (unsigned long long)tv * nl);
        atomicAdd(P.counters + 5, (unsigned long long)a);
      }
    }

    // ---- warp-aggregated accumulation into CTA slots ----
    unsigned pending = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if (valid[v] && lab_out[v] == kUndefined) {
        atomicAdd(P.counters, 1ull);  // slic.hpp:330-331 (reported by the host)
      } else if (valid[v]) {
        pending |= 1u << v;
      }
    }
    for (;;) {
      const unsigned any = __ballot_sync(0xffffffffu, pending != 0);
      if (!any) break;
      const int leader = __ffs(any) - 1;
      const int myv = pending ? __ffs(pending) - 1 : 0;
      uint32_t mylab = 0;
      int myslot = -1;
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (v == myv) {
          mylab = lab_out[v];
          myslot = slot[v];
        }
      const uint32_t L = __shfl_sync(0xffffffffu, mylab, leader);
      const int S = __shfl_sync(0xffffffffu, myslot, leader);
      uint32_t cnt = 0, sxr = 0;
      int64_t sv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) sv[c] = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if ((pending >> v & 1) && lab_out[v] == L) {
          pending &= ~(1u << v);
          ++cnt;
          sxr += (uint32_t)(lx0 + v);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            if (sizeof(T) < 4) sv[c] += (int64_t)p[v][c];
            else sv[c] += __float2ll_rn(p[v][c] * fscale);  // exact: |v| 2^shift < 2^40
          }
        }
      }
      const uint32_t tc = __reduce_add_sync(0xffffffffu, cnt);
      const uint32_t tx = __reduce_add_sync(0xffffffffu, sxr);
      const uint32_t ty = __reduce_add_sync(0xffffffffu, cnt * (uint32_t)ly);
      const uint32_t tz = RANK == 3 ? __reduce_add_sync(0xffffffffu, cnt * (uint32_t)lz) : 0u;
      long long tvs[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (sizeof(T) < 4) {
          tvs[c] = (long long)__reduce_add_sync(0xffffffffu, (uint32_t)sv[c]);
        } else {
          const uint64_t u = (uint64_t)sv[c];
          const int32_t h = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(sv[c] >> 32));
          const uint32_t l1 = __reduce_add_sync(0xffffffffu, (uint32_t)(u & 0xffffu));
          const uint32_t l2 = __reduce_add_sync(0xffffffffu, (uint32_t)((u >> 16) & 0xffffu));
          tvs[c] = (long long)h * 4294967296LL + (long long)l2 * 65536LL + (long long)l1;
        }
      }
      if (lane == leader) {
        if (S >= 0) {
          unsigned long long* a = accs + S * kComp;
#pragma unroll
          for (int c = 0; c < C; ++c) atomicAdd(a + c, (unsigned long long)tvs[c]);
          atomicAdd(a + C, (unsigned long long)tx);
          atomicAdd(a + C + 1, (unsigned long long)ty);
          if (RANK == 3) atomicAdd(a + C + 2, (unsigned long long)tz);
          atomicAdd(a + kStride, (unsigned long long)tc);
        } else {
          // stale label outside the region's candidates: global, absolute coords
          unsigned long long* a = P.acc + (uint64_t)L * kComp;
#pragma unroll
          for (int c = 0; c < C; ++c) atomicAdd(a + c, (unsigned long long)tvs[c]);
          atomicAdd(a + C, (unsigned long long)(tx + (uint64_t)tc * org[0]));
          atomicAdd(a + C + 1, (unsigned long long)(ty + (uint64_t)tc * org[1]));
          if (RANK == 3) atomicAdd(a + C + 2, (unsigned long long)(tz + (uint64_t)tc * org[2]));
          atomicAdd(a + kStride, (unsigned long long)tc);
        }
      }
    }
  }
  __syncthreads();
  // ---- flush CTA slots (one global atomic per non-empty component) ----
  for (int e = tid; e < n * kComp; e += kFastThreads) {
    const int j = e / kComp, i = e - j * kComp;
    const unsigned long long cnt = accs[j * kComp + kStride];
    if (cnt == 0) continue;
    unsigned long long v = accs[j * kComp + i];
    if (i >= C && i < kStride) v += cnt * (unsigned long long)org[i - C];
    if (v) atomicAdd(P.acc + (uint64_t)sm.id[j] * kComp + i, v);
  }
}

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
  size_t b = sizeof(FastSmem);
  b += 2ull * kFastMaxCand * g.channels * sizeof(float);
  b += (size_t)kFastMaxCand * (RXp + R[1] + (g.rank == 3 ? R[2] : 1)) * sizeof(float);
  b += 8 + (size_t)kFastMaxCand * (g.stride + 1) * sizeof(unsigned long long);
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
