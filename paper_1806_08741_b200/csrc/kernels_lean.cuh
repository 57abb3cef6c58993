// K2 lean: the fused assign + delta-accumulate kernel for FULL interior
// regions of 3-D integer volumes (configs 3 and 5). Same exactness contract
// and arithmetic as k_assign_fast (kernels_fast.cuh / DESIGN.md §4.3); the
// work per voxel is restructured so that every per-box cost is shared by
// twice the voxels and the per-voxel history gathers disappear:
//
//  * a warp box is 8x4x8 voxels: each lane owns two 4-voxel runs along x,
//    4 planes apart, so the box geometry, the lower bounds of the
//    candidates, the list compaction and the warp reductions serve 8 voxels
//    per lane instead of 4;
//  * the carried-over distance d_old = D(history[tag][label], x) reads the
//    label's history row from a per-CTA table (every candidate x every tag
//    so far, staged once per region by cp.async) instead of one 16-byte
//    cp.async per voxel; labels outside the region's candidates (rare) read
//    the row from global memory through the same generic pointer;
//  * the spatial part of the candidates' lower bound over a box comes from
//    per-axis tables built once per region;
//  * the search key carries the candidate's record slot in its 6 low bits
//    (key = fp32 bits & ~63 | slot): the winner's record needs no group
//    bookkeeping. The truncation (< 64 ulp, relative < 2^-17) widens the
//    decision margin by tau = 2^-17 (kLeanTau);
//  * regions are full (no clipping): no validity masks, vector loads and
//    stores throughout.
// Regions that are clipped by the volume or the slab run k_assign_fast.
#pragma once

namespace sslic_b200 {

constexpr float kLeanTau = 7.62939453125e-06f;  // 2^-17: key truncation (64 ulp)
constexpr uint32_t kLeanKeyMask = ~63u;
constexpr uint32_t kLeanSentKey = 0x1E800000u;  // bits of 2^-66 (covered keys are below)
constexpr int kLeanQCap = 32;                   // per-warp fp64 re-decision queue

__device__ __forceinline__ float lval(uint32_t key) { return __uint_as_float(key & kLeanKeyMask); }
__device__ __forceinline__ uint32_t lkey(float d, uint32_t slot) {
  return (__float_as_uint(d) & kLeanKeyMask) | slot;
}

// Slot of cluster `id` among the region's candidates (-1 if absent): one
// 8-byte probe {id, slot} per step of linear probing (load factor <= 1/2).
__device__ __forceinline__ int lean_slot(const uint2* ht, uint32_t id) {
  int h = slot_hash(id);
  uint2 e = ht[h];
  while (e.x != id && e.x != 0xffffffffu) {
    h = (h + 1) & (kSlotHash - 1);
    e = ht[h];
  }
  return e.x == id ? (int)e.y : -1;
}

// fp32 d_old (scaled) of a voxel whose label is not a region candidate: the
// same arithmetic as the per-CTA rows, on the row read from global memory.
template <int C>
__device__ __noinline__ float lean_dold_global(const FastParams& P, uint32_t tag, uint32_t L,
                                               float x, float y, float z, const float* pix) {
  constexpr int kStride = C + 3, kS2 = (kStride + 1) & ~1;
  const float2* hg = P.hist32 + ((size_t)tag * (uint32_t)P.g.k + L) * kS2;
  const float xs[3] = {x, y, z};
  float sp = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float2 cc = __ldg(hg + C + a);
    const float t = ((cc.x - xs[a]) + cc.y) * P.inv_grid[a];
    sp = fmaf(t, t, sp);
  }
  float d = sp * (float)P.g.m_sq;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const float2 cc = __ldg(hg + c);
    const float e = (cc.x - pix[c]) + cc.y;
    d = fmaf(e, e, d);
  }
  return d * P.key_scale2;
}

// select x[i] (i in 0..7) without local memory
__device__ __forceinline__ uint32_t lsel8(const uint32_t (&x)[8], int i) {
  const uint32_t a = sel4(x[0], x[1], x[2], x[3], i), b = sel4(x[4], x[5], x[6], x[7], i);
  return (i & 4) ? b : a;
}

// Box and region constants of the lean kernel.
template <int RX, int RY, int RZ>
struct LeanShape {
  static constexpr int BX = 8, BY = 4, BZ = 8;
  static constexpr int NBX = RX / BX, NBY = RY / BY, NBZ = RZ / BZ;
  static constexpr int NBOX = NBX * NBY * NBZ;
  static constexpr int RXp = RX;
  static constexpr int HO = (RX + RY + RZ + 1) & ~1;
  static_assert(RX % BX == 0 && RY % BY == 0 && RZ % BZ == 0, "lean regions tile into boxes");
  static_assert(RX <= 64 && RY <= 64 && RZ <= 64, "6-bit region-local coordinates");
};

template <int C>
__host__ __device__ constexpr int lean_pix_words(int esize) {
  return (4 * C * esize + 3) / 4;  // 32-bit words of one 4-voxel run
}

inline size_t lean_smem_bytes(const Geom& g, const int* R, int cap, int ntags) {
  const int HO = (R[0] + R[1] + R[2] + 1) & ~1;
  const int RS = (HO + 2 * g.channels + 2 + 3) & ~3;
  const int warps = kFastThreads / 32;
  const int s2 = hist32_stride(g.stride);
  const int esize = dtype_size(g.dtype);
  size_t b = sizeof(FastSmem);
  b += (size_t)(cap + 1) * RS * sizeof(float);                       // records
  b += (size_t)cap * (g.stride + 1 + g.channels) * sizeof(int);      // CTA delta slots
  b += (size_t)(R[0] / 8 + R[1] / 4 + R[2] / 4) * cap * sizeof(float);  // spatial LB tables
  b += (size_t)kSlotHash * sizeof(uint2);                              // id -> slot
  b += (size_t)cap * (ntags > 0 ? ntags : 1) * s2 * sizeof(float2);  // history rows
  b += (size_t)warps * 2 * 32 * 16;                                   // next-box label words
  b += (size_t)warps * 2 * 32 * 4 * ((4 * g.channels * esize + 3) / 4);  // next-box pixels
  b += (size_t)warps * (kLeanQCap + 2) * sizeof(uint2);               // fp64 queue
  return (b + 15) & ~(size_t)15;
}

// FIRST: every label word of the slab is undefined (iteration 0 after a
// reset): no word loads, no history rows, no carried-over distances; the
// candidates of a half box are pruned by box_upper_bound instead.
template <int C, typename T, int RXc, int RYc, int RZc, int CAPc, int MINB, int FIRST = 0>
__global__ void __launch_bounds__(kFastThreads, MINB) k_assign_lean(const __grid_constant__ FastParams P) {
  constexpr int RANK = 3;
  constexpr bool kFirst = FIRST != 0;
  using Sh = LeanShape<RXc, RYc, RZc>;
  constexpr int RX = RXc, RY = RYc, RZ = RZc;
  constexpr int kStride = C + RANK;
  constexpr int kComp = kStride + 1;
  constexpr int kCompA = kComp + C;
  constexpr int kS2 = (kStride + 1) & ~1;
  constexpr int kWarps = kFastThreads / 32;
  constexpr int HO = Sh::HO;
  constexpr int RS = (HO + 2 * C + 2 + 3) & ~3;
  constexpr int kCap = CAPc;
  constexpr int kPW = lean_pix_words<C>((int)sizeof(T));
  static_assert(sizeof(T) <= 2, "lean kernel: integer volumes");
  // 32-bit CTA slots: |slot sum| <= region voxels x max value < 2^31
  static_assert((long long)RXc * RYc * RZc * (sizeof(T) == 1 ? 255 : 65535) < (1LL << 31),
                "lean kernel: CTA slot range");
  const Geom& g = P.g;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(smem_raw);
  float* rec = reinterpret_cast<float*>(smem_raw + sizeof(FastSmem));  // [cand+1][RS]
  int* accs = reinterpret_cast<int*>(rec + (size_t)(kCap + 1) * RS);
  float* lbs = reinterpret_cast<float*>(accs + kCap * kCompA);  // [NBX+NBY+2NBZ][kCap]
  uint2* htab2 = reinterpret_cast<uint2*>(lbs + (Sh::NBX + Sh::NBY + 2 * Sh::NBZ) * kCap);
  float2* hs = reinterpret_cast<float2*>(htab2 + kSlotHash);
  const int ntags = (int)P.tag_now;  // tables 0..tag_now-1 hold every carried-over label
  uint4* pf_words = reinterpret_cast<uint4*>(hs + (size_t)kCap * (ntags > 0 ? ntags : 1) * kS2);
  uint32_t* pf_pix = reinterpret_cast<uint32_t*>(pf_words + kWarps * 2 * 32);
  uint2* queues = reinterpret_cast<uint2*>(pf_pix + kWarps * 2 * 32 * kPW);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- region (full: no clipping on any axis) ----
  unsigned rb = blockIdx.x;
  const int rxi = (int)(rb % (unsigned)P.nreg[0]);
  rb /= (unsigned)P.nreg[0];
  const int ryi = (int)(rb % (unsigned)P.nreg[1]);
  const int rzi = (int)(rb / (unsigned)P.nreg[1]);
  const int64_t org[3] = {(int64_t)rxi * RX, (int64_t)ryi * RY, P.reg_z0 + (int64_t)rzi * RZ};
  if (!region_full(P, org, RX, RY, RZ)) return;  // clipped region: k_assign_fast handles it
  const int64_t reg_off = org[0] + org[1] * g.strides[1] + org[2] * g.strides[2];
  uint32_t* const lab_r = P.labels + (reg_off - g.slab_begin * g.plane);
  const T* const img_r = static_cast<const T*>(P.img) + (reg_off - g.data_begin * g.plane) * C;
  const int s1 = (int)g.strides[1], s2 = (int)g.strides[2];
  // lane -> (x run, y, z) of the box; run r sits 4 planes below run 0
  const int xq = lane & 1, yq = (lane >> 1) & 3, zq = lane >> 3;
  const int lane_rel = 4 * xq + yq * s1 + zq * s2;
  const int run_step = 4 * s2;
  const float M = P.margin;
  const float A = P.abs_margin;
  const float ks = P.key_scale;
  const uint32_t lmask = P.codec.label_mask;
  const int lbits = P.codec.label_bits;
  const uint32_t tag_now_bits = P.tag_now << lbits;
  auto box_rel = [&](int b) {
    const int bx = b % Sh::NBX, t = b / Sh::NBX, by = t % Sh::NBY, bz = t / Sh::NBY;
    return bx * Sh::BX + by * Sh::BY * s1 + bz * Sh::BZ * s2 + lane_rel;
  };
  // next-box prefetch, one buffer per run: [warp][run][lane]. Run r of box
  // b + kWarps is issued as soon as run r of box b has been read, so each
  // load has a whole box of work to land behind (one cp.async group per run).
  uint4* const my_pfw = pf_words + (size_t)warp * 2 * 32 + lane;
  uint32_t* const my_pfp = pf_pix + ((size_t)warp * 2 * 32 + lane) * kPW;
  auto prefetch = [&](int bn, int r) {
    if (bn >= Sh::NBOX) return;
    const int q = box_rel(bn) + r * run_step;
    if constexpr (!kFirst) cp_async16(my_pfw + r * 32, lab_r + q);
    const unsigned char* src = reinterpret_cast<const unsigned char*>(img_r + (size_t)q * C);
    uint32_t* dst = my_pfp + (size_t)r * 32 * kPW;
    if constexpr (kPW == 4) cp_async16(dst, src);
    else if constexpr (kPW == 2) cp_async8(dst, src);
    else
#pragma unroll
      for (int i = 0; i < kPW; ++i) cp_async4(dst + i, src + 4 * i);
  };
  prefetch(warp, 0);
  cp_async_commit();
  prefetch(warp, 1);
  cp_async_commit();

  // ---- candidates (k_region_cand) ----
  const int* rc = P.region_cand + (int64_t)blockIdx.x * kRegionCandStride;
  const int total = __ldg(rc);
  const int n = total < P.max_cand ? total : P.max_cand;
  for (int j = tid; j < n; j += kFastThreads) sm.id[j] = __ldg(rc + 1 + j);
  if (tid == 0) {
    sm.n_cand = n;
    sm.stats[0] = sm.stats[1] = sm.stats[2] = 0u;
  }
  if (total > P.max_cand) {  // uniform
    cp_async_wait_all();
    if (tid == 0) atomicAdd(P.counters + 6, 1ull);
    const int64_t hi[3] = {org[0] + RX - 1, org[1] + RY - 1, org[2] + RZ - 1};
    crowded_region<RANK, C>(P, org, hi, org[2], hi[2]);
    return;
  }
  float2* const cxy = reinterpret_cast<float2*>(hs);  // scratch until the history rows land
  static_assert(kS2 >= 3, "cxy scratch fits one history row per candidate");
  for (int j = tid; j <= n; j += kFastThreads) {
    float* r = rec + (size_t)j * RS;
    if (j < n) {
      const int kid = sm.id[j];
      r[HO + 2 * C] = __int_as_float(kid);
      r[HO + 2 * C + 1] = __int_as_float(__ldg(P.chg + kid));
      const float2* c32 = P.cur32 + (int64_t)kid * kS2;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 hl = __ldg(c32 + c);
        r[HO + 2 * c] = hl.x * ks;
        r[HO + 2 * c + 1] = hl.y * ks;
      }
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sm.anc[j][a] = (short)(P.anchors[kid * kMaxRank + a] - org[a]);
        const float2 cp = __ldg(c32 + C + a);
        sm.cpl[j][a] = (cp.x - (float)org[a]) + cp.y;
        cxy[j * 3 + a] = cp;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 2 * C + 2; ++c) r[HO + c] = 0.f;
    }
  }
  for (int i = tid; i < kCap * kCompA / 4; i += kFastThreads)
    reinterpret_cast<int4*>(accs)[i] = make_int4(0, 0, 0, 0);
  for (int i = tid; i < kSlotHash; i += kFastThreads) {
    sm.htab[i] = 0xffff;
    htab2[i] = make_uint2(0xffffffffu, 0u);
  }
  __syncthreads();
  for (int j = tid; j < n; j += kFastThreads) {
    int h = slot_hash((uint32_t)sm.id[j]);
    while (atomicCAS(&sm.htab[h], (unsigned short)0xffff, (unsigned short)j) != 0xffff)
      h = (h + 1) & (kSlotHash - 1);
    h = slot_hash((uint32_t)sm.id[j]);
    while (atomicCAS(&htab2[h].x, 0xffffffffu, (unsigned)sm.id[j]) != 0xffffffffu)
      h = (h + 1) & (kSlotHash - 1);
    htab2[h].y = (unsigned)j;
  }
  {
    // spatial tables (as k_assign_fast): record j, entries sx[RX] | sy[RY] | sz[RZ]
    const float msq = (float)g.m_sq * P.key_scale2;
    const int ox32 = (int)org[0], oy32 = (int)org[1], oz32 = (int)org[2];
    const int sgx = g.grid[0], sgy = g.grid[1], sgz = g.grid[2];
    const float ivx = P.inv_grid[0], ivy = P.inv_grid[1], ivz = P.inv_grid[2];
    for (int j = warp; j <= n; j += kWarps) {
      float* rj = rec + (size_t)j * RS;
      const bool real = j < n;
      const int jj = real ? j : 0;
      const int anx = sm.anc[jj][0], any_ = sm.anc[jj][1], anz = sm.anc[jj][2];
      const float2 ccx = cxy[jj * 3], ccy = cxy[jj * 3 + 1], ccz = cxy[jj * 3 + 2];
      for (int r = lane; r < RX; r += 32) {
        const int dx = r - anx;
        const float t = ((ccx.x - (float)(ox32 + r)) + ccx.y) * ivx;
        rj[r] = real & (dx >= -sgx) & (dx <= sgx) ? msq * (t * t) : kSentinel;
      }
      for (int r0 = lane; r0 < RY + RZ; r0 += 32) {
        const bool isz = r0 >= RY;
        const int r = isz ? r0 - RY : r0;
        const int dx = r - (isz ? anz : any_);
        const int sg = isz ? sgz : sgy;
        const float2 cc = isz ? ccz : ccy;
        const float t = ((cc.x - (float)((isz ? oz32 : oy32) + r)) + cc.y) * (isz ? ivz : ivy);
        rj[RX + r0] = real & (dx >= -sg) & (dx <= sg) ? msq * (t * t) : kSentinel;
      }
    }
    // per axis and box index: window overlap (bmask) and the spatial lower
    // bound of each candidate over the box's extent on that axis
    for (int t = warp; t < Sh::NBX + Sh::NBY + 2 * Sh::NBZ; t += kWarps) {
      const int a = t < Sh::NBX ? 0 : (t < Sh::NBX + Sh::NBY ? 1 : 2);
      const int i = a == 0 ? t : (a == 1 ? t - Sh::NBX : t - Sh::NBX - Sh::NBY);
      const int ext = a == 0 ? 8 : 4;  // x: 8; y: 4; z: half boxes of 4 planes
      const int lo = i * ext, hi = lo + ext - 1;
      const float iv = a == 0 ? ivx : (a == 1 ? ivy : ivz);
      const int s = a == 0 ? sgx : (a == 1 ? sgy : sgz);
      unsigned m2[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        bool c = false;
        float lb = 0.f;
        if (j < n) {
          const int an = sm.anc[j][a];
          c = an + s >= lo && an - s <= hi;
          const float cpl = sm.cpl[j][a];
          const float d = fmaxf(fmaxf((float)lo - cpl, cpl - (float)hi) - 1e-3f, 0.f) * iv;
          lb = msq * (d * d);
        }
        if (j < kCap) lbs[t * kCap + j] = lb;
        m2[h] = __ballot_sync(0xffffffffu, c);
      }
      if (lane == 0) sm.bmask[a][i] = (unsigned long long)m2[1] << 32 | m2[0];
    }
  }
  __syncthreads();  // cxy scratch is read above; the history rows overwrite it
  // history rows of every candidate for every tag so far: hs[j * ntags + t]
  if constexpr (!kFirst) {
    constexpr int kChunks = kS2 / 2;  // 16-byte pieces per row
    for (int i = tid; i < n * kChunks; i += kFastThreads) {
      const int j = i / kChunks, piece = i - j * kChunks;
      const float2* src = P.hist32 + (size_t)(uint32_t)sm.id[j] * kS2 + 2 * piece;
      float2* dst = hs + (size_t)j * ntags * kS2 + 2 * piece;
      for (int t = 0; t < ntags; ++t)
        cp_async16(dst + (size_t)t * kS2, src + (size_t)t * (uint32_t)g.k * kS2);
    }
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();

  // ---- per-warp sweep over the region's boxes ----
  uint2* const queue = queues + (size_t)warp * (kLeanQCap + 2);
  int qn = 0;
  // (diagnostics are counted in shared memory, only when asked for)
  const bool stats = P.eval_count != nullptr;
  const int64_t org0 = org[0], org1 = org[1], org2 = org[2];
  auto redecide = [&](uint2 e) {
    const unsigned ch = redecide_queued<RANK, C, T>(P, sm, accs, org, lab_r, img_r, nullptr, s1,
                                                    s2, false, e);
    if (stats) {
      atomicAdd(&sm.stats[0], 1u);
      if (ch) atomicAdd(&sm.stats[1], ch);
    }
  };
  auto drain = [&]() {
    __syncwarp();
    for (int i = lane; i < qn; i += 32) redecide(queue[i]);
    __syncwarp();
    qn = 0;
  };
  const float M1 = 1.0f + M + kLeanTau;  // amb / below threshold (key truncation included)
  const float M1o = 1.0f + M;            // above threshold (d_old is not truncated)
  const float fx0 = (float)org0, fy0 = (float)org1, fz0 = (float)org2;
#pragma unroll 1
  for (int b = warp; b < Sh::NBOX; b += kWarps) {
    const int bx = b % Sh::NBX, bt = b / Sh::NBX, by = bt % Sh::NBY, bz = bt / Sh::NBY;
    const int rel0 = bx * Sh::BX + by * Sh::BY * s1 + bz * Sh::BZ * s2 + lane_rel;
    const int lx0 = bx * Sh::BX + 4 * xq, ly = by * Sh::BY + yq;
    const float fxv = fx0 + (float)lx0, fyv = fy0 + (float)ly;
    // The two 8x4x4 half boxes (planes bz*8 + 4r + zq) run one after the
    // other through the same code (a rolled loop keeps the kernel small);
    // each is swept over its own pruned candidate list.
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
      const int lz = bz * Sh::BZ + 4 * r + zq;
      const int rel = rel0 + r * run_step;
      const int hz = 2 * bz + r;  // half-box index along z
      uint32_t word[4];
      float p[4][C];
      cp_async_wait_group1();  // this run's group (the other run's may stay in flight)
      __syncwarp();
      {
        if constexpr (kFirst) {
#pragma unroll
          for (int v = 0; v < 4; ++v) word[v] = kUndefined;
        } else {
          const uint4 q = my_pfw[r * 32];
          word[0] = q.x;
          word[1] = q.y;
          word[2] = q.z;
          word[3] = q.w;
        }
        uint32_t w[kPW];
#pragma unroll
        for (int i = 0; i < kPW; ++i) w[i] = my_pfp[(size_t)r * 32 * kPW + i];
        T vals[4 * C];
        memcpy(vals, w, sizeof(vals));
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int c = 0; c < C; ++c) p[v][c] = (float)vals[v * C + c];
      }
      __syncwarp();
      prefetch(b + kWarps, r);  // run r of the warp's next box into the freed buffer
      cp_async_commit();
      // carried-over distances (fp32, scaled) from the per-CTA history rows
      uint32_t oldl[4];
      int oslot[4];
      float dold[4];
      float dmax = 0.f;
      bool any_undef = false;
      unsigned fb = 0;  // labels outside the region's candidates (rows from global memory)
      const float fzv = fz0 + (float)lz;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        if constexpr (kFirst) {
          oldl[v] = lmask;
          oslot[v] = -1;
          dold[v] = kInf;
          any_undef = true;
          continue;
        }
        const uint32_t w = word[v];
        const bool def = w != kUndefined;
        oldl[v] = w & lmask;  // undefined -> lmask (never a label)
        const uint32_t tg = def ? (w >> lbits) : 0u;
        // (the lookup runs once per run of equal labels: most 4-voxel runs
        // of a coherent label map hold one label)
        int sl;
        if (v > 0 && oldl[v] == oldl[v - 1]) sl = oslot[v - 1];
        else sl = def ? lean_slot(htab2, oldl[v]) : -1;
        oslot[v] = sl;
        fb |= (unsigned)(def & (sl < 0)) << v;
        const float2* hr = hs + ((sl >= 0 ? sl : 0) * ntags + (sl >= 0 ? (int)tg : 0)) * kS2;
        float2 cc[kStride];
#pragma unroll
        for (int q = 0; q < kStride; ++q) cc[q] = hr[q];
        const float xs[3] = {fxv + (float)v, fyv, fzv};
        float sp = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float t = ((cc[C + a].x - xs[a]) + cc[C + a].y) * P.inv_grid[a];
          sp = fmaf(t, t, sp);
        }
        float d = sp * (float)g.m_sq;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float e = (cc[c].x - p[v][c]) + cc[c].y;
          d = fmaf(e, e, d);
        }
        dold[v] = def ? d * P.key_scale2 : kInf;
        any_undef |= !def;
      }
      if (fb) {  // rare: same arithmetic on the row read from global memory
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (fb >> v & 1u)
            dold[v] = lean_dold_global<C>(P, word[v] >> lbits, oldl[v], fxv + (float)v, fyv, fzv,
                                          p[v]);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) dmax = fmaxf(dmax, dold[v]);
      if constexpr (!kFirst) {
        dmax = any_undef ? kInf : dmax * (1.0f + M) + A;
        dmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(dmax)));
      }

      // value range of the half box per channel (scaled) for the colour bounds
      float pmin[C], pmax[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        uint32_t lo = 0xffffffffu, hv = 0u;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t o = __float_as_uint(p[v][c]);  // non-negative: order-preserving
          lo = min(lo, o);
          hv = max(hv, o);
        }
        pmin[c] = __uint_as_float(__reduce_min_sync(0xffffffffu, lo)) * ks;
        pmax[c] = __uint_as_float(__reduce_max_sync(0xffffffffu, hv)) * ks;
      }
      // kept candidates: window overlaps the half box and LB <= max d_old
      const unsigned long long bmask = sm.bmask[0][bx] & sm.bmask[1][by] & sm.bmask[2][hz];
      if constexpr (kFirst) {
        // undefined voxels have no finite d_old: the smallest upper bound of a
        // candidate covering the whole half box prunes instead (box_upper_bound)
        const int b0[3] = {bx * Sh::BX, by * Sh::BY, hz * 4};
        const int b1[3] = {b0[0] + Sh::BX - 1, b0[1] + Sh::BY - 1, b0[2] + 3};
        const int sg[3] = {(int)g.grid[0], (int)g.grid[1], (int)g.grid[2]};
        float ub = kInf;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = lane + 32 * h;
          const bool c = (uint32_t)(bmask >> (32 * h)) >> lane & 1u;
          if (j < kCap)
            ub = fminf(ub, box_upper_bound<RANK, C>(sm, rec + j * RS + HO, j, c, pmin, pmax, b0, b1,
                                                    sg, P.inv_grid, (float)g.m_sq * P.key_scale2));
        }
        ub = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(ub)));
        dmax = (ub * (1.0f + 4.0f * M + kLeanTau) + A) * (1.0f + M) + A;
      }
      const float* lbx = lbs + bx * kCap;
      const float* lby = lbs + (Sh::NBX + by) * kCap;
      const float* lbz = lbs + (Sh::NBX + Sh::NBY + hz) * kCap;
      bool keep[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const bool c = (uint32_t)(bmask >> (32 * h)) >> lane & 1u;
        float lb = 0.f;
        if (j < kCap) {
          const float* rr = rec + j * RS;
#pragma unroll
          for (int cc = 0; cc < C; ++cc) {
            const float ch = rr[HO + 2 * cc], cl = fabsf(rr[HO + 2 * cc + 1]);
            const float t = fmaxf(fmaxf(pmin[cc] - ch, ch - pmax[cc]) - cl, 0.f);
            lb = fmaf(t, t, lb);
          }
          lb += lbx[j] + lby[j] + lbz[j];
        }
        keep[h] = c && lb * (1.0f - 4.0f * M) <= dmax;
      }
      int nl;
      __syncwarp();  // the previous half box's sweep has read the list
      {
        const unsigned m0 = __ballot_sync(0xffffffffu, keep[0]);
        const unsigned m1 = __ballot_sync(0xffffffffu, keep[1]);
        const unsigned lt = (1u << lane) - 1u;
        if (keep[0]) sm.wl[warp][__popc(m0 & lt)] = (uint32_t)lane;
        if (keep[1]) sm.wl[warp][__popc(m0) + __popc(m1 & lt)] = (uint32_t)(lane + 32);
        nl = __popc(m0) + __popc(m1);
        if (lane == 0 && (nl & 1)) sm.wl[warp][nl] = (uint32_t)n;  // pad: all-sentinel record
        __syncwarp();
      }
      const int nlp = (nl + 1) & ~1;
      if (stats && lane == 0) atomicAdd(&sm.stats[2], 128u * (unsigned)nl);

      // fp32 argmin with runner-up; keys carry the record slot
      f2 p01[C], p23[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        p01[c] = pk2(p[0][c] * ks, p[1][c] * ks);
        p23[c] = pk2(p[2][c] * ks, p[3][c] * ks);
      }
      const int ox = lx0, oy = RX + ly, oz = RX + RY + lz;
      uint32_t best[4], second[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) best[v] = second[v] = 0xffffffffu;
      const uint2* wl2 = reinterpret_cast<const uint2*>(sm.wl[warp]);
      uint2 pr = wl2[0];
#pragma unroll 1
      for (int jj = 0; jj < nlp; jj += 2) {
        const uint2 cur = pr;
        pr = wl2[(jj >> 1) + 1];
        uint32_t key[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t slot = h ? cur.y : cur.x;
          const float* rr = rec + slot * RS;
          const ulonglong2 sxv = *reinterpret_cast<const ulonglong2*>(rr + ox);
          const float syz = rr[oy] + rr[oz];
          f2 a01 = add2(sxv.x, pk2(syz, syz)), a23 = add2(sxv.y, pk2(syz, syz));
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const float2 hl = *reinterpret_cast<const float2*>(rr + HO + 2 * c);
            const f2 ch = pk2(hl.x, hl.x), cl = pk2(hl.y, hl.y);
            const f2 d01 = add2(sub2(ch, p01[c]), cl);
            const f2 d23 = add2(sub2(ch, p23[c]), cl);
            a01 = fma2(d01, d01, a01);
            a23 = fma2(d23, d23, a23);
          }
          float f0, f1, f2v, f3;
          up2(a01, f0, f1);
          up2(a23, f2v, f3);
          key[h][0] = lkey(f0, slot);
          key[h][1] = lkey(f1, slot);
          key[h][2] = lkey(f2v, slot);
          key[h][3] = lkey(f3, slot);
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

      // ---- decisions (predicated; fp64 re-decision only for undecided voxels) ----
      uint32_t nword[4], newl[4];
      int wslot[4];
      unsigned exact_mask = 0, amb_mask = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const bool live = best[v] < kLeanSentKey;
        const int slot = (int)(best[v] & 63u);
        const int2 ic = *reinterpret_cast<const int2*>(rec + slot * RS + HO + 2 * C);
        const uint32_t kid = (uint32_t)ic.x;
        const float bv = lval(best[v]);
        const float thr = fmaf(bv, M1, A);
        const bool amb = lval(second[v]) <= thr;
        const bool same = (kid == oldl[v]) & (ic.y <= (int)(word[v] >> lbits));
        const bool below = thr < dold[v];
        const bool above = bv > fmaf(dold[v], M1o, A);
        const bool upd = !amb & !same & below;
        const bool kp = !amb & (same | above);
        nword[v] = live & upd ? (tag_now_bits | kid) : word[v];
        exact_mask |= (unsigned)(live & !upd & !kp) << v;
        amb_mask |= (unsigned)amb << v;
        wslot[v] = slot;
        newl[v] = nword[v] & lmask;
      }
      if ((nword[0] != word[0]) | (nword[1] != word[1]) | (nword[2] != word[2]) |
          (nword[3] != word[3]))
        *reinterpret_cast<uint4*>(lab_r + rel) = make_uint4(nword[0], nword[1], nword[2], nword[3]);

      // ---- deltas: +new / -old for voxels whose label value changed ----
      unsigned chm = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) chm |= (unsigned)(newl[v] != oldl[v]) << v;
      if (stats) {  // uniform
        const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)__popc(chm));
        if (lane == 0 && c) atomicAdd(&sm.stats[1], c);
      }
      unsigned pending = chm | chm << 4;
      if (__any_sync(0xffffffffu, any_undef)) {
        unsigned undef = 0, olddef = 0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          undef += (unsigned)((newl[v] == lmask) & !(exact_mask >> v & 1u));
          olddef |= (unsigned)(oldl[v] != lmask) << v;
        }
        pending = chm | (chm & olddef) << 4;
        const unsigned tu = __reduce_add_sync(0xffffffffu, undef);
        if (lane == 0 && tu) atomicAdd(P.counters, (unsigned long long)tu);  // slic.hpp:330-331
      }
      const unsigned npend = __reduce_add_sync(0xffffffffu, (unsigned)__popc(pending));
      if (npend != 0) {
        bool per_lane = npend <= sparse_deltas(C);
        if (!per_lane) {
          const int fbit = pending ? __ffs(pending) - 1 : 0;
          const uint32_t first = sel8(newl, oldl, fbit);
          const unsigned anyp = __ballot_sync(0xffffffffu, pending != 0);
          const uint32_t l0 = __shfl_sync(0xffffffffu, first, __ffs(anyp) - 1);
          const unsigned same = __ballot_sync(0xffffffffu, pending != 0 && first == l0);
          per_lane = 4 * __popc(same) < 3 * __popc(anyp);
        }
        if (per_lane) {
          // per sign: consecutive voxels of one label merge into the run's
          // first voxel, then each head adds into its CTA slot
#pragma unroll
          for (int sg = 0; sg < 2; ++sg) {
            int iv[4][C], xs[4], cn[4];
            bool pf[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              pf[v] = pending >> (v + 4 * sg) & 1u;
              xs[v] = lx0 + v;
              cn[v] = 1;
#pragma unroll
              for (int c = 0; c < C; ++c) iv[v][c] = (int)p[v][c];
            }
#pragma unroll
            for (int v = 3; v >= 1; --v) {
              const uint32_t lv = sg ? oldl[v] : newl[v], lp = sg ? oldl[v - 1] : newl[v - 1];
              if (pf[v] && pf[v - 1] && lv == lp) {
#pragma unroll
                for (int c = 0; c < C; ++c) iv[v - 1][c] += iv[v][c];
                xs[v - 1] += xs[v];
                cn[v - 1] += cn[v];
                pf[v] = false;
              }
            }
            const int sgn = sg ? -1 : 1;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              if (!pf[v]) continue;
              const uint32_t L = sg ? oldl[v] : newl[v];
              const int S = sg ? oslot[v] : wslot[v];
              if (S >= 0) {
                int* a = accs + S * kCompA;
#pragma unroll
                for (int c = 0; c < C; ++c) atomicAdd(a + c, sgn * iv[v][c]);
                atomicAdd(a + C, sgn * xs[v]);
                atomicAdd(a + C + 1, sgn * cn[v] * ly);
                atomicAdd(a + C + 2, sgn * cn[v] * lz);
                atomicAdd(a + kStride, sgn * cn[v]);
              } else {  // label outside the region's candidates: global, absolute
                unsigned long long* a = P.acc + (uint64_t)L * kComp;
                const long long cl = sgn * cn[v];
#pragma unroll
                for (int c = 0; c < C; ++c)
                  atomicAdd(a + c, (unsigned long long)(long long)(sgn * iv[v][c]));
                atomicAdd(a + C, (unsigned long long)(sgn * xs[v] + cl * org0));
                atomicAdd(a + C + 1, (unsigned long long)(cl * (ly + org1)));
                atomicAdd(a + C + 2, (unsigned long long)(cl * (lz + org2)));
                atomicAdd(a + kStride, (unsigned long long)cl);
              }
            }
          }
          pending = 0;
        }
#pragma unroll 1
        for (;;) {  // warp-aggregated per label (half boxes dominated by one label)
          const unsigned any = __ballot_sync(0xffffffffu, pending != 0);
          if (!any) break;
          const int leader = __ffs(any) - 1;
          uint32_t mylab = 0;
          if (pending) mylab = sel8(newl, oldl, __ffs(pending) - 1);
          const uint32_t L = __shfl_sync(0xffffffffu, mylab, leader);
          int cnt = 0, sxr = 0, syr = 0, szr = 0;
          int sv[C];
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
              for (int c = 0; c < C; ++c) sv[c] += sgn * (int)p[v][c];
            }
          }
          int tx, ty, tz, tc;
          redux_pair(sxr, syr, tx, ty);
          redux_pair(szr, cnt, tz, tc);
          int tvs[C];
#pragma unroll
          for (int c = 0; c < C; ++c) tvs[c] = (int)__reduce_add_sync(0xffffffffu, (uint32_t)sv[c]);
          if (lane == leader) {
            const int S = lean_slot(htab2, L);
            if (S >= 0) {
              int* a = accs + S * kCompA;
#pragma unroll
              for (int c = 0; c < C; ++c)
                if (tvs[c]) atomicAdd(a + c, tvs[c]);
              if (tx) atomicAdd(a + C, tx);
              if (ty) atomicAdd(a + C + 1, ty);
              if (tz) atomicAdd(a + C + 2, tz);
              if (tc) atomicAdd(a + kStride, tc);
            } else {
              unsigned long long* a = P.acc + (uint64_t)L * kComp;
#pragma unroll
              for (int c = 0; c < C; ++c)
                if (tvs[c]) atomicAdd(a + c, (unsigned long long)(long long)tvs[c]);
              atomicAdd(a + C, (unsigned long long)(tx + (long long)tc * org0));
              atomicAdd(a + C + 1, (unsigned long long)(ty + (long long)tc * org1));
              atomicAdd(a + C + 2, (unsigned long long)(tz + (long long)tc * org2));
              if (tc) atomicAdd(a + kStride, (unsigned long long)(long long)tc);
            }
          }
        }
      }

      // ---- undecided voxels: per-warp queue, re-decided in fp64 32 at a time ----
      const unsigned my_q = (unsigned)__popc(exact_mask);
      const unsigned nq = __reduce_add_sync(0xffffffffu, my_q);
      if (nq != 0) {  // uniform (at most 128 per half box <= 2 x kLeanQCap)
        if (qn + (int)nq > kLeanQCap) drain();
        unsigned incl = my_q;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        if ((int)nq <= kLeanQCap) {
          int pos = qn + (int)(incl - my_q);
#pragma unroll
          for (int v = 0; v < 4; ++v)
            if (exact_mask >> v & 1u) {
              const uint32_t info = (uint32_t)(lx0 + v) | (uint32_t)ly << 6 | (uint32_t)lz << 12 |
                                    (amb_mask >> v & 1u) << 18 | (uint32_t)wslot[v] << 19;
              queue[pos++] = make_uint2(word[v], info);
            }
          qn += (int)nq;
          if (qn >= 32) drain();
        } else {  // a burst larger than the queue: each lane re-decides its own
#pragma unroll 1
          for (int v = 0; v < 4; ++v) {
            __syncwarp();
            if (exact_mask >> v & 1u) {
              const uint32_t info = (uint32_t)(lx0 + v) | (uint32_t)ly << 6 | (uint32_t)lz << 12 |
                                    (amb_mask >> v & 1u) << 18 | (uint32_t)wslot[v] << 19;
              redecide(make_uint2(word[v], info));
            }
          }
          __syncwarp();
        }
      }
    }
  }
  if (qn > 0) drain();
  cp_async_wait_all();
  __syncthreads();
  if (stats && tid == 0) {
    atomicAdd(P.counters + 5, (unsigned long long)sm.stats[0]);
    atomicAdd(P.counters + 7, (unsigned long long)sm.stats[1]);
    atomicAdd(P.eval_count, (unsigned long long)sm.stats[2]);
  }
  // ---- flush CTA slots (one global atomic per non-zero component) ----
  for (int t = tid; t < n * kComp; t += kFastThreads) {
    const int j = t / kComp, cp = t - j * kComp;
    long long v = (long long)accs[j * kCompA + cp];
    if (cp >= C && cp < kStride) v += (long long)accs[j * kCompA + kStride] * org[cp - C];
    if (v) atomicAdd(P.acc + (uint64_t)sm.id[j] * kComp + cp, (unsigned long long)v);
  }
}

}  // namespace sslic_b200
