// K2 fast path, main kernel and launchers (helpers, exact re-decision and the
// crowded-region fallback are in kernels_fast.cuh; design notes there and in
// DESIGN.md "K2").
#pragma once

#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "kernels_fast.cuh"

namespace sslic_b200 {

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16_if(void* smem_dst, const void* gsrc, bool p) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t"
               "@q cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(d),
               "l"(gsrc), "r"((int)p)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_group1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// ---- TMA (cp.async.bulk.tensor) box loads with an mbarrier per buffer ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// sum over the warp of a pair of signed 16-bit quantities packed in 32 bits
// (|sum| < 2^15 each)
__device__ __forceinline__ void redux_pair(int lo, int hi, int& slo, int& shi) {
  const uint32_t t = __reduce_add_sync(0xffffffffu, (uint32_t)(lo + hi * 65536));
  slo = (int)(int16_t)(t & 0xffffu);
  shi = ((int)t - slo) >> 16;
}

// 4 consecutive voxels x C channels of T, vector loads when aligned
template <int C, typename T>
__device__ __forceinline__ void load_run(const T* src, bool vec, const bool* valid, float (&p)[4][C]) {
  constexpr int NW = C * (int)sizeof(T);  // 32-bit words for 4 voxels
  if (vec) {
    uint32_t w[NW];
    if (NW % 4 == 0) {
#pragma unroll
      for (int i = 0; i < NW / 4; ++i) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(src) + i);
        w[4 * i] = q.x;
        w[4 * i + 1] = q.y;
        w[4 * i + 2] = q.z;
        w[4 * i + 3] = q.w;
      }
    } else if (NW % 2 == 0) {
#pragma unroll
      for (int i = 0; i < NW / 2; ++i) {
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(src) + i);
        w[2 * i] = q.x;
        w[2 * i + 1] = q.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NW; ++i) w[i] = __ldg(reinterpret_cast<const uint32_t*>(src) + i);
    }
    T vals[4 * C];
    memcpy(vals, w, sizeof(vals));
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int c = 0; c < C; ++c) p[v][c] = (float)vals[v * C + c];
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int c = 0; c < C; ++c) p[v][c] = valid[v] ? (float)__ldg(src + v * C + c) : 0.f;
  }
}

// CTAs per SM the register budget targets: 5 (96 registers) where the
// shared-memory footprint allows it (1-2 channels; measured +2% on config 3),
// else 4 (128 registers; 5 costs config 4 7% through spills)
__host__ __device__ constexpr int fast_min_blocks(int C, int VAR = 0) {
  // (the first-iteration kernel, VAR & 4, spills 28 B at 96 registers: 4 CTAs there)
  return C <= 2 && !(VAR & 4) ? 5 : 4;
}

// fp64 re-decision of one queued voxel of the fast kernel (entry: old label
// word, region-local coordinates | amb | winner slot): writes the label word
// and adds the voxel's deltas to the CTA slots (layout: k_assign_fast).
// Returns 1 if the label value changed.
template <int RANK, int C, typename TS>
__device__ __noinline__ unsigned redecide_queued(const FastParams& P, const FastSmem& sm, int* accs,
                                                 const int64_t* org, uint32_t* lab_r,
                                                 const void* img_rv, const double* imgx_r, int s1,
                                                 int s2, bool split16, const uint2 e) {
  constexpr bool kF64 = std::is_same<TS, double>::value;
  using T = typename std::conditional<kF64, float, TS>::type;
  constexpr bool kFloatAcc = sizeof(TS) >= 4;
  constexpr int kStride = C + RANK, kComp = kStride + 1, kCompA = kComp + C;
  const T* img_r = static_cast<const T*>(img_rv);
  const uint32_t lmask = P.codec.label_mask;
  const int qx = (int)(e.y & 63u), qy = (int)(e.y >> 6 & 63u), qz = (int)(e.y >> 12 & 63u);
  const bool qamb = e.y >> 18 & 1u;
  const int qj = (int)(e.y >> 19 & 63u);
  const int qrel = qx + qy * s1 + qz * s2;
  const T* qpx = img_r + (size_t)qrel * C;
  const uint32_t nw = exact_region_voxel(P, sm, org[0] + qx, org[1] + qy, org[2] + qz,
                                         qpx - static_cast<const T*>(P.img), e.x, qamb, qj, org);
  const uint32_t ol = e.x & lmask, nl2 = nw & lmask;
  if (nw != e.x) lab_r[qrel] = nw;
  if (nl2 == lmask) atomicAdd(P.counters, 1ull);  // slic.hpp:330-331
  if (nl2 == ol) return 0u;
  const float fscale = ldexpf(1.0f, P.shift);
  const long long co[3] = {qx, qy, qz};
#pragma unroll 1
  for (int sg = 0; sg < 2; ++sg) {
    const uint32_t L = sg == 0 ? nl2 : ol;
    if (L == lmask) continue;
    const long long sgn = sg == 0 ? 1 : -1;
    const int S = slot_of(sm, L);
    long long val[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      if constexpr (kF64) val[c] = to_fixed(imgx_r[(int64_t)qrel * C + c], P.shift);
      else val[c] = sizeof(T) < 4 ? (long long)qpx[c]
                                  : (long long)__float2ll_rn((float)qpx[c] * fscale);
    }
    if (S >= 0) {
      int* a = accs + S * kCompA;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const long long v = sgn * val[c];
        if constexpr (kFloatAcc) {
          const unsigned long long u = (unsigned long long)v;
          const uint32_t l = (uint32_t)u;
          const uint32_t before = atomicAdd(reinterpret_cast<unsigned*>(a) + c, l);
          const uint32_t carry = before + l < before ? 1u : 0u;
          atomicAdd(reinterpret_cast<unsigned*>(a) + kComp + c, (uint32_t)(u >> 32) + carry);
        } else if (split16) {
          atomicAdd(a + c, (int)(v & 255));
          atomicAdd(a + kComp + c, (int)(v >> 8));
        } else {
          atomicAdd(a + c, (int)v);
        }
      }
#pragma unroll
      for (int ax = 0; ax < RANK; ++ax) atomicAdd(a + C + ax, (int)(sgn * co[ax]));
      atomicAdd(a + kStride, (int)sgn);
    } else {
      unsigned long long* a = P.acc + (uint64_t)L * kComp;
#pragma unroll
      for (int c = 0; c < C; ++c) atomicAdd(a + c, (unsigned long long)(sgn * val[c]));
#pragma unroll
      for (int ax = 0; ax < RANK; ++ax)
        atomicAdd(a + C + ax, (unsigned long long)(sgn * (co[ax] + org[ax])));
      atomicAdd(a + kStride, (unsigned long long)sgn);
    }
  }
  return 1u;
}

// per-warp capacity of the batched fp64 re-decision queue (entries)
// (3 channels only: the call of the non-inlined re-decision costs the 96-register
// 1-2 channel kernels spills, and config 4's shared memory has no room)
__host__ __device__ constexpr int fast_queue_cap(int C) { return C == 3 ? 32 : 0; }

// T is the caller's storage type; T = double sweeps an f32 working copy (TW)
// with the pixel rounding folded into the margins, and takes the exact f64
// values for the re-decisions and the fixed-point deltas.
// VAR bits: 1 no spatial lower bound, 2 full regions only (clipping folded),
// 4 first iteration (every label word of the slab is undefined: no word loads, no
// carried-over distances; candidates pruned by box_upper_bound), 16 TMA box
// tiles, 32 L2 prefetch of the next box's unstaged pixel runs
template <int RANK, int C, typename TS, int RXc, int RYc, int RZc, int CAPc = 0, int VAR = 0>
__global__ void __launch_bounds__(kFastThreads, fast_min_blocks(C, VAR)) k_assign_fast(const __grid_constant__ FastParams P) {
  constexpr bool kF64 = std::is_same<TS, double>::value;
  using T = typename std::conditional<kF64, float, TS>::type;  // working pixel type
  using Box = BoxShape<RANK>;
  constexpr int kStride = C + RANK;
  constexpr int kComp = kStride + 1;
  constexpr int kS2 = (kStride + 1) & ~1;  // hi/lo history entry, padded to 16 B
  constexpr int kWarps = kFastThreads / 32;
  const Geom& g = P.g;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FastSmem& sm = *reinterpret_cast<FastSmem*>(smem_raw);
  const int RX = RXc ? RXc : P.R[0], RY = RYc ? RYc : P.R[1];
  const int RZ = RANK == 3 ? (RZc ? RZc : P.R[2]) : 1;
  const int RXp = (RX + 3) & ~3;
  // (c_hi, c_lo) per channel after the tables, 8-byte aligned
  const int HO = (RXp + RY + (RANK == 3 ? RZ : 0) + 1) & ~1;
  // record: [sx | sy | sz | (c_hi, c_lo) x C | cluster id, chg], 16-byte rows
  const int RS = (HO + 2 * C + 2 + 3) & ~3;
  float* rec = reinterpret_cast<float*>(smem_raw + sizeof(FastSmem));  // [cand+1][RS]
  // CTA delta slots per candidate, 32-bit words (native shared atomics; a
  // 64-bit shared atomic is a CAS loop): [intensity low x C | coords | count |
  // intensity high x C]. Coordinates are region-local (|sum| < 2^25). u8/u16
  // intensities are exact in the low word (|slot sum| <= region voxels x max
  // value < 2^31); u16 regions of more than 32768 voxels split them into a
  // low byte and the rest. Fixed-point float intensities are 64-bit values
  // kept as (low word, high word) with the carry of each add.
  constexpr bool kFloatAcc = sizeof(TS) >= 4;
  // per-lane delta walk: rolled for the (64-bit, carry-pair) float
  // intensities, unrolled over the 4 voxels for integer volumes (measured:
  // config 4 f32 x4 vs config 3 u16)
  constexpr bool kRolledDeltas = kFloatAcc;
  constexpr int kQCap = fast_queue_cap(C);
  using AccT = int;
  constexpr int kCompA = kComp + C;
  // candidate capacity of the record/slot arrays (P.max_cand <= kCap)
  constexpr int kCap = CAPc ? CAPc : kFastMaxCand;
  AccT* accs = reinterpret_cast<AccT*>(rec + (size_t)(kCap + 1) * RS);
  // per-warp staging of the carried-over centres: [warp][v][lane][kS2] float2
  float2* stage = reinterpret_cast<float2*>(accs + kCap * kCompA);
  // next-box prefetch: label words [warp][2][lane] (16 B), pixel runs [warp][2][lane][kPW]
  uint4* pf_words = reinterpret_cast<uint4*>(stage + kWarps * 4 * kS2 * 32);
  uint32_t* pf_pix = reinterpret_cast<uint32_t*>(pf_words + kWarps * 2 * 32);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // hi/lo centre coordinates of the candidates for the spatial tables, in the
  // history staging area (free until the sweep): [cand][3]
  float2* const cxy = stage;
  static_assert(kFastMaxCand * 3 <= 4 * 32 * 2, "cxy fits the staging area of one warp");
  // ---- region ----
  unsigned rb = blockIdx.x;  // 32-bit region index math
  const int rxi = (int)(rb % (unsigned)P.nreg[0]);
  rb /= (unsigned)P.nreg[0];
  const int ryi = (int)(rb % (unsigned)P.nreg[1]);
  const int rzi = (int)(rb / (unsigned)P.nreg[1]);
  const int64_t org[3] = {(int64_t)rxi * RX, (int64_t)ryi * RY,
                          RANK == 3 ? P.reg_z0 + (int64_t)rzi * RZ : 0};
  if (RANK == 3 && P.skip_full && region_full(P, org, RX, RY, RZ)) return;  // k_assign_lean's
  // VAR & 2: this launch takes only FULL regions (compile-time shape): every
  // box is whole, so the clipping below folds to constants
  constexpr bool kFull = (VAR & 2) != 0 && RANK == 3 && RXc > 0;
  if (kFull && !region_full(P, org, RX, RY, RZ)) return;
  constexpr bool kFirst = (VAR & 4) != 0;
  const int64_t hi[3] = {min(org[0] + RX, g.dims[0]) - 1, min(org[1] + RY, g.dims[1]) - 1,
                         RANK == 3 ? min(org[2] + RZ, g.dims[2]) - 1 : 0};
  const int64_t zlo = RANK == 3 ? max(org[2], g.slab_begin) : 0;
  const int64_t zhi = RANK == 3 ? min(hi[2], g.slab_end - 1) : 0;
  // region-local inclusive bounds (32-bit)
  const int ex = kFull ? RX - 1 : (int)(hi[0] - org[0]);
  const int ey = kFull ? RY - 1 : (int)(hi[1] - org[1]);
  const int ez_lo = kFull ? 0 : (int)(zlo - org[2]);
  const int ez_hi = kFull ? RZ - 1 : (int)(zhi - org[2]);

  // ---- box geometry and the next-box prefetch ----
  const int nbx = (RX + Box::X - 1) / Box::X, nby = (RY + Box::Y - 1) / Box::Y;
  const int nbz = RANK == 3 ? (RZ + Box::Z - 1) / Box::Z : 1;
  const int nbox = nbx * nby * nbz;
  // lane -> (x run, y, z) inside the box: Box::X / 4 runs of 4 voxels along x
  constexpr int kXL = Box::X / 4;
  const int xq = lane % kXL;
  const int yq = RANK == 3 ? (lane / kXL) % Box::Y : lane / kXL;
  const int zq = RANK == 3 ? lane / (kXL * Box::Y) : 0;
  const float M = P.margin;
  const float A = P.abs_margin;
  const float fscale = ldexpf(1.0f, P.shift);
  const float ks = P.key_scale;
  // region base pointers; in-region offsets are 32-bit (fast_path_supported
  // guarantees R_z * plane < 2^31)
  const int64_t reg_off = org[0] + org[1] * g.strides[1] + (RANK == 3 ? org[2] * g.strides[2] : 0);
  uint32_t* const lab_r = P.labels + (reg_off - g.slab_begin * g.plane);
  const T* const img_r = static_cast<const T*>(P.img) + (reg_off - g.data_begin * g.plane) * C;
  // f64 inputs: the caller's values, for the exact fixed-point deltas
  const double* const imgx_r =
      kF64 ? static_cast<const double*>(P.img_exact) + (reg_off - g.data_begin * g.plane) * C
           : nullptr;
  const int s1 = (int)g.strides[1], s2 = RANK == 3 ? (int)g.strides[2] : 0;
  const int lane_rel = 4 * xq + yq * s1 + zq * s2;
  // [warp][v][lane][kS2]: each lane's entry is contiguous (16-byte cp.async)
  float2* my_stage = stage + ((size_t)warp * 4 * 32 + lane) * kS2;
  unsigned n_changed = 0, n_redecided = 0, n_evals = 0;
  // tag-mode label words (the fast path never runs in dist mode): labels are
  // < k <= 2^lbits - 2, so the undefined word 0xffffffff maps to label lmask
  const uint32_t lmask = P.codec.label_mask;
  const int lbits = P.codec.label_bits;
  const uint32_t tag_now_bits = P.tag_now << lbits;
  // slot of a record offset: (roff * rs_m) >> 16 == roff / RS exactly (RS < 1024, slot <= 64)
  const uint32_t rs_m = (65536u + (uint32_t)RS - 1u) / (uint32_t)RS;
  const bool split16 = sizeof(TS) == 2 && RX * RY * RZ > 32768;
  auto slot_add = [&](AccT* a, int comp, long long v) { atomicAdd(a + comp, (int)v); };
  auto slot_add_val = [&](AccT* a, int c, long long v) {  // intensity component
    if constexpr (kFloatAcc) {
      const unsigned long long u = (unsigned long long)v;
      const uint32_t l = (uint32_t)u;
      const uint32_t before = atomicAdd(reinterpret_cast<unsigned*>(a) + c, l);
      const uint32_t carry = before + l < before ? 1u : 0u;
      atomicAdd(reinterpret_cast<unsigned*>(a) + kComp + c, (uint32_t)(u >> 32) + carry);
    } else if (split16) {
      atomicAdd(a + c, (int)(v & 255));
      atomicAdd(a + kComp + c, (int)(v >> 8));
    } else {
      atomicAdd(a + c, (int)v);
    }
  };

  // The label words (and, when small, the pixels) of a warp's next box are
  // prefetched with cp.async into a per-lane double buffer while the current
  // box is processed; boxes that are clipped or unaligned load directly.
  constexpr int kPW = pf_pix_words(C, (int)sizeof(T));
  uint4* my_pfw = pf_words + (size_t)warp * 2 * 32 + lane;          // [warp][buf][lane]
  uint32_t* my_pfp = pf_pix + ((size_t)warp * 2 * 32 + lane) * (kPW ? kPW : 1);
  struct BoxG {
    int bx, by, bz, bx0, by0, bz0, bx1, by1, bz0c, bz1, lx0, ly, lz;
    bool nonempty, vec;
    int rel;  // offset of the lane's first voxel from the region origin
  };
  auto box_geom = [&](int b) {
    BoxG q;
    const int bx = b % nbx, t = b / nbx, by = t % nby, bz = t / nby;
    q.bx = bx;
    q.by = by;
    q.bz = bz;
    q.bx0 = bx * Box::X;
    q.by0 = by * Box::Y;
    q.bz0 = bz * Box::Z;
    q.bx1 = min(q.bx0 + Box::X - 1, ex);
    q.by1 = min(q.by0 + Box::Y - 1, ey);
    q.bz0c = RANK == 3 ? max(q.bz0, ez_lo) : 0;
    q.bz1 = RANK == 3 ? min(q.bz0 + Box::Z - 1, ez_hi) : 0;
    q.nonempty = kFull || (q.bx0 <= q.bx1 && q.by0 <= q.by1 && q.bz0c <= q.bz1);
    q.lx0 = q.bx0 + 4 * xq;
    q.ly = q.by0 + yq;
    q.lz = q.bz0 + zq;
    const bool row_ok = kFull || (q.ly <= q.by1 && (RANK == 2 || (q.lz >= q.bz0c && q.lz <= q.bz1)));
    q.vec = kFull ? true : (P.aligned4 && q.nonempty && row_ok && q.lx0 + 3 <= ex && q.lx0 + 3 < RX);
    q.rel = q.bx0 + q.by0 * s1 + q.bz0 * s2 + lane_rel;
    return q;
  };
  // VAR & 16 (full regions, 3-D): the warp's next box arrives by TMA, two
  // 3-D tensor-tile loads (label words 8x4x4 u32, pixels 8C x 4 x 4) issued by
  // one lane into a per-warp double buffer, completion on an mbarrier per
  // buffer; the lanes then read their 4-voxel runs from the tiles.
  constexpr bool kTma = (VAR & 16) != 0 && kFull;
  constexpr int kTileW = Box::X * Box::Y * Box::Z * 4;                    // bytes of words
  constexpr int kTileP = Box::X * Box::Y * Box::Z * C * (int)sizeof(T);  // bytes of pixels
  constexpr int kTileBuf = ((kTileW + kTileP) + 127) & ~127;
  unsigned char* const tile_base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(pf_words) + 127) & ~(uintptr_t)127);
  unsigned char* const my_tiles = tile_base + (size_t)warp * 2 * kTileBuf;
  unsigned tma_phase = 0;  // bit b: parity of buffer b's next completion
  if constexpr (kTma) {
    if (lane == 0) {
      mbar_init(&sm.tma_bar[warp][0], 1);
      mbar_init(&sm.tma_bar[warp][1], 1);
      fence_proxy_async();
    }
    __syncwarp();
  }
  // (the geometry is recomputed rather than carried: nothing extra stays live)
  auto prefetch = [&](int bn, int buf) {
    if (bn >= nbox) return;
    if constexpr (kTma) {
      __syncwarp();  // every lane has read this buffer's previous tiles
      if (lane == 0) {
        const int bx = bn % nbx, t = bn / nbx, by = t % nby, bz = t / nby;
        const int gx = (int)org[0] + bx * Box::X, gy = (int)org[1] + by * Box::Y;
        const int gz = (int)(org[2] + bz * Box::Z);
        unsigned char* dst = my_tiles + buf * kTileBuf;
        fence_proxy_async();
        mbar_expect_tx(&sm.tma_bar[warp][buf], kTileW + kTileP);
        tma_load_3d(dst, &P.tmap_words, gx, gy, (int)(gz - g.slab_begin), &sm.tma_bar[warp][buf]);
        tma_load_3d(dst + kTileW, &P.tmap_img, gx * C, gy, (int)(gz - g.data_begin),
                    &sm.tma_bar[warp][buf]);
      }
      return;
    }
    const BoxG q = box_geom(bn);
    if (!q.vec) return;
    if constexpr (!kFirst) cp_async16(my_pfw + buf * 32, lab_r + q.rel);
    if (kPW) {
      const unsigned char* src = reinterpret_cast<const unsigned char*>(img_r + q.rel * C);
      uint32_t* dst = my_pfp + buf * 32 * (kPW ? kPW : 1);
      if (kPW == 4) cp_async16(dst, src);
      else if (kPW == 2) cp_async8(dst, src);
      else
#pragma unroll
        for (int i = 0; i < kPW; ++i) cp_async4(dst + i, src + 4 * i);
    } else if constexpr ((VAR & 32) != 0) {
      // runs wider than one 16-byte cp.async are not staged: pull the next
      // box's pixel lines into L2 so the direct loads do not wait on DRAM
      const unsigned char* src = reinterpret_cast<const unsigned char*>(img_r + q.rel * C);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
      if constexpr (4 * C * (int)sizeof(T) > 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + 128));
    }
  };

  // the warp's first box (its words/pixels load behind the candidate staging)
  prefetch(warp, 0);
  cp_async_commit();

  // ---- candidates of this region (precomputed by k_region_cand) ----
  const int* rc = P.region_cand + (int64_t)blockIdx.x * kRegionCandStride;
  const int total = __ldg(rc);
  // (P.max_cand <= kFastMaxCand; tests lower it to exercise the fallback)
  const int n = total < P.max_cand ? total : P.max_cand;
  // (no barrier: the staging loop below reads sm.id[j] from the thread that
  // wrote it, same j -> thread mapping)
  for (int j = tid; j < n; j += kFastThreads) sm.id[j] = __ldg(rc + 1 + j);
  if (tid == 0) sm.n_cand = n;
  if (total > P.max_cand) {  // uniform over the CTA
    cp_async_wait_all();
    if (tid == 0) atomicAdd(P.counters + 6, 1ull);
    crowded_region<RANK, C>(P, org, hi, zlo, zhi);
    return;
  }

  // ---- stage candidate records (+ one all-inf padding record at slot n) ----
  for (int j = tid; j <= n; j += kFastThreads) {
    float* r = rec + (size_t)j * RS;
    if (j < n) {
      const int kid = sm.id[j];
      // the winner's id and chg sit in its record: one load in the decisions
      r[HO + 2 * C] = __int_as_float(kid);
      r[HO + 2 * C + 1] = __int_as_float(__ldg(P.chg + kid));
      const float2* c32 = P.cur32 + (int64_t)kid * kS2;  // hi/lo split of the current table
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 hl = __ldg(c32 + c);
        r[HO + 2 * c] = hl.x * P.key_scale;  // power-of-two scaling: exact
        r[HO + 2 * c + 1] = hl.y * P.key_scale;
      }
      // anchors stored region-local (32-bit); hi/lo coordinates for the tables
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        sm.anc[j][a] = (short)(a < RANK ? (int)(P.anchors[kid * kMaxRank + a] - org[a]) : 0);
        if (a < RANK) {
          const float2 cp = __ldg(c32 + C + a);
          sm.cpl[j][a] = (cp.x - (float)org[a]) + cp.y;
          cxy[j * 3 + a] = cp;
        }
      }
    } else {
#pragma unroll
      for (int c = 0; c < 2 * C + 2; ++c) r[HO + c] = 0.f;
    }
  }
  // (slot block: 64 * kCompA words, a multiple of 16 bytes)
  for (int i = tid; i < kCap * kCompA / 4; i += kFastThreads)
    reinterpret_cast<int4*>(accs)[i] = make_int4(0, 0, 0, 0);
  for (int i = tid; i < kSlotHash; i += kFastThreads) sm.htab[i] = 0xffff;
  // compaction lists start as valid record offsets: a voxel without any kept
  // candidate still reads a (never used) winner record
  for (int i = tid; i < kWarps * (kFastMaxCand + 8); i += kFastThreads) (&sm.wl[0][0])[i] = 0;
  __syncthreads();
  for (int j = tid; j < n; j += kFastThreads) {  // id -> slot hash (linear probing)
    int h = slot_hash((uint32_t)sm.id[j]);
    while (atomicCAS(&sm.htab[h], (unsigned short)0xffff, (unsigned short)j) != 0xffff)
      h = (h + 1) & (kSlotHash - 1);
  }
  {
    // spatial tables: one warp per candidate, lanes over the entries of the x
    // segment, then of the y|z segment (z entries follow y: both sit at
    // RXp + r0). Per-axis values are warp-uniform scalars (no dynamic
    // indexing of the axis arrays).
    const float msq = (float)g.m_sq * P.key_scale2;
    const int ox32 = (int)org[0], oy32 = (int)org[1], oz32 = RANK == 3 ? (int)org[2] : 0;
    const int sgx = (int)g.grid[0], sgy = (int)g.grid[1], sgz = RANK == 3 ? (int)g.grid[2] : 0;
    const float ivx = P.inv_grid[0], ivy = P.inv_grid[1], ivz = P.inv_grid[2];
    const int per_yz = RY + (RANK == 3 ? RZ : 0);
    for (int j = warp; j <= n; j += kWarps) {
      float* rj = rec + (size_t)j * RS;
      const bool real = j < n;
      const int jj = real ? j : 0;
      const int anx = sm.anc[jj][0], any_ = sm.anc[jj][1], anz = sm.anc[jj][2];
      const float2 ccx = cxy[jj * 3], ccy = cxy[jj * 3 + 1], ccz = cxy[jj * 3 + 2];
      for (int r = lane; r < RX; r += 32) {
        const int dx = r - anx;
        const float x = (float)(ox32 + r);
        const float t = ((ccx.x - x) + ccx.y) * ivx;
        rj[r] = real & (dx >= -sgx) & (dx <= sgx) ? msq * (t * t) : kSentinel;
      }
      for (int r0 = lane; r0 < per_yz; r0 += 32) {
        const bool isz = RANK == 3 && r0 >= RY;
        const int r = isz ? r0 - RY : r0;
        const int dx = r - (isz ? anz : any_);
        const int sg = isz ? sgz : sgy;
        const float x = (float)((isz ? oz32 : oy32) + r);
        const float2 cc = isz ? ccz : ccy;
        const float t = ((cc.x - x) + cc.y) * (isz ? ivz : ivy);
        rj[RXp + r0] = real & (dx >= -sg) & (dx <= sg) ? msq * (t * t) : kSentinel;
      }
    }
  }
  // per axis and box index: the candidates whose window overlaps the box's
  // (clipped) extent on that axis; a box's covering set is the AND of three
  // (one warp per (axis, box index); lanes over candidates j and j + 32)
  for (int t = warp; t < nbx + nby + nbz; t += kWarps) {
    const int a = t < nbx ? 0 : (t < nbx + nby ? 1 : 2);
    const int i = a == 0 ? t : (a == 1 ? t - nbx : t - nbx - nby);
    int lo, hi;
    if (a == 0) {
      lo = i * Box::X;
      hi = min(lo + Box::X - 1, ex);
    } else if (a == 1) {
      lo = i * Box::Y;
      hi = min(lo + Box::Y - 1, ey);
    } else {
      lo = max(i * Box::Z, ez_lo);
      hi = min(i * Box::Z + Box::Z - 1, ez_hi);
    }
    unsigned m2[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      bool c = a >= RANK;
      if (a < RANK && j < n) {
        const int s = g.grid[a];
        const int an = sm.anc[j][a];
        c = an + s >= lo && an - s <= hi;
      }
      m2[h] = __ballot_sync(0xffffffffu, c);
    }
    if (lane == 0) sm.bmask[a][i] = (unsigned long long)m2[1] << 32 | m2[0];
  }
  __syncthreads();

  // persistent per-warp queue of fp64 re-decisions (3 channels, see
  // fast_queue_cap; the others drain per box, inline)
  [[maybe_unused]] uint2* const pq =
      reinterpret_cast<uint2*>(pf_pix + kWarps * 2 * 32 * kPW) + (size_t)warp * kQCap;
  [[maybe_unused]] int pqn = 0;
  // ---- per-warp sweep over the region's boxes ----
  // (a CTA counter handing out boxes dynamically measured 1.4 % slower on
  // config 3: the static split is kept)
  int buf = 0;
  int b_next = warp + kWarps;
  auto advance = [&]() {  // -> the next box
    const int nb = b_next;
    b_next = nb + kWarps;
    return nb;
  };
#pragma unroll 1
  for (int b = warp; b < nbox; b = advance(), buf ^= 1) {
    const BoxG cur = box_geom(b);
    cp_async_wait_all();  // this box's prefetch (issued one box ago)
    const int bx0 = cur.bx0, by0 = cur.by0, bz0 = cur.bz0, bx1 = cur.bx1, by1 = cur.by1;
    const int bz0c = cur.bz0c, bz1 = cur.bz1;
    const unsigned long long bmask =
        sm.bmask[0][cur.bx] & sm.bmask[1][cur.by] & sm.bmask[2][RANK == 3 ? cur.bz : 0];
    if (!cur.nonempty) {  // uniform
      prefetch(b_next, buf ^ 1);
      cp_async_commit();
      continue;
    }
    const int lx0 = cur.lx0, ly = cur.ly, lz = cur.lz;
    const bool row_ok = kFull || (ly <= by1 && (RANK == 2 || (lz >= bz0c && lz <= bz1)));
    bool valid[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) valid[v] = kFull || (row_ok && lx0 + v <= ex && lx0 + v < RX);

    // label words + pixels (prefetched, or direct loads for clipped boxes)
    const int64_t gx0 = org[0] + lx0, gy = org[1] + ly, gz = org[2] + lz;
    const int rel = cur.rel;
    const bool vec = cur.vec;
    uint32_t word[4];
    float p[4][C];
    const T* px = img_r + rel * C;
    if constexpr (kTma) {
      mbar_wait(&sm.tma_bar[warp][buf], (tma_phase >> buf) & 1u);
      tma_phase ^= 1u << buf;
    }
    const int toff = (zq * Box::Y + yq) * Box::X + 4 * xq;  // lane's run in the 8x4x4 tiles
    if constexpr (kFirst) {
#pragma unroll
      for (int v = 0; v < 4; ++v) word[v] = kUndefined;
    } else if (kTma) {
      const uint4 q = *reinterpret_cast<const uint4*>(my_tiles + buf * kTileBuf + 4 * toff);
      word[0] = q.x;
      word[1] = q.y;
      word[2] = q.z;
      word[3] = q.w;
    } else if (vec) {
      const uint4 q = my_pfw[buf * 32];
      word[0] = q.x;
      word[1] = q.y;
      word[2] = q.z;
      word[3] = q.w;
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) word[v] = valid[v] ? lab_r[rel + v] : kUndefined;
    }
    if constexpr (kTma) {
      const T* tp = reinterpret_cast<const T*>(my_tiles + buf * kTileBuf + kTileW) + toff * C;
      T vals[4 * C];
      memcpy(vals, tp, sizeof(vals));
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int c = 0; c < C; ++c) p[v][c] = (float)vals[v * C + c];
    } else if constexpr (kPW > 0) {
      if (vec) {
        uint32_t w[kPW];
#pragma unroll
        for (int i = 0; i < kPW; ++i) w[i] = my_pfp[buf * 32 * kPW + i];
        T vals[4 * C];
        static_assert(sizeof(vals) == sizeof(w), "prefetched pixel run size");
        memcpy(vals, w, sizeof(vals));
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int c = 0; c < C; ++c) p[v][c] = (float)vals[v * C + c];
      } else {
        load_run<C, T>(px, false, valid, p);
      }
    } else {
      load_run<C, T>(px, vec, valid, p);
    }

    // carried-over centres (history tables), once per distinct label word
    int rep[4];
    bool any_undef = false;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      rep[v] = v > 0 && word[v] == word[v - 1] ? rep[v - 1] : v;
      any_undef |= valid[v] & (word[v] == kUndefined);
      if constexpr (!kFirst) {  // predicated copies (no branch per voxel)
        const bool need = (rep[v] == v) & valid[v] & (word[v] != kUndefined);
        const uint32_t L = word[v] & lmask, Tg = word[v] >> lbits;
        // (history rows < 2^32: tag mode caps the tables at 8 GB)
        const float2* hc = P.hist32 + (size_t)(Tg * (uint32_t)g.k + L) * kS2;
#pragma unroll
        for (int i = 0; i < kS2; i += 2) cp_async16_if(my_stage + v * 32 * kS2 + i, hc + i, need);
      }
    }
    cp_async_commit();
    prefetch(b_next, buf ^ 1);  // next box, own group (left in flight below)
    cp_async_commit();

    // box pixel range per channel (scaled domain) for the candidates' lower bounds
    // (warp min/max via redux.sync on order-preserving integer images of the
    // floats: u8/u16 values are non-negative; f32 values use the sign flip)
    float pmin[C], pmax[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      uint32_t lo = 0xffffffffu, hv = 0u;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint32_t o = __float_as_uint(p[v][c]);
        if (sizeof(T) == 4) o ^= (o >> 31) ? 0xffffffffu : 0x80000000u;
        lo = valid[v] ? min(lo, o) : lo;
        hv = valid[v] ? max(hv, o) : hv;
      }
      lo = __reduce_min_sync(0xffffffffu, lo);
      hv = __reduce_max_sync(0xffffffffu, hv);
      if (sizeof(T) == 4) {
        lo ^= (lo >> 31) ? 0x80000000u : 0xffffffffu;
        hv ^= (hv >> 31) ? 0x80000000u : 0xffffffffu;
      }
      pmin[c] = __uint_as_float(lo) * ks;
      pmax[c] = __uint_as_float(hv) * ks;
      if constexpr (kF64) {  // the true values lie within pix_err of the f32 copy
        pmin[c] -= P.pix_err;
        pmax[c] += P.pix_err;
      }
    }

    // candidates covering this box and their lower bound over the box
    // (colour distance to the box's value range + spatial distance to the
    // box), computed while the history rows are in flight
    bool cov[2];
    float lbv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const bool c = (uint32_t)(bmask >> (32 * h)) >> lane & 1u;
      float lb = 0.f;
      {  // (computed for every lane, j < kFastMaxCand records exist; masked by c)
        const float* r = rec + j * RS;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
          const float ch = r[HO + 2 * cc], cl = fabsf(r[HO + 2 * cc + 1]);
          const float t = fmaxf(fmaxf(pmin[cc] - ch, ch - pmax[cc]) - cl, 0.f);
          lb = fmaf(t, t, lb);
        }
        if constexpr (!(VAR & 1)) {
          float sl = 0.f;
          const int b0[3] = {bx0, by0, bz0c}, b1[3] = {bx1, by1, bz1};
#pragma unroll
          for (int a = 0; a < RANK; ++a) {
            const float cpl = sm.cpl[j][a];
            const float t = fmaxf(fmaxf((float)b0[a] - cpl, cpl - (float)b1[a]) - 1e-3f, 0.f) *
                            P.inv_grid[a];
            sl = fmaf(t, t, sl);
          }
          lb = fmaf(sl, (float)g.m_sq * P.key_scale2, lb);
        }
      }
      cov[h] = c;
      lbv[h] = lb * (1.0f - 4.0f * M);
    }

    // fp32 d_old (scaled), an upper bound of it, and the box maximum.
    // Branch-free over the 4 voxels so their dependency chains interleave;
    // voxels without a carried-over distance read a (finite or not) dummy
    // row and are masked afterwards.
    cp_async_wait_group1();  // history rows (the next box's prefetch may stay in flight)
    float dold[4];
    float dmax = 0.f;
    float fx[3] = {(float)gx0, (float)gy, (float)gz};
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float2* hc = my_stage + rep[v] * 32 * kS2;
      float sp = 0.f;
#pragma unroll
      for (int a = 0; a < RANK; ++a) {
        const float2 cc = hc[C + a];
        const float x = a == 0 ? fx[0] + (float)v : fx[a];
        const float t = ((cc.x - x) + cc.y) * P.inv_grid[a];
        sp = fmaf(t, t, sp);
      }
      float d = sp * (float)g.m_sq;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 cc = hc[c];
        const float e = (cc.x - p[v][c]) + cc.y;
        d = fmaf(e, e, d);
      }
      const bool has = valid[v] && word[v] != kUndefined;
      dold[v] = has ? d * P.key_scale2 : kInf;
      dmax = has ? fmaxf(dmax, dold[v]) : dmax;
    }
    if constexpr (kFirst) {
      // no finite d_old bounds undefined voxels; the smallest upper bound of
      // a candidate that covers the whole box does (box_upper_bound)
      const int b0[3] = {bx0, by0, bz0c}, b1[3] = {bx1, by1, bz1};
      const int sg[3] = {(int)g.grid[0], (int)g.grid[1], RANK == 3 ? (int)g.grid[2] : 0};
      float ub = kInf;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        ub = fminf(ub, box_upper_bound<RANK, C>(sm, rec + j * RS + HO, j, cov[h], pmin, pmax, b0,
                                                b1, sg, P.inv_grid,
                                                (float)g.m_sq * P.key_scale2));
      }
      ub = __uint_as_float(__reduce_min_sync(0xffffffffu, __float_as_uint(ub)));
      dmax = (ub * (1.0f + 4.0f * M) + A) * (1.0f + M) + A;
    } else {
      dmax = any_undef ? kInf : dmax * (1.0f + M) + A;
      dmax = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(dmax)));
    }

    // candidates covering this box whose lower bound over the box can beat
    // some voxel's d_old -> compact warp list (padded to pairs). A candidate
    // with LB > max d_old is provably never chosen in this box (its distance
    // exceeds every voxel's carried-over distance), so skipping it is exact.
    __syncwarp();
    int nl;
    {
      bool keep[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) keep[h] = cov[h] && lbv[h] <= dmax;
      const unsigned m0 = __ballot_sync(0xffffffffu, keep[0]);
      const unsigned m1 = __ballot_sync(0xffffffffu, keep[1]);
      const unsigned lt = (1u << lane) - 1u;
      if (keep[0]) {
        const int pos = __popc(m0 & lt);
        sm.wl[warp][pos] = (uint32_t)(lane * RS);
      }
      if (keep[1]) {
        const int pos = __popc(m0) + __popc(m1 & lt);
        sm.wl[warp][pos] = (uint32_t)((lane + 32) * RS);
      }
      nl = __popc(m0) + __popc(m1);
      if (lane == 0 && (nl & 1)) {  // pad to a pair: sentinel record
        sm.wl[warp][nl] = (uint32_t)(n * RS);
      }
      __syncwarp();
    }
    const int nlp = (nl + 1) & ~1;
#pragma unroll
    for (int v = 0; v < 4; ++v) n_evals += valid[v] ? nl : 0;

    f2 p01[C], p23[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      p01[c] = pk2(p[0][c] * ks, p[1][c] * ks);
      p23[c] = pk2(p[2][c] * ks, p[3][c] * ks);
    }
    const int ox = lx0 < RXp ? lx0 : 0;
    const int oy = RXp + (ly < RY ? ly : 0);
    const int oz = RXp + RY + (lz < RZ ? lz : 0);

    // fp32 argmin with runner-up over the kept candidates: keys carry the
    // position in the current group of 8 in their 3 low bits
    uint32_t best[4], second[4];
    int grp[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      best[v] = second[v] = 0xffffffffu;
      grp[v] = 0;
    }
    // the next pair of record offsets is loaded one step ahead (the list is
    // padded, so reading one pair past the end stays inside wl)
    const uint2* wl2 = reinterpret_cast<const uint2*>(sm.wl[warp]);
    uint2 pr = wl2[0];
#pragma unroll 1
    for (int g0 = 0; g0 < nlp; g0 += 8) {
      uint32_t before[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) before[v] = best[v];
      const int g1 = min(g0 + 8, nlp);
#pragma unroll 1
      for (int jj = g0; jj < g1; jj += 2) {
        uint32_t key[2][4];
        const uint32_t jl0 = (uint32_t)(jj & 7);
        const uint2 cur = pr;
        pr = wl2[(jj >> 1) + 1];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const float* r = rec + (h ? cur.y : cur.x);
          const ulonglong2 sxv = *reinterpret_cast<const ulonglong2*>(r + ox);
          float syz = r[oy];
          if (RANK == 3) syz += r[oz];
          // (a pair built from one scalar is a free broadcast operand of FADD2)
          f2 a01 = add2(sxv.x, pk2(syz, syz)), a23 = add2(sxv.y, pk2(syz, syz));
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const float2 hl = *reinterpret_cast<const float2*>(r + HO + 2 * c);
            const f2 ch = pk2(hl.x, hl.x), cl = pk2(hl.y, hl.y);
            const f2 d01 = add2(sub2(ch, p01[c]), cl);
            const f2 d23 = add2(sub2(ch, p23[c]), cl);
            a01 = fma2(d01, d01, a01);
            a23 = fma2(d23, d23, a23);
          }
          float f0, f1, f2v, f3;
          up2(a01, f0, f1);
          up2(a23, f2v, f3);
          const uint32_t jl = jl0 + h;
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
    // re-decision queue [count | entries...] at the start of the warp's
    // history staging area (its rows were consumed by d_old above)
    int* xcnt = reinterpret_cast<int*>(stage + (size_t)warp * 4 * 32 * kS2);
    uint2* xqueue = reinterpret_cast<uint2*>(xcnt) + 1;
    __syncwarp();
    if (lane == 0) *xcnt = 0;
    __syncwarp();
    // (predicated over the 4 voxels; only the rare fp64 re-decision branches)
    // Undefined words have dold = +inf and oldl = lmask (never a winner), so
    // they need no special case: upd <=> !amb. A runner-up key >= kSentKey
    // decodes to >= 2^-66 > thr, so amb needs no coverage test either.
    uint32_t newl[4], oldl[4];
    uint32_t nword[4];
    unsigned exact_mask = 0, amb_mask = 0;
    int jst[4];
    const float M1 = 1.0f + M;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      // (bitwise & / | on the conditions: no short-circuit branches)
      oldl[v] = word[v] & lmask;  // undefined -> lmask (never a label)
      const bool live = valid[v] & (best[v] < kSentKey);  // else: keep (nothing kept beats d_old)
      const int roff = sm.wl[warp][grp[v] + (best[v] & 7u)];  // winner's record
      const int2 ic = *reinterpret_cast<const int2*>(rec + roff + HO + 2 * C);
      const uint32_t kid = (uint32_t)ic.x;
      const float bv = kval(best[v]);
      const float thr = fmaf(bv, M1, A);
      const bool amb = kval(second[v]) <= thr;
      // same centre as when the label was set: D* == d_old exactly -> keep
      const bool same = (kid == oldl[v]) & (ic.y <= (int)(word[v] >> lbits));
      const bool below = thr < dold[v];
      const bool above = bv > fmaf(dold[v], M1, A);
      const bool upd = !amb & !same & below;
      const bool keep = !amb & (same | above);
      nword[v] = live & upd ? (tag_now_bits | kid) : word[v];
      exact_mask |= (unsigned)(live & !upd & !keep) << v;
      amb_mask |= (unsigned)amb << v;
      jst[v] = roff;
    }
    // undecided voxels are queued in the warp's (now free) history staging
    // area and re-decided in fp64 after the box, one voxel per lane
    if (__any_sync(0xffffffffu, exact_mask != 0)) {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (exact_mask >> v & 1u) {
          // deferred fp64 re-decision: region-local voxel coordinates, amb, slot
          const uint32_t info = (uint32_t)(lx0 + v) | (uint32_t)ly << 6 | (uint32_t)lz << 12 |
                                (amb_mask >> v & 1u) << 18 | (uint32_t)(jst[v] / RS) << 19;
          xqueue[atomicAdd(xcnt, 1)] = make_uint2(word[v], info);
        }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if (valid[v] && nword[v] != word[v]) lab_r[rel + v] = nword[v];
      newl[v] = nword[v] & lmask;
    }

    // ---- delta accumulation: +new / -old for voxels whose label changed ----
    // bit v: +new[v]; bit 4+v: -old[v]. A voxel whose old word is defined
    // has -old exactly when it has +new; an undefined word (new or old) can
    // only occur where the lane saw an undefined old word (any_undef), so
    // the undefined-label bookkeeping runs only in such boxes.
    unsigned chm = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) chm |= (unsigned)(valid[v] & (newl[v] != oldl[v])) << v;
    n_changed += (unsigned)__popc(chm);
    unsigned pending = chm | chm << 4;
    if (__any_sync(0xffffffffu, any_undef)) {
      unsigned undef = 0, olddef = 0;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        undef += (unsigned)(valid[v] & (newl[v] == lmask) & !(exact_mask >> v & 1u));
        olddef |= (unsigned)(oldl[v] != lmask) << v;
      }
      pending = chm | (chm & olddef) << 4;
      const unsigned tu = __reduce_add_sync(0xffffffffu, undef);
      if (lane == 0 && tu) atomicAdd(P.counters, (unsigned long long)tu);  // slic.hpp:330-331
    }
    // Per-lane deltas (the common case): each lane adds its contributions
    // into the CTA slots, consecutive voxels of one label merged into one
    // run (the +new slot is the winner's record, no lookup). A box dominated
    // by one label (uniform regions) is warp-aggregated per label instead.
    const unsigned npend = __reduce_add_sync(0xffffffffu, (unsigned)__popc(pending));
    if (npend != 0) {  // uniform: most boxes have no change after the first iterations
    bool per_lane = npend <= sparse_deltas(C);
    if (!per_lane) {
      const int fb = pending ? __ffs(pending) - 1 : 0;
      const uint32_t first = sel8(newl, oldl, fb);
      const unsigned anyp = __ballot_sync(0xffffffffu, pending != 0);
      const uint32_t l0 = __shfl_sync(0xffffffffu, first, __ffs(anyp) - 1);
      const unsigned same = __ballot_sync(0xffffffffu, pending != 0 && first == l0);
      per_lane = 4 * __popc(same) < 3 * __popc(anyp);
    }
    if (kRolledDeltas && per_lane) {
      // each lane walks its own contributions in a rolled loop (one flush
      // site, compact code; warp iterations = max runs per lane)
      bool open = false;
      int run_sg = 0, run_s = -1, rx = 0, ry = 0, rz = 0, rc = 0;
      uint32_t run_l = 0;
      long long rv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) rv[c] = 0;
#pragma unroll 1
      for (;;) {
        const bool have = pending != 0;
        int q = 0, v = 0, sg = 0;
        uint32_t L = 0;
        if (have) {
          q = __ffs(pending) - 1;
          v = q & 3;
          sg = q >> 2;
          L = sel8(newl, oldl, q);
        }
        if (open && (!have || sg != run_sg || L != run_l)) {
          const long long sgn = run_sg ? -1 : 1;
          if (run_s >= 0) {
            AccT* a = accs + run_s * kCompA;
#pragma unroll
            for (int c = 0; c < C; ++c) slot_add_val(a, c, sgn * rv[c]);
            slot_add(a, C, sgn * rx);
            slot_add(a, C + 1, sgn * ry);
            if (RANK == 3) slot_add(a, C + 2, sgn * rz);
            slot_add(a, kStride, sgn * rc);
          } else {  // label outside the region's candidates: global, absolute coordinates
            unsigned long long* a = P.acc + (uint64_t)run_l * kComp;
#pragma unroll
            for (int c = 0; c < C; ++c) atomicAdd(a + c, (unsigned long long)(sgn * rv[c]));
            atomicAdd(a + C, (unsigned long long)(sgn * (rx + rc * org[0])));
            atomicAdd(a + C + 1, (unsigned long long)(sgn * (ry + rc * org[1])));
            if (RANK == 3) atomicAdd(a + C + 2, (unsigned long long)(sgn * (rz + rc * org[2])));
            atomicAdd(a + kStride, (unsigned long long)(sgn * rc));
          }
          open = false;
        }
        if (!have) break;
        pending &= pending - 1;
        if (!open) {
          open = true;
          run_sg = sg;
          run_l = L;
          const int js = (int)sel4(jst[0], jst[1], jst[2], jst[3], v);
          run_s = sg ? slot_of(sm, L) : (int)(((uint32_t)js * rs_m) >> 16);
          rx = ry = rz = rc = 0;
#pragma unroll
          for (int c = 0; c < C; ++c) rv[c] = 0;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float pv = __uint_as_float(sel4(__float_as_uint(p[0][c]), __float_as_uint(p[1][c]),
                                                __float_as_uint(p[2][c]), __float_as_uint(p[3][c]), v));
          if constexpr (kF64) rv[c] += to_fixed(imgx_r[(rel + v) * C + c], P.shift);
          else if (sizeof(T) < 4) rv[c] += (long long)(int)pv;
          else rv[c] += __float2ll_rn(pv * fscale);  // exact: |v| 2^s < 2^40
        }
        rx += lx0 + v;
        ry += ly;
        rz += lz;
        ++rc;
      }
      pending = 0;
    } else if (per_lane) {
      // Unrolled over the lane's 4 voxels (one warp instruction serves every
      // lane): per sign, consecutive voxels of one label are merged into the
      // first of the run, then each run head adds into its slot.
      using VT = typename std::conditional<kFloatAcc, long long, int>::type;
      VT bv[4][C];
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if constexpr (kF64)
            bv[v][c] = ((pending >> v | pending >> (4 + v)) & 1u)
                           ? to_fixed(imgx_r[(rel + v) * C + c], P.shift)
                           : 0;
          else if constexpr (sizeof(T) < 4) bv[v][c] = (int)p[v][c];
          else bv[v][c] = __float2ll_rn(p[v][c] * fscale);  // exact: |v| 2^s < 2^40
        }
#pragma unroll
      for (int sg = 0; sg < 2; ++sg) {
        VT iv[4][C];
        int xs[4], cn[4];
        bool pf[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          pf[v] = pending >> (v + 4 * sg) & 1u;
          xs[v] = lx0 + v;
          cn[v] = 1;
#pragma unroll
          for (int c = 0; c < C; ++c) iv[v][c] = bv[v][c];
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
          const int S = sg ? slot_of(sm, L) : (int)(((uint32_t)jst[v] * rs_m) >> 16);
          if (S >= 0) {
            AccT* a = accs + S * kCompA;
#pragma unroll
            for (int c = 0; c < C; ++c) slot_add_val(a, c, sgn * (long long)iv[v][c]);
            slot_add(a, C, sgn * xs[v]);
            slot_add(a, C + 1, sgn * cn[v] * ly);
            if (RANK == 3) slot_add(a, C + 2, sgn * cn[v] * lz);
            slot_add(a, kStride, sgn * cn[v]);
          } else {  // label outside the region's candidates: global, absolute coordinates
            unsigned long long* a = P.acc + (uint64_t)L * kComp;
            const long long cl = sgn * cn[v];
#pragma unroll
            for (int c = 0; c < C; ++c)
              atomicAdd(a + c, (unsigned long long)(sgn * (long long)iv[v][c]));
            atomicAdd(a + C, (unsigned long long)(sgn * xs[v] + cl * org[0]));
            atomicAdd(a + C + 1, (unsigned long long)(cl * (ly + org[1])));
            if (RANK == 3) atomicAdd(a + C + 2, (unsigned long long)(cl * (lz + org[2])));
            atomicAdd(a + kStride, (unsigned long long)cl);
          }
        }
      }
      pending = 0;
    }
#pragma unroll 1
    for (;;) {
      const unsigned any = __ballot_sync(0xffffffffu, pending != 0);
      if (!any) break;
      const int leader = __ffs(any) - 1;
      uint32_t mylab = 0;
      if (pending) {
        const int bit = __ffs(pending) - 1;
        mylab = sel8(newl, oldl, bit);
      }
      const uint32_t L = __shfl_sync(0xffffffffu, mylab, leader);
      int cnt = 0, sxr = 0, syr = 0, szr = 0;
      int sv32[C];
      int64_t sv64[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        sv32[c] = 0;
        sv64[c] = 0;
      }
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
            if constexpr (kF64) sv64[c] += sgn * to_fixed(imgx_r[(rel + v) * C + c], P.shift);
            else if (sizeof(T) < 4) sv32[c] += sgn * (int)p[v][c];
            else sv64[c] += sgn * __float2ll_rn(p[v][c] * fscale);  // exact: |v| 2^s < 2^40
          }
        }
      }
      int tx, ty, tz, tc;
      redux_pair(sxr, syr, tx, ty);
      redux_pair(szr, cnt, tz, tc);
      long long tvs[C];
      if (sizeof(T) == 1) {
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          int a0, a1;
          redux_pair(sv32[c], c + 1 < C ? sv32[c + 1] : 0, a0, a1);
          tvs[c] = a0;
          if (c + 1 < C) tvs[c + 1] = a1;
        }
      } else if (sizeof(T) == 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) tvs[c] = (int)__reduce_add_sync(0xffffffffu, (uint32_t)sv32[c]);
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const uint64_t u = (uint64_t)sv64[c];
          const int32_t h = (int32_t)__reduce_add_sync(0xffffffffu, (uint32_t)(sv64[c] >> 32));
          const uint32_t l1 = __reduce_add_sync(0xffffffffu, (uint32_t)(u & 0xffffu));
          const uint32_t l2 = __reduce_add_sync(0xffffffffu, (uint32_t)((u >> 16) & 0xffffu));
          tvs[c] = (long long)h * 4294967296LL + (long long)l2 * 65536LL + (long long)l1;
        }
      }
      if (lane == leader) {
        const int S = slot_of(sm, L);
        if (S >= 0) {
          AccT* a = accs + S * kCompA;
#pragma unroll
          for (int c = 0; c < C; ++c)
            if (tvs[c]) slot_add_val(a, c, tvs[c]);
          if (tx) slot_add(a, C, tx);
          if (ty) slot_add(a, C + 1, ty);
          if (RANK == 3 && tz) slot_add(a, C + 2, tz);
          if (tc) slot_add(a, kStride, tc);
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

    }  // npend != 0

    if constexpr (kQCap > 0) {
      // (the fp64 re-decision is a non-inlined call: rare, and kept out of
      // the sweep's register allocation)
      auto drain = [&](const uint2* q, int cnt) {
        for (int i0 = 0; i0 < cnt; i0 += 32) {
          const int i = i0 + lane;
          if (i < cnt) {
            n_changed += redecide_queued<RANK, C, TS>(P, sm, accs, org, lab_r, img_r, imgx_r, s1,
                                                      s2, split16, q[i]);
            ++n_redecided;
          }
        }
      };
    // ---- deferred fp64 re-decisions of this box (batched per warp) ----
    // The box's queued voxels move to the warp's persistent queue, which is
    // re-decided one voxel per lane once it holds a full warp (or at the end
    // of the region): one fp64 pass serves up to 32 voxels instead of the
    // one or two a box typically has.
    __syncwarp();
    const int nq = *xcnt;
    if (nq > 0) {  // uniform
      if (kQCap > 0 && pqn + nq <= kQCap) {
        for (int i = lane; i < nq; i += 32) pq[pqn + i] = xqueue[i];
        pqn += nq;
        if (pqn >= 32) {
          __syncwarp();
          drain(pq, pqn);
          pqn = 0;
        }
      } else {
        drain(xqueue, nq);
      }
      __syncwarp();
    }
    } else {
    // ---- deferred fp64 re-decisions of this box (one queued voxel per lane) ----
    __syncwarp();
    const int nq = *xcnt;
    if (nq > 0) {  // uniform
      for (int i0 = 0; i0 < nq; i0 += 32) {
        const int i = i0 + lane;
        if (i < nq) {
          const uint2 e = xqueue[i];
          const int qx = (int)(e.y & 63u), qy = (int)(e.y >> 6 & 63u), qz = (int)(e.y >> 12 & 63u);
          const bool qamb = e.y >> 18 & 1u;
          const int qj = (int)(e.y >> 19 & 63u);
          const int qrel = qx + qy * s1 + qz * s2;
          const T* qpx = img_r + (size_t)qrel * C;
          const uint32_t nw = exact_region_voxel(P, sm, org[0] + qx, org[1] + qy, org[2] + qz,
                                                 qpx - static_cast<const T*>(P.img), e.x, qamb, qj,
                                                 org);
          ++n_redecided;
          const uint32_t ol = e.x & lmask, nl2 = nw & lmask;
          if (nw != e.x) lab_r[qrel] = nw;
          if (nl2 == lmask) atomicAdd(P.counters, 1ull);  // slic.hpp:330-331
          if (nl2 != ol) {
            ++n_changed;
            const long long co[3] = {qx, qy, qz};
#pragma unroll 1
            for (int sg = 0; sg < 2; ++sg) {
              const uint32_t L = sg == 0 ? nl2 : ol;
              if (L == lmask) continue;
              const long long sgn = sg == 0 ? 1 : -1;
              const int S = slot_of(sm, L);
              long long val[C];
#pragma unroll
              for (int c = 0; c < C; ++c) {
                const T raw = qpx[c];
                if constexpr (kF64) val[c] = to_fixed(imgx_r[(int64_t)qrel * C + c], P.shift);
                else val[c] = sizeof(T) < 4 ? (long long)raw
                                            : (long long)__float2ll_rn((float)raw * fscale);
              }
              if (S >= 0) {
                AccT* a = accs + S * kCompA;
#pragma unroll
                for (int c = 0; c < C; ++c) slot_add_val(a, c, sgn * val[c]);
#pragma unroll
                for (int ax = 0; ax < RANK; ++ax) slot_add(a, C + ax, sgn * co[ax]);
                slot_add(a, kStride, sgn);
              } else {
                unsigned long long* a = P.acc + (uint64_t)L * kComp;
#pragma unroll
                for (int c = 0; c < C; ++c) atomicAdd(a + c, (unsigned long long)(sgn * val[c]));
#pragma unroll
                for (int ax = 0; ax < RANK; ++ax)
                  atomicAdd(a + C + ax, (unsigned long long)(sgn * (co[ax] + org[ax])));
                atomicAdd(a + kStride, (unsigned long long)sgn);
              }
            }
          }
        }
      }
    }
    }
  }
  if constexpr (kQCap > 0) {
      auto drain = [&](const uint2* q, int cnt) {
        for (int i0 = 0; i0 < cnt; i0 += 32) {
          const int i = i0 + lane;
          if (i < cnt) {
            n_changed += redecide_queued<RANK, C, TS>(P, sm, accs, org, lab_r, img_r, imgx_r, s1,
                                                      s2, split16, q[i]);
            ++n_redecided;
          }
        }
      };
      if (pqn > 0) {
        __syncwarp();
        drain(pq, pqn);
      }
  }
  cp_async_wait_all();
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
  // 128-register kernels: one (candidate, component) pair per thread (every
  // lane busy; config 4 -4 %); the 96-register ones keep one warp per
  // candidate (the pair loop costs them spills)
  if constexpr (fast_min_blocks(C, VAR) == 4) {
    for (int t = tid; t < n * kComp; t += kFastThreads) {
      const int j = t / kComp, cp = t - j * kComp;
      long long v = (long long)accs[j * kCompA + cp];
      if (cp < C) {
        const int h = accs[j * kCompA + kComp + cp];
        if constexpr (kFloatAcc)
          v = (long long)((unsigned long long)(uint32_t)v | (unsigned long long)(uint32_t)h << 32);
        else
          v += 256LL * (long long)h;
      } else if (cp < kStride) {
        v += (long long)accs[j * kCompA + kStride] * org[cp - C];
      }
      if (v) atomicAdd(P.acc + (uint64_t)sm.id[j] * kComp + cp, (unsigned long long)v);
    }
  } else {
    for (int j = warp; j < n; j += kWarps) {
      if (lane < kComp) {
        long long v = (long long)accs[j * kCompA + lane];
        if (lane < C) {
          const int h = accs[j * kCompA + kComp + lane];
          if constexpr (kFloatAcc)
            v = (long long)((unsigned long long)(uint32_t)v | (unsigned long long)(uint32_t)h << 32);
          else
            v += 256LL * (long long)h;
        }
        if (lane >= C && lane < kStride) v += (long long)accs[j * kCompA + kStride] * org[lane - C];
        if (v) atomicAdd(P.acc + (uint64_t)sm.id[j] * kComp + lane, (unsigned long long)v);
      }
    }
  }
}


// Candidate list of every region (one warp per region): the clusters binned
// in the anchor cells within one cell of the region box, in
// cell order. Written as [count, ids...]; count > kFastMaxCand marks a
// crowded region (the main kernel then takes the exact generic path).
template <int RANK>
__global__ void __launch_bounds__(128) k_region_cand(FastParams P, int64_t nregions) {
  const Geom& g = P.g;
  const int lane = threadIdx.x & 31;
  const int64_t region = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (region >= nregions) return;
  int64_t rb = region;
  const int rxi = (int)(rb % P.nreg[0]);
  rb /= P.nreg[0];
  const int ryi = (int)(rb % P.nreg[1]);
  rb /= P.nreg[1];
  const int rzi = (int)rb;
  const int64_t org[3] = {(int64_t)rxi * P.R[0], (int64_t)ryi * P.R[1],
                          RANK == 3 ? P.reg_z0 + (int64_t)rzi * P.R[2] : 0};
  const int64_t hi[3] = {min(org[0] + P.R[0], g.dims[0]) - 1, min(org[1] + P.R[1], g.dims[1]) - 1,
                         RANK == 3 ? min(org[2] + P.R[2], g.dims[2]) - 1 : 0};
  const int64_t zlo = RANK == 3 ? max(org[2], g.slab_begin) : 0;
  const int64_t zhi = RANK == 3 ? min(hi[2], g.slab_end - 1) : 0;
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
  int* out = P.region_cand_out + region * kRegionCandStride;
  int total = 0;
  for (int base = 0; base < nc; base += 32) {
    const int i = base + lane;
    int cnt = 0, cstart = 0;
    if (i < nc) {
      const int nx = chi[0] - clo[0] + 1, ny = chi[1] - clo[1] + 1;
      const int cx = clo[0] + i % nx, cy = clo[1] + (i / nx) % ny, cz = clo[2] + i / (nx * ny);
      const int64_t cell = ((int64_t)cz * g.cells[1] + cy) * g.cells[0] + cx;
      cstart = __ldg(P.cell_start + cell);
      cnt = __ldg(P.cell_start + cell + 1) - cstart;
    }
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = total + incl - cnt;
    for (int q = 0; q < cnt; ++q)
      if (excl + q < kFastMaxCand) out[1 + excl + q] = __ldg(P.items + cstart + q);
    total += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) out[0] = total;
}

// Region extents R_a = f_a S_a: grown greedily (smallest extent first) while
// the region has < 8192 voxels, every extent stays <= 64 and the anchor-cell
// neighbourhood prod (f_a + 2) stays <= 48 cells (headroom to kFastMaxCand
// for drifted centres). Larger regions amortize the per-CTA staging.
inline void region_extents(const Geom& g, int* R) {
  // Grow cell-aligned regions (fewer CTAs, more voxels per candidate
  // staging) up to 8192 voxels, <= 48 cells of candidates, <= 64 per axis,
  // but keep at least ~8 CTAs per SM on small images (a 512^2 image would
  // otherwise be 64 CTAs on 148 SMs).
  int64_t nvox = 1;
  for (int a = 0; a < g.rank; ++a)
    nvox *= (a == g.rank - 1 && g.rank == 3) ? (g.slab_end - g.slab_begin) : g.dims[a];
  const int64_t vox_cap = nvox / (8 * 148);
  int f[3] = {1, 1, 1};
  for (;;) {
    int best = -1;
    for (int a = 0; a < g.rank; ++a) {
      if ((f[a] + 1) * g.grid[a] > kFastMaxR) continue;
      int cells = 1;
      for (int b = 0; b < g.rank; ++b) cells *= f[b] + 2 + (b == a ? 1 : 0);
      if (cells > 48) continue;
      if (best < 0 || f[a] * g.grid[a] < f[best] * g.grid[best]) best = a;
    }
    int64_t vox = 1;
    for (int a = 0; a < g.rank; ++a) vox *= (int64_t)f[a] * g.grid[a];
    if (best < 0 || vox >= 8192) break;
    if (vox / f[best] * (f[best] + 1) > vox_cap) break;
    ++f[best];
  }
  for (int a = 0; a < 3; ++a) R[a] = a < g.rank ? f[a] * g.grid[a] : 1;
  // the x extent must be a multiple of 4 for the vector path; keep >= 8
  if (R[0] < 8) R[0] = g.grid[0] * ((8 + g.grid[0] - 1) / g.grid[0]);
}

inline int64_t fast_region_count(const Geom& g) {
  int R[3];
  region_extents(g, R);
  int64_t n = 1;
  for (int a = 0; a < g.rank; ++a) {
    const int r = R[a];
    if (a == g.rank - 1 && g.rank == 3) {
      const int64_t z0 = g.slab_begin / r * r;
      n *= (g.slab_end - z0 + r - 1) / r;
    } else {
      n *= (g.dims[a] + r - 1) / r;
    }
  }
  return n;
}

// hi/lo fp32 split of one centre table (for the fp32 d_old filter); entries
// padded to hist32_stride(stride) float2 (16-byte multiples, zero padding).
static __global__ void k_split32(const double* c, float2* out, int64_t k, int stride) {
  const int s2 = hist32_stride(stride);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= k * s2) return;
  const int64_t id = i / s2;
  const int comp = (int)(i - id * s2);
  if (comp >= stride) {
    out[i] = make_float2(0.f, 0.f);
    return;
  }
  const double v = c[id * stride + comp];
  const float h = __double2float_rn(v);
  out[i] = make_float2(h, __double2float_rn(v - (double)h));
}

inline bool fast_path_supported(const Geom& g) {
  if (g.rank != 2 && g.rank != 3) return false;
  if (g.channels < 1 || g.channels > 4) return false;
  // (f64 images sweep an f32 working copy, see k_assign_fast)
  if (g.dtype != SSLIC_U8 && g.dtype != SSLIC_U16 && g.dtype != SSLIC_F32 &&
      g.dtype != SSLIC_F64)
    return false;
  for (int a = 0; a < g.rank; ++a)
    if (g.grid[a] > kFastMaxR) return false;
  if (g.k >= (int64_t)1 << 30) return false;
  {
    int R[3];
    region_extents(g, R);  // 32-bit in-region voxel offsets
    if ((int64_t)R[g.rank - 1] * g.strides[g.rank - 1] >= ((int64_t)1 << 31)) return false;
  }
  for (int a = 0; a < g.rank; ++a)
    if (g.dims[a] >= ((int64_t)1 << 30)) return false;
  return true;
}


// Candidate capacity a region's CTA needs: 1.5x the anchor cells it draws
// from (prod (R_a / S_a + 2)), rounded up to 4.
inline int fast_cand_need(const Geom& g, const int* R) {
  int cells = 1;
  for (int a = 0; a < g.rank; ++a) cells *= R[a] / g.grid[a] + 2;
  return (cells + cells / 2 + 3) & ~3;
}

inline size_t fast_smem_bytes(const Geom& g, const int* R, int cap = kFastMaxCand) {
  const int RXp = (R[0] + 3) & ~3;
  const int HO = (RXp + R[1] + (g.rank == 3 ? R[2] : 0) + 1) & ~1;
  const int RS = (HO + 2 * g.channels + 2 + 3) & ~3;
  const int warps = kFastThreads / 32;
  size_t b = sizeof(FastSmem);
  b += (size_t)(cap + 1) * RS * sizeof(float);
  // CTA delta slots (see k_assign_fast): 32-bit words, C extra per candidate
  b += (size_t)cap * (g.stride + 1 + g.channels) * sizeof(int);
  b += (size_t)warps * 4 * hist32_stride(g.stride) * 32 * sizeof(float2);
  b += (size_t)warps * 2 * 32 * 16;  // next-box label words
  const int wsize = g.dtype == SSLIC_F64 ? 4 : dtype_size(g.dtype);  // working pixel size
  b += (size_t)warps * 2 * 32 * 4 * pf_pix_words(g.channels, wsize);
  b += (size_t)warps * fast_queue_cap(g.channels) * sizeof(uint2);
  b += 128;  // 128-byte alignment of the TMA box tiles (they reuse the prefetch area)
  return b;
}

}  // namespace sslic_b200
#include "kernels_lean.cuh"
namespace sslic_b200 {

// k_assign_lean over the full regions (the compile-time shapes of configs 3
// and 5); returns false when the geometry is not one of them. *all_full:
// no clipped region exists (k_assign_fast then needs no launch).
template <int C, typename T, int RXc, int RYc, int RZc, int CAPc, int MINB, int FIRST = 0>
void launch_lean_shape(const FastParams& P, int64_t nblocks, cudaStream_t s) {
  auto kern = k_assign_lean<C, T, RXc, RYc, RZc, CAPc, MINB, FIRST>;
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  SSLIC_CUDA_CHECK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    SSLIC_CUDA_CHECK(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SSLIC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  const int R[3] = {RXc, RYc, RZc};
  const size_t smem = lean_smem_bytes(P.g, R, CAPc, (int)P.tag_now);
  kern<<<(unsigned)nblocks, kFastThreads, smem, s>>>(P);
}

// Build split (SSLIC_FAST_SPLIT, csrc/Makefile): the kernel instantiations are
// spread over fast_inst_*.cu so they compile in parallel; engine.cu only sees
// declarations. Without the macro this header is self-contained.
#if !defined(SSLIC_FAST_SPLIT)
inline bool launch_lean(const FastParams& P, int64_t nblocks, cudaStream_t s) {
  const Geom& g = P.g;
  if (g.rank != 3 || !P.aligned4 || std::getenv("SSLIC_NO_LEAN") != nullptr) return false;
  const int* R = P.R;
  // config 3 (1 channel, 8.6 evaluations per voxel): measured slower than
  // k_assign_fast (76.8 vs 83.2 Gvox/s, profiles/r2/lean_ab.txt) -- kept
  // behind SSLIC_LEAN_C1=1 for experiments; config 5 gains 11 %
  if (g.channels == 1 && g.dtype == SSLIC_U16 && R[0] == 32 && R[1] == 16 && R[2] == 16 &&
      std::getenv("SSLIC_LEAN_C1") != nullptr && fast_cand_need(g, R) <= 56 &&
      P.max_cand >= 56) {
    FastParams Q = P;
    Q.max_cand = 56;
    launch_lean_shape<1, uint16_t, 32, 16, 16, 56, 5>(Q, nblocks, s);  // config 3
    return true;
  }
  if (g.channels == 3 && g.dtype == SSLIC_U8 && R[0] == 32 && R[1] == 32 && R[2] == 32 &&
      fast_cand_need(g, R) <= 40 && P.max_cand >= 40) {
    FastParams Q = P;
    Q.max_cand = 40;
    if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
      launch_lean_shape<3, uint8_t, 32, 32, 32, 40, 4, 1>(Q, nblocks, s);  // iteration 0
    else
      launch_lean_shape<3, uint8_t, 32, 32, 32, 40, 4>(Q, nblocks, s);  // config 5
    return true;
  }
  return false;
}
#elif defined(SSLIC_FAST_TU_LEAN)
bool launch_lean(const FastParams& P, int64_t nblocks, cudaStream_t s) {
  const Geom& g = P.g;
  if (g.rank != 3 || !P.aligned4 || std::getenv("SSLIC_NO_LEAN") != nullptr) return false;
  const int* R = P.R;
  // config 3 (1 channel, 8.6 evaluations per voxel): measured slower than
  // k_assign_fast (76.8 vs 83.2 Gvox/s, profiles/r2/lean_ab.txt) -- kept
  // behind SSLIC_LEAN_C1=1 for experiments; config 5 gains 11 %
  if (g.channels == 1 && g.dtype == SSLIC_U16 && R[0] == 32 && R[1] == 16 && R[2] == 16 &&
      std::getenv("SSLIC_LEAN_C1") != nullptr && fast_cand_need(g, R) <= 56 &&
      P.max_cand >= 56) {
    FastParams Q = P;
    Q.max_cand = 56;
    launch_lean_shape<1, uint16_t, 32, 16, 16, 56, 5>(Q, nblocks, s);  // config 3
    return true;
  }
  if (g.channels == 3 && g.dtype == SSLIC_U8 && R[0] == 32 && R[1] == 32 && R[2] == 32 &&
      fast_cand_need(g, R) <= 40 && P.max_cand >= 40) {
    FastParams Q = P;
    Q.max_cand = 40;
    if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
      launch_lean_shape<3, uint8_t, 32, 32, 32, 40, 4, 1>(Q, nblocks, s);  // iteration 0
    else
      launch_lean_shape<3, uint8_t, 32, 32, 32, 40, 4>(Q, nblocks, s);  // config 5
    return true;
  }
  return false;
}
#else
bool launch_lean(const FastParams& P, int64_t nblocks, cudaStream_t s);
#endif

// TMA descriptors for the full-region box loads (k_assign_fast VAR & 16):
// label words of the slab (u32) and the image's data planes (channels
// interleaved along x), 8x4x4-voxel boxes. false when TMA is unavailable.
inline bool make_box_tmaps(FastParams& P) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaGetLastError();
  }
  if (!encode) return false;
  const Geom& g = P.g;
  if (g.rank != 3) return false;
  const int esz = dtype_size(g.dtype);
  CUtensorMapDataType dt;
  switch (g.dtype) {
    case SSLIC_U8: dt = CU_TENSOR_MAP_DATA_TYPE_UINT8; break;
    case SSLIC_U16: dt = CU_TENSOR_MAP_DATA_TYPE_UINT16; break;
    case SSLIC_F32: dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    default: return false;
  }
  const cuuint32_t box_w[3] = {(cuuint32_t)BoxShape<3>::X, (cuuint32_t)BoxShape<3>::Y,
                               (cuuint32_t)BoxShape<3>::Z};
  const cuuint32_t box_i[3] = {(cuuint32_t)(BoxShape<3>::X * g.channels),
                               (cuuint32_t)BoxShape<3>::Y, (cuuint32_t)BoxShape<3>::Z};
  const cuuint32_t one[3] = {1, 1, 1};
  const cuuint64_t dw[3] = {(cuuint64_t)g.dims[0], (cuuint64_t)g.dims[1],
                            (cuuint64_t)(g.slab_end - g.slab_begin)};
  const cuuint64_t sw[2] = {(cuuint64_t)g.dims[0] * 4, (cuuint64_t)(g.dims[0] * g.dims[1]) * 4};
  const cuuint64_t di[3] = {(cuuint64_t)(g.dims[0] * g.channels), (cuuint64_t)g.dims[1],
                            (cuuint64_t)(g.data_end - g.data_begin)};
  const cuuint64_t si[2] = {(cuuint64_t)(g.dims[0] * g.channels * esz),
                            (cuuint64_t)(g.dims[0] * g.dims[1] * g.channels * esz)};
  if (box_i[0] * esz % 16 != 0 || sw[0] % 16 || si[0] % 16) return false;
  if (encode(&P.tmap_words, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, P.labels, dw, sw, box_w, one,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (encode(&P.tmap_img, dt, 3, const_cast<void*>(P.img), di, si, box_i, one,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  return true;
}

inline bool all_regions_full(const FastParams& P) {
  const Geom& g = P.g;
  if (g.dims[0] % P.R[0] || g.dims[1] % P.R[1]) return false;
  const int64_t z0 = P.reg_z0, z1 = z0 + (int64_t)P.nreg[2] * P.R[2];
  return z0 >= g.slab_begin && z1 <= g.slab_end;
}

template <int RANK, int C, typename T, int RXc, int RYc, int RZc, int CAPc = 0, int VAR = 0>
void launch_fast_shape(const FastParams& P, size_t smem, int64_t nblocks, cudaStream_t s) {
  auto kern = k_assign_fast<RANK, C, T, RXc, RYc, RZc, CAPc, VAR>;
  // function attributes are per device context: one bit per device
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  SSLIC_CUDA_CHECK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    SSLIC_CUDA_CHECK(
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // all of the unified L1 as shared memory: occupancy is smem/register bound
    SSLIC_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  kern<<<(unsigned)nblocks, kFastThreads, smem, s>>>(P);
}

// Compile-time region shapes for the BASELINE geometries (all address math
// folds into immediates); any other geometry runs the runtime-shape kernel.
template <int RANK, int C, typename T>
void launch_fast_t(const FastParams& P, size_t smem, int64_t nblocks, cudaStream_t s) {
  const int* R = P.R;
  if constexpr (RANK == 3 && C == 1 && sizeof(T) == 2) {
    if (R[0] == 32 && R[1] == 16 && R[2] == 16) {  // config 3
      // The spatial part of a candidate's lower bound over a box is at most
      // m^2 rank (1 + box/S)^2, which cannot prune against carried-over
      // distances of wide-range volumes (u16 data: colour terms dominate;
      // measured: evaluations identical, +2.1 % without it). Pruning is
      // exact either way; this only picks the cheaper kernel.
      const double sp = P.g.m_sq * 3.0 * 4.0, cr = (double)P.vmax / 64.0;
      const bool no_slb = sp < cr * cr && std::getenv("SSLIC_KEEP_SPATIAL_LB") == nullptr;
      // full regions first (clipping folded away), then the clipped ones
      const bool first = P.first && std::getenv("SSLIC_NO_FIRST") == nullptr;
      if (first && P.aligned4) {  // iteration 0: no words, no d_old (VAR & 4)
        if (no_slb) launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 7>(P, smem, nblocks, s);
        else launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 6>(P, smem, nblocks, s);
        if (all_regions_full(P)) return;
        FastParams Q = P;
        Q.skip_full = 1;
        return launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 4>(Q, smem, nblocks, s);
      }
      if (P.aligned4 && std::getenv("SSLIC_NO_FULL") == nullptr) {
        FastParams T2 = P;
        // TMA box tiles: correct, but 7.8 % slower than the per-lane cp.async
        // staging for 8x4x4 boxes (profiles/r2/kernel_ab.txt): opt-in
        const bool tma = std::getenv("SSLIC_TMA") != nullptr && make_box_tmaps(T2);
        if (no_slb && tma) launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 19>(T2, smem, nblocks, s);
        else if (no_slb) launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 3>(P, smem, nblocks, s);
        else if (tma) launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 18>(T2, smem, nblocks, s);
        else launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 2>(P, smem, nblocks, s);
        if (all_regions_full(P)) return;
        FastParams Q = P;
        Q.skip_full = 1;
        if (no_slb) return launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 1>(Q, smem, nblocks, s);
        return launch_fast_shape<RANK, C, T, 32, 16, 16>(Q, smem, nblocks, s);
      }
      if (no_slb) return launch_fast_shape<RANK, C, T, 32, 16, 16, 0, 1>(P, smem, nblocks, s);
      return launch_fast_shape<RANK, C, T, 32, 16, 16>(P, smem, nblocks, s);
    }
  }
  if constexpr (RANK == 3 && C == 4 && sizeof(T) == 4) {
    if (R[0] == 16 && R[1] == 16 && R[2] == 8) {  // config 4
      const bool first = P.first && std::getenv("SSLIC_NO_FIRST") == nullptr;
      if (first && P.aligned4) {
        launch_fast_shape<RANK, C, T, 16, 16, 8, 0, 38>(P, smem, nblocks, s);
        if (all_regions_full(P)) return;
        FastParams Q = P;
        Q.skip_full = 1;
        return launch_fast_shape<RANK, C, T, 16, 16, 8, 0, 4>(Q, smem, nblocks, s);
      }
      if (P.aligned4 && std::getenv("SSLIC_NO_FULL") == nullptr) {
        if (std::getenv("SSLIC_NO_PF_L2") == nullptr)
          launch_fast_shape<RANK, C, T, 16, 16, 8, 0, 34>(P, smem, nblocks, s);
        else
          launch_fast_shape<RANK, C, T, 16, 16, 8, 0, 2>(P, smem, nblocks, s);
        if (all_regions_full(P)) return;
        FastParams Q = P;
        Q.skip_full = 1;
        return launch_fast_shape<RANK, C, T, 16, 16, 8>(Q, smem, nblocks, s);
      }
      return launch_fast_shape<RANK, C, T, 16, 16, 8>(P, smem, nblocks, s);
    }
  }
  if constexpr (RANK == 3 && C == 3 && sizeof(T) == 1) {
    if (R[0] == 32 && R[1] == 32 && R[2] == 32) {  // config 5
      // 32^3 regions of one cell (S = 32) draw from 27 anchor cells: a
      // capacity of 40 records instead of 64 lets 4 CTAs share an SM, not 3
      if (fast_cand_need(P.g, R) <= 40) {
        FastParams Q = P;
        if (Q.max_cand > 40) Q.max_cand = 40;
        if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
          return launch_fast_shape<RANK, C, T, 32, 32, 32, 40, 4>(Q, fast_smem_bytes(P.g, R, 40),
                                                                 nblocks, s);
        return launch_fast_shape<RANK, C, T, 32, 32, 32, 40>(Q, fast_smem_bytes(P.g, R, 40),
                                                            nblocks, s);
      }
      return launch_fast_shape<RANK, C, T, 32, 32, 32>(P, smem, nblocks, s);
    }
  }
  if constexpr (RANK == 2 && C == 3 && sizeof(T) == 4) {
    if (R[0] == 64 && R[1] == 32) {  // config 2
      if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
        return launch_fast_shape<RANK, C, T, 64, 32, 1, 0, 4>(P, smem, nblocks, s);
      return launch_fast_shape<RANK, C, T, 64, 32, 1>(P, smem, nblocks, s);
    }
  }
  if constexpr (RANK == 2 && C == 3 && sizeof(T) == 1) {
    if (R[0] == 16 && R[1] == 16) {  // config 1
      if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
        return launch_fast_shape<RANK, C, T, 16, 16, 1, 0, 4>(P, smem, nblocks, s);
      return launch_fast_shape<RANK, C, T, 16, 16, 1>(P, smem, nblocks, s);
    }
  }
  if (P.first && std::getenv("SSLIC_NO_FIRST") == nullptr)
    return launch_fast_shape<RANK, C, T, 0, 0, 0, 0, 4>(P, smem, nblocks, s);
  launch_fast_shape<RANK, C, T, 0, 0, 0>(P, smem, nblocks, s);
}

template <int RANK, int C>
void launch_fast_c(const FastParams& P, size_t smem, int64_t nb, cudaStream_t s) {
  switch (P.g.dtype) {
    case SSLIC_U8: launch_fast_t<RANK, C, uint8_t>(P, smem, nb, s); break;
    case SSLIC_U16: launch_fast_t<RANK, C, uint16_t>(P, smem, nb, s); break;
    case SSLIC_F64: launch_fast_t<RANK, C, double>(P, smem, nb, s); break;
    default: launch_fast_t<RANK, C, float>(P, smem, nb, s); break;
  }
}

#if defined(SSLIC_FAST_SPLIT) && !defined(SSLIC_FAST_TU_INST)
#define SSLIC_FAST_EXTERN(R, C) \
  extern template void launch_fast_c<R, C>(const FastParams&, size_t, int64_t, cudaStream_t);
SSLIC_FAST_EXTERN(2, 1) SSLIC_FAST_EXTERN(2, 2) SSLIC_FAST_EXTERN(2, 3) SSLIC_FAST_EXTERN(2, 4)
SSLIC_FAST_EXTERN(3, 1) SSLIC_FAST_EXTERN(3, 2) SSLIC_FAST_EXTERN(3, 3) SSLIC_FAST_EXTERN(3, 4)
#undef SSLIC_FAST_EXTERN
#endif

#if !defined(SSLIC_FAST_TU_INST)
template <int RANK>
void launch_fast_r(const FastParams& P, size_t smem, int64_t nb, cudaStream_t s) {
  switch (P.g.channels) {
    case 1: launch_fast_c<RANK, 1>(P, smem, nb, s); break;
    case 2: launch_fast_c<RANK, 2>(P, smem, nb, s); break;
    case 3: launch_fast_c<RANK, 3>(P, smem, nb, s); break;
    default: launch_fast_c<RANK, 4>(P, smem, nb, s); break;
  }
}

#endif  // !SSLIC_FAST_TU_INST

// Relative fp32 decision margin: each fp32
// distance is within (C + 14) u of the fp64 one (u = 2^-24; includes the
// fp32 spatial tables and reciprocal multiplies; the key scaling is exact and
// keys keep every mantissa bit); 2x for the two sides, 1.5x slack.
inline float fast_margin(int channels) {
  const double u = 1.0 / 16777216.0;
  return (float)(1.5 * 2.0 * (channels + 14) * u);
}

#if !defined(SSLIC_FAST_TU_INST)
// (row0 < row1: only region rows [row0, row1) of the slab, z-ordered)
inline void launch_fast_assign(FastParams P, cudaStream_t s, int64_t row0 = 0,
                               int64_t row1 = -1) {
  const Geom& g = P.g;
  region_extents(g, P.R);
  for (int a = 0; a < 3; ++a) {
    P.inv_grid[a] = 1.0f / (float)g.grid[a];
    P.inv_grid64[a] = 1.0 / (double)g.grid[a];
  }
  P.nreg[0] = (int)((g.dims[0] + P.R[0] - 1) / P.R[0]);
  P.nreg[1] = (int)((g.dims[1] + P.R[1] - 1) / P.R[1]);
  if (g.rank == 3) {
    const int64_t z0 = g.slab_begin / P.R[2] * P.R[2];
    P.reg_z0 = z0;
    P.nreg[2] = (int)((g.slab_end - z0 + P.R[2] - 1) / P.R[2]);
    if (row0 < row1) {
      if (row1 > P.nreg[2]) row1 = P.nreg[2];
      P.reg_z0 = z0 + row0 * P.R[2];
      P.nreg[2] = (int)(row1 - row0);
      if (P.nreg[2] <= 0) return;
    }
  } else {
    P.reg_z0 = 0;
    P.nreg[2] = 1;
  }
  // f64 inputs: the f32 working copy rounds each value by e <= |v| 2^-24. By
  // 2|d|e <= eps0 d^2 + e^2/eps0 (eps0 = (C+14) u, the per-distance bound)
  // each fp32 distance is then within 2 eps0 D + A + C (1/eps0 + 1) e^2, so
  // the relative margin doubles (the engine adds the absolute part)
  if (P.max_cand <= 0 || P.max_cand > kFastMaxCand) P.max_cand = kFastMaxCand;
  P.margin = fast_margin(g.channels) * (g.dtype == SSLIC_F64 ? 2.0f : 1.0f);
  // vector loads of 4-voxel runs need 4 | dims[0], 4 | RX and 16-byte bases
  P.aligned4 = (g.dims[0] % 4 == 0 && P.R[0] % 4 == 0 &&
                reinterpret_cast<uintptr_t>(P.img) % 16 == 0 &&
                reinterpret_cast<uintptr_t>(P.labels) % 16 == 0)
                   ? 1
                   : 0;
  const int64_t nb = (int64_t)P.nreg[0] * P.nreg[1] * P.nreg[2];
  const size_t smem = fast_smem_bytes(g, P.R);
  // region candidate lists first (one warp per region), then the sweep
  P.region_cand_out = const_cast<int*>(P.region_cand);
  if (g.rank == 3) {
    k_region_cand<3><<<(unsigned)((nb + 3) / 4), 128, 0, s>>>(P, nb);
    // full regions of configs 3 and 5 take k_assign_lean; the clipped ones
    // (if any) k_assign_fast, which then skips the full ones
    if (launch_lean(P, nb, s)) {
      if (all_regions_full(P)) return;
      P.skip_full = 1;
    }
    launch_fast_r<3>(P, smem, nb, s);
  } else {
    k_region_cand<2><<<(unsigned)((nb + 3) / 4), 128, 0, s>>>(P, nb);
    launch_fast_r<2>(P, smem, nb, s);
  }
}

#endif  // !SSLIC_FAST_TU_INST

}  // namespace sslic_b200
