// Shared device-side definitions for the SSLIC hot path on sm_100a.
//
// Exactness rule: every fp64 operation that must reproduce the reference
// bit-for-bit goes through __dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn, which the
// compiler never contracts into FMA (the reference is built with
// -ffp-contract=off, proj/CMakeLists.txt:18-20).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/sslic_b200.h"

namespace sslic_b200 {

constexpr int kMaxRank = 4;  // image.hpp:25
constexpr uint32_t kUndefined = 0xffffffffu;

// Exceptions thrown by host code and mapped to status codes at the C ABI.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define SSLIC_CUDA_CHECK(expr)                                                        \
  do {                                                                                \
    cudaError_t err__ = (expr);                                                       \
    if (err__ != cudaSuccess)                                                         \
      throw ::sslic_b200::Error(err__ == cudaErrorMemoryAllocation ? SSLIC_ENOMEM     \
                                                                   : SSLIC_ECUDA,     \
                                std::string(#expr) + ": " + cudaGetErrorString(err__)); \
  } while (0)

// Geometry of one image / slab, passed by value to kernels.
struct Geom {
  int rank;
  int channels;
  int stride;                // channels + rank (ClusterTable::stride, slic.hpp:78)
  int dtype;
  int64_t dims[kMaxRank];    // full image extents (1 for unused axes)
  int64_t strides[kMaxRank]; // image.hpp:88-97
  int grid[kMaxRank];        // S per axis (1 for unused axes)
  int cells[kMaxRank];       // ceil(d/S) (1 for unused axes)
  int64_t k;                 // cluster count (table rows)
  int64_t ncells;            // prod cells: anchor-cell bins
  double m_sq;               // weight_m * weight_m (slic.hpp:281)
  // Slab along the last axis: voxels with last coord in [slab_begin, slab_end)
  // are owned; the device image holds planes [data_begin, data_end).
  int64_t slab_begin, slab_end, data_begin, data_end;
  int64_t plane;             // voxels per plane of the last axis
};

// ---- native dtype loads (conversion to fp64 is exact for every dtype) ----
__device__ __forceinline__ double load_value(const void* base, int dtype, int64_t idx) {
  switch (dtype) {
    case SSLIC_U8: return (double)__ldg(static_cast<const uint8_t*>(base) + idx);
    case SSLIC_U16: return (double)__ldg(static_cast<const uint16_t*>(base) + idx);
    case SSLIC_F32: return (double)__ldg(static_cast<const float*>(base) + idx);
    default: return __ldg(static_cast<const double*>(base) + idx);
  }
}

// Pointer to the first channel of the voxel at global flat offset `off`.
__device__ __forceinline__ int64_t data_index(const Geom& g, int64_t off) {
  return (off - g.data_begin * g.plane) * g.channels;
}

// squared_distance_raw (slic.hpp:156-171), exact fp64, fixed order:
// color = ((0 + d0^2) + d1^2) + ..., spatial likewise over axes,
// D = color + m^2 * spatial.
__device__ __forceinline__ double exact_distance(const double* ctr, const double* pix,
                                                 const int64_t* coord, const Geom& g) {
  double color = 0.0;
  for (int c = 0; c < g.channels; ++c) {
    const double d = __dsub_rn(ctr[c], pix[c]);
    color = __dadd_rn(color, __dmul_rn(d, d));
  }
  double spatial = 0.0;
  for (int a = 0; a < g.rank; ++a) {
    const double d = __ddiv_rn(__dsub_rn(ctr[g.channels + a], (double)coord[a]), (double)g.grid[a]);
    spatial = __dadd_rn(spatial, __dmul_rn(d, d));
  }
  return __dadd_rn(color, __dmul_rn(g.m_sq, spatial));
}

// Label words. Tag mode packs (iteration tag, label) into one uint32 so no
// per-voxel distance buffer is needed.
struct LabelCodec {
  int label_bits;     // 32 in dist mode
  uint32_t label_mask;
  __device__ __forceinline__ uint32_t label(uint32_t w) const {
    return w == kUndefined ? kUndefined : (w & label_mask);
  }
  __device__ __forceinline__ uint32_t tag(uint32_t w) const {
    return label_bits >= 32 ? 0u : (w >> label_bits);
  }
  __device__ __forceinline__ uint32_t pack(uint32_t lab, uint32_t t) const {
    return label_bits >= 32 ? lab : ((t << label_bits) | lab);
  }
};

// llround for the non-negative-or-not centre coordinates (slic.hpp:179).
__device__ __forceinline__ int64_t anchor_of(double c) { return llround(c); }

// Fixed-point scale for exact, order-independent int64 accumulation of
// intensities: integer dtypes use scale 2^0; float dtypes use
// 2^shift with shift chosen per image so |v| * 2^shift < 2^40.
__device__ __forceinline__ int64_t to_fixed(double v, int shift) {
  return __double2ll_rn(ldexp(v, shift));
}

}  // namespace sslic_b200
