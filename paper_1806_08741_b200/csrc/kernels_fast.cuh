// Fast assignment path (fp32 filter + exact fp64 recheck). See DESIGN.md.
#pragma once

#include "common.cuh"
#include "kernels_exact.cuh"

namespace sslic_b200 {

inline bool fast_path_supported(const Geom&) { return false; }

inline void launch_fast_assign(const Geom&, const void*, const double*, const double*,
                               const int*, const int*, const int*, uint32_t*, LabelCodec,
                               uint32_t, int, unsigned long long*, unsigned long long*,
                               unsigned long long*, cudaStream_t) {}

}  // namespace sslic_b200
