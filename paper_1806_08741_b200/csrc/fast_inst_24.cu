// k_assign_fast instantiations for rank 2, 4 channel(s) (all dtypes and
// region shapes): one translation unit per (rank, channels) so the library's
// kernels compile in parallel (csrc/Makefile, SSLIC_FAST_SPLIT).
#define SSLIC_FAST_TU_INST
#include "kernels_fast_main.cuh"

namespace sslic_b200 {
template void launch_fast_c<2, 4>(const FastParams&, size_t, int64_t, cudaStream_t);
}  // namespace sslic_b200
