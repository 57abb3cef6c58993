// k_assign_lean instantiations (launch_lean): their own translation unit
// (csrc/Makefile, SSLIC_FAST_SPLIT).
#define SSLIC_FAST_TU_INST
#define SSLIC_FAST_TU_LEAN
#include "kernels_fast_main.cuh"
