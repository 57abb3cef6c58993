// Seeded synthetic volumes for the five BASELINE.json configs, generated on
// the device straight into HBM. Counter-based hashing keyed by (seed, voxel)
// makes every z-slab independently reproducible, so a sharded run generates
// exactly the bytes a single-GPU run would. The per-voxel
// construction lives in synth_gen.h, shared with the CPU generator of the
// bench's reference arm (oracle/synth_ref.c); this file is compiled with
// -fmad=false so the device bytes equal the host's (tests/test_gpu_synth.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sslic_b200.h"
#include "synth_gen.h"

namespace {

__global__ void k_seeds(SynthSpec s, SynthSeed* table) {
  const int64_t nb = syn_bin_count(&s);
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id < nb) table[id] = syn_seed(&s, id);
}

__global__ void k_synth(SynthSpec s, const SynthSeed* table, void* out) {
  const int64_t n = s.dims[0] * s.dims[1] * (s.z_end - s.z_begin);
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n;
       li += (int64_t)gridDim.x * blockDim.x)
    syn_voxel(&s, table, li, out);
}

}  // namespace

extern "C" int sslic_synth_generate(int config, int rank, const int64_t* dims, int channels,
                                    int dtype, uint64_t seed, int64_t z_begin, int64_t z_end,
                                    void* dev_out, void* stream) {
  static const int want_dt[6] = {0, SSLIC_U8, SSLIC_F32, SSLIC_U16, SSLIC_F32, SSLIC_U8};
  SynthSpec s{};
  if (config < 1 || config > 5 || dtype != want_dt[config] ||
      syn_spec(&s, config, rank, dims, channels, seed, z_begin, z_end) != 0)
    return SSLIC_EINVAL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nb = syn_bin_count(&s);
  SynthSeed* table = nullptr;
  if (cudaMallocAsync(&table, nb * sizeof(SynthSeed), st) != cudaSuccess) return SSLIC_ENOMEM;
  k_seeds<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(s, table);
  const int64_t n = s.dims[0] * s.dims[1] * (s.z_end - s.z_begin);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_synth<<<(unsigned)blocks, 256, 0, st>>>(s, table, dev_out);
  cudaFreeAsync(table, st);
  return cudaGetLastError() == cudaSuccess ? SSLIC_OK : SSLIC_ECUDA;
}
