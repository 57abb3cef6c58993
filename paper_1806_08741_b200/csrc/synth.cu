// Seeded synthetic volumes for the five BASELINE.json configs, generated on
// the device straight into HBM. Counter-based hashing keyed by (seed, voxel)
// makes every z-slab independently reproducible, so a sharded run generates
// exactly the bytes a single-GPU run would.
//
// Construction (BASELINE.json "configs"): Voronoi cells from a
// jittered seed grid (one uniform seed per bin, exact nearest seed found in
// the bin neighbourhood), per-cell random means, the config's shading /
// membranes / drift, and additive noise (Irwin-Hall sum of 4 hashed uniforms,
// rescaled to unit variance). The public datasets of the paper (Visible
// Human, FIB-SEM) are not available; these stand in with their shapes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/sslic_b200.h"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(mix64(seed ^ mix64(a)) ^ b);
}
__device__ __forceinline__ float u01(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }
// approximately standard normal: Irwin-Hall(4), variance 4/12 -> rescaled
__device__ __forceinline__ float gauss(uint64_t seed, uint64_t idx, uint64_t stream) {
  const uint64_t h1 = hash3(seed, idx, stream * 2 + 1);
  const uint64_t h2 = mix64(h1);
  const float s = u01(h1) + u01(h1 << 24) + u01(h2) + u01(h2 << 24);
  return (s - 2.0f) * 1.7320508f;
}

struct Spec {
  int rank, channels, dtype, config;
  int64_t dims[3];
  int bins[3];        // jittered seed grid
  float binsz[3];
  int reach[3];       // neighbourhood radius in bins for the exact nearest seed
  uint64_t seed;
  int64_t z_begin, z_end;
};

// Seed position of every bin (one uniform seed per bin).
__global__ void k_seeds(Spec s, float4* table) {
  const int64_t nb = (int64_t)s.bins[0] * s.bins[1] * s.bins[2];
  const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= nb) return;
  const int bx = (int)(id % s.bins[0]), by = (int)((id / s.bins[0]) % s.bins[1]);
  const int bz = (int)(id / ((int64_t)s.bins[0] * s.bins[1]));
  const uint64_t h = hash3(s.seed, (uint64_t)id, 0x5EED);
  table[id] = make_float4((bx + u01(h)) * s.binsz[0], (by + u01(h << 20)) * s.binsz[1],
                          s.rank == 3 ? (bz + u01(h << 40)) * s.binsz[2] : 0.0f, 0.0f);
}

__global__ void k_synth(Spec s, const float4* table, void* out) {
  const int64_t plane = s.dims[0] * s.dims[1];
  const int64_t n = plane * (s.z_end - s.z_begin);
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < n;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = li % s.dims[0];
    const int64_t y = (li / s.dims[0]) % s.dims[1];
    const int64_t z = s.rank == 3 ? s.z_begin + li / plane : 0;
    const int64_t gidx = s.rank == 3 ? z * plane + y * s.dims[0] + x : y * s.dims[0] + x;
    const float px = x + 0.5f, py = y + 0.5f, pz = z + 0.5f;
    const int bx = min((int)(px / s.binsz[0]), s.bins[0] - 1);
    const int by = min((int)(py / s.binsz[1]), s.bins[1] - 1);
    const int bz = s.rank == 3 ? min((int)(pz / s.binsz[2]), s.bins[2] - 1) : 0;
    float d1 = 3.4e38f, d2 = 3.4e38f;
    uint64_t cell = 0;
    const int rz = s.rank == 3 ? s.reach[2] : 0;
    for (int oz = -rz; oz <= rz; ++oz) {
      const int cz = bz + oz;
      if (cz < 0 || cz >= s.bins[2]) continue;
      for (int oy = -s.reach[1]; oy <= s.reach[1]; ++oy) {
        const int cy = by + oy;
        if (cy < 0 || cy >= s.bins[1]) continue;
        for (int ox = -s.reach[0]; ox <= s.reach[0]; ++ox) {
          const int cx = bx + ox;
          if (cx < 0 || cx >= s.bins[0]) continue;
          const float4 p = __ldg(table + ((int64_t)cz * s.bins[1] + cy) * s.bins[0] + cx);
          const float dx = p.x - px, dy = p.y - py, dz = p.z - (s.rank == 3 ? pz : 0.0f);
          const float d = dx * dx + dy * dy + dz * dz;
          if (d < d1) {
            d2 = d1;
            d1 = d;
            cell = ((uint64_t)cz * s.bins[1] + cy) * s.bins[0] + cx;
          } else if (d < d2) {
            d2 = d;
          }
        }
      }
    }
    const uint64_t ch = hash3(s.seed, cell, 0xCE11);
    switch (s.config) {
      case 1: {  // 2D RGB u8, ramp + sigma 8
        uint8_t* o = static_cast<uint8_t*>(out) + li * 3;
        const float ramp = 40.0f * (float)x / (float)s.dims[0] - 20.0f;
        for (int c = 0; c < 3; ++c) {
          const float mean = 255.0f * u01(mix64(ch + c));
          float v = mean + ramp + 8.0f * gauss(s.seed, gidx, c);
          v = fminf(fmaxf(rintf(v), 0.0f), 255.0f);
          o[c] = (uint8_t)v;
        }
        break;
      }
      case 2: {  // 2D RGB f32, sinusoidal shading 0.1 + sigma 0.03
        float* o = static_cast<float*>(out) + li * 3;
        const float shade = 0.1f * __sinf(6.2831853f * (float)x / 512.0f) *
                            __cosf(6.2831853f * (float)y / 384.0f);
        for (int c = 0; c < 3; ++c) {
          const float mean = u01(mix64(ch + c));
          o[c] = mean + shade + 0.03f * gauss(s.seed, gidx, c);
        }
        break;
      }
      case 3: {  // 3D u16, dark blurred membranes, Poisson-like noise
        uint16_t* o = static_cast<uint16_t*>(out) + li;
        const float mean = 5000.0f + 55000.0f * u01(ch);
        // half-gap to the bisector plane ~ (d2 - d1) / (2 |p2 - p1|) ~ (sqrt(d2)-sqrt(d1))/2
        const float w = 0.5f * (sqrtf(d2) - sqrtf(d1));
        const float memb = __expf(-(w * w) / (2.0f * 1.5f * 1.5f));  // 3-voxel blur
        const float lvl = mean * (1.0f - 0.85f * memb);
        float v = lvl + sqrtf(lvl) * gauss(s.seed, gidx, 0);
        v = fminf(fmaxf(rintf(v), 0.0f), 65535.0f);
        *o = (uint16_t)v;
        break;
      }
      case 4: {  // 3D 4-channel f32, 30% of cells near zero in random channels
        float* o = static_cast<float*>(out) + li * 4;
        const bool dark = u01(mix64(ch ^ 0xDA7C)) < 0.3f;
        unsigned subset = (unsigned)(mix64(ch ^ 0x5B5E7) & 0xF);
        if (dark && subset == 0) subset = 1u << (mix64(ch ^ 0x1) & 3);
        for (int c = 0; c < 4; ++c) {
          float mean = u01(mix64(ch + c));
          if (dark && (subset >> c & 1)) mean *= 0.02f;
          o[c] = mean + 0.05f * gauss(s.seed, gidx, c);
        }
        break;
      }
      default: {  // 5: 3D RGB u8, z-dependent drift + sigma 6
        uint8_t* o = static_cast<uint8_t*>(out) + li * 3;
        const float t = (float)z / (float)s.dims[2];
        const float drift[3] = {30.0f * t, -20.0f * t, 25.0f * __sinf(3.14159265f * t)};
        for (int c = 0; c < 3; ++c) {
          const float mean = 20.0f + 215.0f * u01(mix64(ch + c));
          float v = mean + drift[c] + 6.0f * gauss(s.seed, gidx, c);
          v = fminf(fmaxf(rintf(v), 0.0f), 255.0f);
          o[c] = (uint8_t)v;
        }
        break;
      }
    }
  }
}

}  // namespace

extern "C" int sslic_synth_generate(int config, int rank, const int64_t* dims, int channels,
                                    int dtype, uint64_t seed, int64_t z_begin, int64_t z_end,
                                    void* dev_out, void* stream) {
  static const int want_rank[6] = {0, 2, 2, 3, 3, 3};
  static const int want_ch[6] = {0, 3, 3, 1, 4, 3};
  static const int want_dt[6] = {0, SSLIC_U8, SSLIC_F32, SSLIC_U16, SSLIC_F32, SSLIC_U8};
  if (config < 1 || config > 5 || rank != want_rank[config] || channels != want_ch[config] ||
      dtype != want_dt[config])
    return SSLIC_EINVAL;
  Spec s{};
  s.rank = rank;
  s.channels = channels;
  s.dtype = dtype;
  s.config = config;
  s.seed = seed;
  for (int a = 0; a < 3; ++a) s.dims[a] = a < rank ? dims[a] : 1;
  if (rank == 2) {
    z_begin = 0;
    z_end = 1;
  }
  if (z_begin < 0 || z_end > s.dims[2] || z_end <= z_begin) return SSLIC_EINVAL;
  s.z_begin = z_begin;
  s.z_end = z_end;
  // Seed-grid sizes: config 1: 200 cells (20x10), 2: 4000 (80x50),
  // 3: ~30000 (31^3), 4: 8000 (20^3), 5: one per ~40^3.
  int b[3] = {1, 1, 1};
  switch (config) {
    case 1: b[0] = 20; b[1] = 10; break;
    case 2: b[0] = 80; b[1] = 50; break;
    case 3: b[0] = b[1] = b[2] = 31; break;
    case 4: b[0] = b[1] = b[2] = 20; break;
    default:
      for (int a = 0; a < 3; ++a) b[a] = (int)((s.dims[a] + 39) / 40);
  }
  float maxdiag2 = 0.0f;
  for (int a = 0; a < 3; ++a) {
    s.bins[a] = a < rank ? b[a] : 1;
    s.binsz[a] = (float)s.dims[a] / (float)s.bins[a];
    if (a < rank) maxdiag2 += s.binsz[a] * s.binsz[a];
  }
  // A seed k bins away along axis a is >= (k-1)*binsz[a] away; the own seed
  // is <= the bin diagonal away, so reach = floor(diag / binsz) + 1 is exact.
  for (int a = 0; a < 3; ++a)
    s.reach[a] = a < rank ? (int)floorf(sqrtf(maxdiag2) / s.binsz[a]) + 1 : 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nb = (int64_t)s.bins[0] * s.bins[1] * s.bins[2];
  float4* table = nullptr;
  if (cudaMallocAsync(&table, nb * sizeof(float4), st) != cudaSuccess) return SSLIC_ENOMEM;
  k_seeds<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(s, table);
  const int64_t n = s.dims[0] * s.dims[1] * (z_end - z_begin);
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_synth<<<(unsigned)blocks, threads, 0, st>>>(s, table, dev_out);
  cudaFreeAsync(table, st);
  return cudaGetLastError() == cudaSuccess ? SSLIC_OK : SSLIC_ECUDA;
}
