/* Seeded synthetic volumes for the five BASELINE.json configs: the per-voxel
 * generator, shared by the device kernel (synth.cu) and the CPU generator the
 * bench's reference arm uses (oracle/synth_ref.c), so both produce the same
 * bytes without the reference arm loading the product library.
 *
 * Plain C, single precision, only IEEE-exact operations (+ - * /, sqrtf,
 * rintf, integer hashing, power-of-two scaling): compiled without FMA
 * contraction on both sides (nvcc -fmad=false, gcc -ffp-contract=off), every
 * value is bitwise reproducible. exp/sin/cos are fixed polynomials over
 * explicit range reductions, not the libraries' (which differ between the
 * host libm and the device).
 *
 * Construction (BASELINE.json "configs"): Voronoi cells from a
 * jittered seed grid (one uniform seed per bin, exact nearest seed found in
 * the bin neighbourhood), per-cell random means, the config's shading /
 * membranes / drift, and additive noise (Irwin-Hall sum of 4 hashed uniforms,
 * rescaled to unit variance). The paper's datasets (Visible Human, FIB-SEM)
 * are not available; these stand in with their shapes. */
#ifndef SSLIC_SYNTH_GEN_H
#define SSLIC_SYNTH_GEN_H

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD static inline
#endif

typedef struct {
  int rank, channels, config;
  int64_t dims[3];
  int bins[3];  /* jittered seed grid */
  float binsz[3];
  int reach[3]; /* neighbourhood radius in bins for the exact nearest seed */
  uint64_t seed;
  int64_t z_begin, z_end;
} SynthSpec;

typedef struct {
  float x, y, z, w;
} SynthSeed;

SYN_HD uint64_t syn_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
SYN_HD uint64_t syn_hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return syn_mix64(syn_mix64(seed ^ syn_mix64(a)) ^ b);
}
SYN_HD float syn_u01(uint64_t h) { return (float)(h >> 40) * (1.0f / 16777216.0f); }
/* approximately standard normal: Irwin-Hall(4), variance 4/12, rescaled */
SYN_HD float syn_gauss(uint64_t seed, uint64_t idx, uint64_t stream) {
  const uint64_t h1 = syn_hash3(seed, idx, stream * 2 + 1);
  const uint64_t h2 = syn_mix64(h1);
  const float a = syn_u01(h1), b = syn_u01(h1 << 24), c = syn_u01(h2), d = syn_u01(h2 << 24);
  const float s = ((a + b) + c) + d;
  return (s - 2.0f) * 1.7320508f;
}
/* 2^n for integer n in [-126, 127], exact (built from the exponent bits) */
SYN_HD float syn_pow2(int n) {
#ifdef __CUDA_ARCH__
  return __int_as_float((n + 127) << 23);
#else
  union {
    uint32_t u;
    float f;
  } v;
  v.u = (uint32_t)(n + 127) << 23;
  return v.f;
#endif
}
/* exp(x) for x in [-80, 0]: x = n ln2 + r, |r| <= ln2/2, degree-6 Taylor */
SYN_HD float syn_exp(float x) {
  if (x < -80.0f) x = -80.0f;
  const float n = rintf(x * 1.44269504f);
  const float r = (x - n * 0.693145752f) - n * 1.42860677e-6f;
  float p = 1.0f / 720.0f;
  p = p * r + 1.0f / 120.0f;
  p = p * r + 1.0f / 24.0f;
  p = p * r + 1.0f / 6.0f;
  p = p * r + 0.5f;
  p = p * r + 1.0f;
  p = p * r + 1.0f;
  return p * syn_pow2((int)n);
}
/* sin(x) for |x| < ~1e4: x = q pi/2 + r, |r| <= pi/4, Taylor on r */
SYN_HD float syn_sin(float x) {
  const float q = rintf(x * 0.636619772f);
  const float r = (x - q * 1.57079601f) - q * 3.13916473e-7f;
  const float r2 = r * r;
  float s = -1.0f / 5040.0f;
  s = s * r2 + 1.0f / 120.0f;
  s = s * r2 - 1.0f / 6.0f;
  s = (s * r2) * r + r;
  float c = 1.0f / 40320.0f;
  c = c * r2 - 1.0f / 720.0f;
  c = c * r2 + 1.0f / 24.0f;
  c = c * r2 - 0.5f;
  c = c * r2 + 1.0f;
  const int quad = ((int)q) & 3;
  return quad == 0 ? s : quad == 1 ? c : quad == 2 ? -s : -c;
}
SYN_HD float syn_cos(float x) { return syn_sin(x + 1.57079633f); }
SYN_HD float syn_clamp(float v, float lo, float hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Seed-grid sizes: config 1: 200 cells (20x10), 2: 4000 (80x50),
 * 3: ~30000 (31^3), 4: 8000 (20^3), 5: one per ~40^3. Returns 0 or -1. */
SYN_HD int syn_spec(SynthSpec* s, int config, int rank, const int64_t* dims, int channels,
                    uint64_t seed, int64_t z_begin, int64_t z_end) {
  int a, b[3] = {1, 1, 1};
  float maxdiag2 = 0.0f, diag;
  const int want_rank = config <= 2 ? 2 : 3;
  const int want_ch = config == 3 ? 1 : (config == 4 ? 4 : 3);
  if (config < 1 || config > 5 || rank != want_rank || channels != want_ch) return -1;
  s->rank = rank;
  s->channels = channels;
  s->config = config;
  s->seed = seed;
  for (a = 0; a < 3; ++a) s->dims[a] = a < rank ? dims[a] : 1;
  if (rank == 2) {
    z_begin = 0;
    z_end = 1;
  }
  if (z_begin < 0 || z_end > s->dims[2] || z_end <= z_begin) return -1;
  s->z_begin = z_begin;
  s->z_end = z_end;
  switch (config) {
    case 1: b[0] = 20; b[1] = 10; break;
    case 2: b[0] = 80; b[1] = 50; break;
    case 3: b[0] = b[1] = b[2] = 31; break;
    case 4: b[0] = b[1] = b[2] = 20; break;
    default:
      for (a = 0; a < 3; ++a) b[a] = (int)((s->dims[a] + 39) / 40);
  }
  for (a = 0; a < 3; ++a) {
    s->bins[a] = a < rank ? b[a] : 1;
    s->binsz[a] = (float)s->dims[a] / (float)s->bins[a];
    if (a < rank) maxdiag2 += s->binsz[a] * s->binsz[a];
  }
  /* A seed k bins away along axis a is >= (k-1)*binsz[a] away; the own seed
   * is <= the bin diagonal away, so reach = floor(diag / binsz) + 1 is exact. */
  diag = sqrtf(maxdiag2);
  for (a = 0; a < 3; ++a) s->reach[a] = a < rank ? (int)(diag / s->binsz[a]) + 1 : 0;
  return 0;
}

SYN_HD int64_t syn_bin_count(const SynthSpec* s) {
  return (int64_t)s->bins[0] * s->bins[1] * s->bins[2];
}

/* Seed position of bin `id` (one uniform seed per bin). */
SYN_HD SynthSeed syn_seed(const SynthSpec* s, int64_t id) {
  const int bx = (int)(id % s->bins[0]), by = (int)((id / s->bins[0]) % s->bins[1]);
  const int bz = (int)(id / ((int64_t)s->bins[0] * s->bins[1]));
  const uint64_t h = syn_hash3(s->seed, (uint64_t)id, 0x5EED);
  SynthSeed p;
  p.x = ((float)bx + syn_u01(h)) * s->binsz[0];
  p.y = ((float)by + syn_u01(h << 20)) * s->binsz[1];
  p.z = s->rank == 3 ? ((float)bz + syn_u01(h << 40)) * s->binsz[2] : 0.0f;
  p.w = 0.0f;
  return p;
}

/* Voxel li (local index within planes [z_begin, z_end)) into out (native
 * dtype, channels interleaved, `out` points at the slab's first voxel). */
SYN_HD void syn_voxel(const SynthSpec* s, const SynthSeed* table, int64_t li, void* out) {
  const int64_t plane = s->dims[0] * s->dims[1];
  const int64_t x = li % s->dims[0];
  const int64_t y = (li / s->dims[0]) % s->dims[1];
  const int64_t z = s->rank == 3 ? s->z_begin + li / plane : 0;
  const int64_t gidx = s->rank == 3 ? z * plane + y * s->dims[0] + x : y * s->dims[0] + x;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f, pz = (float)z + 0.5f;
  int bx = (int)(px / s->binsz[0]), by = (int)(py / s->binsz[1]);
  int bz = s->rank == 3 ? (int)(pz / s->binsz[2]) : 0;
  float d1 = 3.4e38f, d2 = 3.4e38f;
  uint64_t cell = 0, ch;
  int oz, oy, ox, c;
  const int rz = s->rank == 3 ? s->reach[2] : 0;
  if (bx > s->bins[0] - 1) bx = s->bins[0] - 1;
  if (by > s->bins[1] - 1) by = s->bins[1] - 1;
  if (bz > s->bins[2] - 1) bz = s->bins[2] - 1;
  for (oz = -rz; oz <= rz; ++oz) {
    const int cz = bz + oz;
    if (cz < 0 || cz >= s->bins[2]) continue;
    for (oy = -s->reach[1]; oy <= s->reach[1]; ++oy) {
      const int cy = by + oy;
      if (cy < 0 || cy >= s->bins[1]) continue;
      for (ox = -s->reach[0]; ox <= s->reach[0]; ++ox) {
        const int cx = bx + ox;
        if (cx < 0 || cx >= s->bins[0]) continue;
        {
          const int64_t bid = ((int64_t)cz * s->bins[1] + cy) * s->bins[0] + cx;
          const SynthSeed p = table[bid];
          const float dx = p.x - px, dy = p.y - py, dz = p.z - (s->rank == 3 ? pz : 0.0f);
          const float d = (dx * dx + dy * dy) + dz * dz;
          if (d < d1) {
            d2 = d1;
            d1 = d;
            cell = (uint64_t)bid;
          } else if (d < d2) {
            d2 = d;
          }
        }
      }
    }
  }
  ch = syn_hash3(s->seed, cell, 0xCE11);
  switch (s->config) {
    case 1: { /* 2D RGB u8, linear ramp + sigma 8, clamped */
      uint8_t* o = (uint8_t*)out + li * 3;
      const float ramp = 40.0f * (float)x / (float)s->dims[0] - 20.0f;
      for (c = 0; c < 3; ++c) {
        const float mean = 255.0f * syn_u01(syn_mix64(ch + (uint64_t)c));
        const float v = (mean + ramp) + 8.0f * syn_gauss(s->seed, (uint64_t)gidx, (uint64_t)c);
        o[c] = (uint8_t)syn_clamp(rintf(v), 0.0f, 255.0f);
      }
      break;
    }
    case 2: { /* 2D RGB f32, sinusoidal shading (amplitude 0.1) + sigma 0.03 */
      float* o = (float*)out + li * 3;
      const float shade = (0.1f * syn_sin(6.2831853f * (float)x / 512.0f)) *
                          syn_cos(6.2831853f * (float)y / 384.0f);
      for (c = 0; c < 3; ++c) {
        const float mean = syn_u01(syn_mix64(ch + (uint64_t)c));
        o[c] = (mean + shade) + 0.03f * syn_gauss(s->seed, (uint64_t)gidx, (uint64_t)c);
      }
      break;
    }
    case 3: { /* 3D u16, dark blurred membranes, Poisson-like noise */
      uint16_t* o = (uint16_t*)out + li;
      const float mean = 5000.0f + 55000.0f * syn_u01(ch);
      /* half-gap to the bisector ~ (sqrt(d2) - sqrt(d1)) / 2; 3-voxel blur */
      const float w = 0.5f * (sqrtf(d2) - sqrtf(d1));
      const float memb = syn_exp(-(w * w) / 4.5f);
      const float lvl = mean * (1.0f - 0.85f * memb);
      const float v = lvl + sqrtf(lvl) * syn_gauss(s->seed, (uint64_t)gidx, 0);
      *o = (uint16_t)syn_clamp(rintf(v), 0.0f, 65535.0f);
      break;
    }
    case 4: { /* 3D 4-channel f32, 30% of cells near zero in random channels */
      float* o = (float*)out + li * 4;
      const int dark = syn_u01(syn_mix64(ch ^ 0xDA7C)) < 0.3f;
      unsigned subset = (unsigned)(syn_mix64(ch ^ 0x5B5E7) & 0xF);
      if (dark && subset == 0) subset = 1u << (syn_mix64(ch ^ 0x1) & 3);
      for (c = 0; c < 4; ++c) {
        float mean = syn_u01(syn_mix64(ch + (uint64_t)c));
        if (dark && ((subset >> c) & 1)) mean = mean * 0.02f;
        o[c] = mean + 0.05f * syn_gauss(s->seed, (uint64_t)gidx, (uint64_t)c);
      }
      break;
    }
    default: { /* 5: 3D RGB u8, z-dependent drift + sigma 6 */
      uint8_t* o = (uint8_t*)out + li * 3;
      const float t = (float)z / (float)s->dims[2];
      float drift[3];
      drift[0] = 30.0f * t;
      drift[1] = -20.0f * t;
      drift[2] = 25.0f * syn_sin(3.14159265f * t);
      for (c = 0; c < 3; ++c) {
        const float mean = 20.0f + 215.0f * syn_u01(syn_mix64(ch + (uint64_t)c));
        const float v = (mean + drift[c]) + 6.0f * syn_gauss(s->seed, (uint64_t)gidx, (uint64_t)c);
        o[c] = (uint8_t)syn_clamp(rintf(v), 0.0f, 255.0f);
      }
      break;
    }
  }
}

#endif
