/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the SSLIC hot path (see
 * sslic_oracle.h). Every function cites the reference lines it restates.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, like
 * proj/CMakeLists.txt:18-20).
 */
#include "sslic_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int64_t pixel_count(int rank, const int64_t* dims) {
  int64_t n = 1;
  for (int a = 0; a < rank; ++a) n *= dims[a];
  return n;
}

static void strides_of(int rank, const int64_t* dims, int64_t* strides) {
  /* image.hpp:88-97 — stride[0] = 1, axis 0 fastest. */
  int64_t acc = 1;
  for (int a = 0; a < rank; ++a) {
    strides[a] = acc;
    acc *= dims[a];
  }
}

static void decode(int64_t off, int rank, const int64_t* dims, int64_t* coord) {
  /* image.hpp:127-136 */
  for (int a = 0; a < rank; ++a) {
    coord[a] = off % dims[a];
    off /= dims[a];
  }
}

static int64_t clamp64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

int64_t orc_cluster_count(int rank, const int64_t* dims, const int64_t* grid) {
  /* slic.hpp:212-216 */
  int64_t k = 1;
  for (int a = 0; a < rank; ++a) k *= (dims[a] + grid[a] - 1) / grid[a];
  return k;
}

void orc_init_centers(int rank, const int64_t* dims, int channels, const double* data,
                      const int64_t* grid, double* centers) {
  /* slic.hpp:206-230: cells enumerated row-major (axis 0 fastest), centre at
   * min(cell*S + S/2, d-1), intensity read there. */
  int64_t cells[4], strides[4], cell[4] = {0, 0, 0, 0};
  strides_of(rank, dims, strides);
  for (int a = 0; a < rank; ++a) cells[a] = (dims[a] + grid[a] - 1) / grid[a];
  const int64_t k = orc_cluster_count(rank, dims, grid);
  const int stride = channels + rank;
  for (int64_t id = 0; id < k; ++id) {
    int64_t off = 0, coord[4];
    for (int a = 0; a < rank; ++a) {
      coord[a] = cell[a] * grid[a] + grid[a] / 2;
      if (coord[a] > dims[a] - 1) coord[a] = dims[a] - 1;
      off += coord[a] * strides[a];
    }
    for (int c = 0; c < channels; ++c) centers[id * stride + c] = data[off * channels + c];
    for (int a = 0; a < rank; ++a) centers[id * stride + channels + a] = (double)coord[a];
    for (int a = 0; a < rank; ++a) {
      if (++cell[a] < cells[a]) break;
      cell[a] = 0;
    }
  }
}

double orc_gradient_sq(int rank, const int64_t* dims, int channels, const double* data,
                       const int64_t* coord) {
  /* color.hpp:71-102: axes in order, channels in order, h = 2 central,
   * h = 1 one-sided at borders, axes of extent 1 skipped. */
  int64_t strides[4];
  strides_of(rank, dims, strides);
  int64_t base = 0;
  for (int a = 0; a < rank; ++a) base += coord[a] * strides[a];
  double g = 0.0;
  for (int a = 0; a < rank; ++a) {
    if (dims[a] == 1) continue;
    int64_t lo = base, hi = base;
    double h = 2.0;
    if (coord[a] == 0) {
      hi += strides[a];
      h = 1.0;
    } else if (coord[a] == dims[a] - 1) {
      lo -= strides[a];
      h = 1.0;
    } else {
      hi += strides[a];
      lo -= strides[a];
    }
    for (int c = 0; c < channels; ++c) {
      const double d = (data[hi * channels + c] - data[lo * channels + c]) / h;
      g += d * d;
    }
  }
  return g;
}

void orc_perturb_centers(int rank, const int64_t* dims, int channels, const double* data,
                         double* centers, int64_t k) {
  /* slic.hpp:236-267: 3^n hood at llround(centre) clamped, row-major scan,
   * first strict minimum wins; centre := (I(best), best). */
  int64_t strides[4];
  strides_of(rank, dims, strides);
  const int stride = channels + rank;
  for (int64_t id = 0; id < k; ++id) {
    double* ctr = centers + id * stride;
    int64_t lo[4], hi[4], cur[4], best[4];
    for (int a = 0; a < rank; ++a) {
      const int64_t anchor = llround(ctr[channels + a]);
      lo[a] = clamp64(anchor - 1, 0, dims[a]);
      hi[a] = clamp64(anchor + 2, lo[a], dims[a]) - 1; /* clamp_region, image.hpp:158-167 */
      cur[a] = lo[a];
    }
    int first = 1;
    double best_g = 0.0;
    for (;;) {
      const double g = orc_gradient_sq(rank, dims, channels, data, cur);
      if (first || g < best_g) {
        first = 0;
        best_g = g;
        memcpy(best, cur, sizeof(best));
      }
      int a = 0;
      for (; a < rank; ++a) {
        if (++cur[a] <= hi[a]) break;
        cur[a] = lo[a];
      }
      if (a == rank) break;
    }
    int64_t off = 0;
    for (int a = 0; a < rank; ++a) off += best[a] * strides[a];
    for (int c = 0; c < channels; ++c) ctr[c] = data[off * channels + c];
    for (int a = 0; a < rank; ++a) ctr[channels + a] = (double)best[a];
  }
}

double orc_distance(const double* center, const double* pixel, const int64_t* coord,
                    int channels, int rank, const int64_t* grid, double m_sq) {
  /* slic.hpp:156-171 — fixed left-to-right order, no contraction. */
  double color = 0.0;
  for (int c = 0; c < channels; ++c) {
    const double d = center[c] - pixel[c];
    color += d * d;
  }
  double spatial = 0.0;
  for (int a = 0; a < rank; ++a) {
    const double d = (center[channels + a] - (double)coord[a]) / (double)grid[a];
    spatial += d * d;
  }
  return color + m_sq * spatial;
}

void orc_assign(int rank, const int64_t* dims, int channels, const double* data,
                const double* centers, int64_t k, const int64_t* grid, double weight_m,
                uint32_t* labels, double* dists) {
  /* slic.hpp:275-310: clusters in ascending id, window [llround(c)-S,
   * llround(c)+S] clamped (slic.hpp:175-184), strict < update. */
  int64_t strides[4];
  strides_of(rank, dims, strides);
  const int stride = channels + rank;
  const double m_sq = weight_m * weight_m;
  for (int64_t id = 0; id < k; ++id) {
    const double* ctr = centers + id * stride;
    int64_t lo[4], hi[4], cur[4];
    int empty = 0;
    for (int a = 0; a < rank; ++a) {
      const int64_t anchor = llround(ctr[channels + a]);
      lo[a] = clamp64(anchor - grid[a], 0, dims[a]);
      hi[a] = clamp64(anchor + grid[a] + 1, lo[a], dims[a]) - 1;
      if (hi[a] < lo[a]) empty = 1;
      cur[a] = lo[a];
    }
    if (empty) continue;
    for (;;) {
      int64_t off = 0;
      for (int a = 0; a < rank; ++a) off += cur[a] * strides[a];
      const double d = orc_distance(ctr, data + off * channels, cur, channels, rank, grid, m_sq);
      if (d < dists[off]) {
        dists[off] = d;
        labels[off] = (uint32_t)id;
      }
      int a = 0;
      for (; a < rank; ++a) {
        if (++cur[a] <= hi[a]) break;
        cur[a] = lo[a];
      }
      if (a == rank) break;
    }
  }
}

int orc_accumulate(int rank, const int64_t* dims, int channels, const double* data,
                   const uint32_t* labels, int64_t k, int64_t slab_rows, double* sums,
                   int64_t* counts) {
  /* accumulate_region (slic.hpp:315-346) per slab of `slab_rows` rows of the
   * last axis (decompose, parallel.hpp:31-44), each slab row-major from
   * zero, merged in slab order (ClusterAccumulatorMap::merge,
   * slic.hpp:133-143; run_slic slic.hpp:402-408). slab_rows <= 0 means one
   * whole-image pass (the test oracle, oracles.hpp:187-204). */
  const int stride = channels + rank;
  const int64_t n = pixel_count(rank, dims);
  const int64_t last = dims[rank - 1];
  const int64_t rows = slab_rows > 0 ? slab_rows : last;
  const int64_t plane = n / last;
  double* part = (double*)malloc(sizeof(double) * (size_t)(k * stride));
  memset(sums, 0, sizeof(double) * (size_t)(k * stride));
  memset(counts, 0, sizeof(int64_t) * (size_t)k);
  int status = 0;
  for (int64_t z0 = 0; z0 < last && status == 0; z0 += rows) {
    const int64_t z1 = z0 + rows < last ? z0 + rows : last;
    memset(part, 0, sizeof(double) * (size_t)(k * stride));
    int64_t cur[4] = {0, 0, 0, 0};
    cur[rank - 1] = z0;
    for (int64_t off = z0 * plane; off < z1 * plane; ++off) {
      const uint32_t l = labels[off];
      if (l == ORC_UNDEFINED) { status = -1; break; }
      if ((int64_t)l >= k) { status = -2; break; }
      double* s = part + (int64_t)l * stride;
      for (int c = 0; c < channels; ++c) s[c] += data[off * channels + c];
      for (int a = 0; a < rank; ++a) s[channels + a] += (double)cur[a];
      ++counts[l];
      for (int a = 0; a < rank; ++a) {
        if (++cur[a] < dims[a]) break;
        cur[a] = 0;
      }
    }
    for (int64_t i = 0; i < k * stride; ++i) sums[i] += part[i];
  }
  free(part);
  return status;
}

double orc_update(double* centers, int64_t k, int stride, const double* sums,
                  const int64_t* counts) {
  /* slic.hpp:359-371: mean per component, count 0 keeps the centre,
   * residual^2 accumulated in (k, i) order. */
  double residual_sq = 0.0;
  for (int64_t id = 0; id < k; ++id) {
    if (counts[id] == 0) continue;
    for (int i = 0; i < stride; ++i) {
      const double nv = sums[id * stride + i] / (double)counts[id];
      const double delta = nv - centers[id * stride + i];
      centers[id * stride + i] = nv;
      residual_sq += delta * delta;
    }
  }
  return sqrt(residual_sq);
}

int orc_run_slic(int rank, const int64_t* dims, int channels, const double* data,
                 const int64_t* grid, double weight_m, int max_iterations, int has_threshold,
                 double threshold, uint32_t* labels, double* centers, double* residuals,
                 int* iterations_done) {
  /* slic.hpp:52-64 validate, 384-415 driver. */
  if (rank < 1 || rank > 4 || channels < 1) return -3;
  for (int a = 0; a < rank; ++a)
    if (grid[a] < 1 || grid[a] > dims[a]) return -3;
  if (!(weight_m > 0.0) || max_iterations < 0) return -3;

  const int64_t n = pixel_count(rank, dims);
  const int64_t k = orc_cluster_count(rank, dims, grid);
  const int stride = channels + rank;
  const int iterations = max_iterations > 0 ? max_iterations : (rank <= 2 ? 10 : 5);

  orc_init_centers(rank, dims, channels, data, grid, centers);
  orc_perturb_centers(rank, dims, channels, data, centers, k);

  double* dists = (double*)malloc(sizeof(double) * (size_t)n);
  double* sums = (double*)malloc(sizeof(double) * (size_t)(k * stride));
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t i = 0; i < n; ++i) {
    dists[i] = INFINITY;
    labels[i] = ORC_UNDEFINED;
  }
  int status = 0, done = 0;
  for (int it = 0; it < iterations; ++it) {
    orc_assign(rank, dims, channels, data, centers, k, grid, weight_m, labels, dists);
    if (orc_accumulate(rank, dims, channels, data, labels, k, grid[rank - 1], sums, counts) != 0) {
      status = -1;
      break;
    }
    const double r = orc_update(centers, k, stride, sums, counts);
    residuals[done++] = r;
    if (has_threshold && r <= threshold) break;
  }
  if (iterations_done) *iterations_done = done;
  free(dists);
  free(sums);
  free(counts);
  return status;
}

/* ---------------------------------------------------------------------- */
/* Connectivity                                                            */
/* ---------------------------------------------------------------------- */

/* io.hpp:432-454: boundary = any face neighbour (either side, every axis)
 * with a different label. */
void orc_mask_label_contour(int rank, const int64_t* dims, int channels, const double* img,
                            const uint32_t* labels, double* out) {
  int64_t n = 1, stride[4];
  for (int a = 0; a < rank; ++a) {
    stride[a] = n;
    n *= dims[a];
  }
  for (int64_t off = 0; off < n; ++off) {
    int boundary = 0;
    int64_t rem = off;
    for (int a = 0; a < rank; ++a) {
      const int64_t c = rem % dims[a];
      rem /= dims[a];
      if (c > 0 && labels[off - stride[a]] != labels[off]) boundary = 1;
      if (c + 1 < dims[a] && labels[off + stride[a]] != labels[off]) boundary = 1;
    }
    for (int ch = 0; ch < channels; ++ch)
      out[off * channels + ch] = boundary ? 0.0 : img[off * channels + ch];
  }
}

/* color.hpp:21-24: IEC 61966-2-1 transfer function on [0, 1]. */
static double orc_linearize(double u) {
  return u <= 0.04045 ? u / 12.92 : pow((u + 0.055) / 1.055, 2.4);
}
/* color.hpp:27-31: CIE 1976 pivot, eps = 216/24389, kappa = 24389/27. */
static double orc_pivot(double t) {
  const double eps = 216.0 / 24389.0, kappa = 24389.0 / 27.0;
  return t > eps ? cbrt(t) : (kappa * t + 16.0) / 116.0;
}
/* color.hpp:36-52: sRGB (D65) -> linear -> XYZ (2 degree) -> Lab. */
void orc_srgb_to_lab(int64_t n, const double* rgb, double* lab) {
  for (int64_t i = 0; i < n; ++i) {
    const double r = orc_linearize(rgb[3 * i] / 255.0);
    const double g = orc_linearize(rgb[3 * i + 1] / 255.0);
    const double b = orc_linearize(rgb[3 * i + 2] / 255.0);
    const double x = 0.4124564 * r + 0.3575761 * g + 0.1804375 * b;
    const double y = 0.2126729 * r + 0.7151522 * g + 0.0721750 * b;
    const double z = 0.0193339 * r + 0.1191920 * g + 0.9503041 * b;
    const double fx = orc_pivot(x / 0.95047), fy = orc_pivot(y / 1.0), fz = orc_pivot(z / 1.08883);
    lab[3 * i] = 116.0 * fy - 16.0;
    lab[3 * i + 1] = 500.0 * (fx - fy);
    lab[3 * i + 2] = 200.0 * (fy - fz);
  }
}

int64_t orc_size_threshold(int rank, const int64_t* grid) {
  /* connectivity.hpp:34-38 */
  int64_t p = 1;
  for (int a = 0; a < rank; ++a) p *= grid[a];
  return p / 4;
}

typedef struct {
  int64_t* v;
  int64_t n, cap;
} vec64;

static void vpush(vec64* s, int64_t x) {
  if (s->n == s->cap) {
    s->cap = s->cap ? s->cap * 2 : 256;
    s->v = (int64_t*)realloc(s->v, sizeof(int64_t) * (size_t)s->cap);
  }
  s->v[s->n++] = x;
}

/* Face-connected component of `label` containing `seed` (the pixel set of
 * connectivity.hpp:46-99; the order of `out` is irrelevant to every caller).
 * visited is all-zero on entry and restored before returning. */
static void fill_component(const uint32_t* labels, int rank, const int64_t* dims,
                           const int64_t* strides, int64_t seed, uint32_t label,
                           uint8_t* visited, vec64* out, vec64* stack) {
  out->n = 0;
  stack->n = 0;
  vpush(stack, seed);
  visited[seed] = 1;
  int64_t coord[4];
  while (stack->n) {
    const int64_t off = stack->v[--stack->n];
    vpush(out, off);
    decode(off, rank, dims, coord);
    for (int a = 0; a < rank; ++a) {
      if (coord[a] > 0) {
        const int64_t nb = off - strides[a];
        if (!visited[nb] && labels[nb] == label) {
          visited[nb] = 1;
          vpush(stack, nb);
        }
      }
      if (coord[a] + 1 < dims[a]) {
        const int64_t nb = off + strides[a];
        if (!visited[nb] && labels[nb] == label) {
          visited[nb] = 1;
          vpush(stack, nb);
        }
      }
    }
  }
  for (int64_t i = 0; i < out->n; ++i) visited[out->v[i]] = 0;
}

void orc_finalize(int rank, const int64_t* dims, const uint32_t* labels, const double* centers,
                  int channels, int64_t k, const int64_t* grid, uint8_t* markers) {
  /* connectivity.hpp:125-173 */
  int64_t strides[4];
  strides_of(rank, dims, strides);
  const int64_t n = pixel_count(rank, dims);
  const int64_t min_size = orc_size_threshold(rank, grid);
  const int stride = channels + rank;
  uint8_t* visited = (uint8_t*)calloc((size_t)n, 1);
  vec64 comp = {0, 0, 0}, stack = {0, 0, 0};
  for (int64_t id = 0; id < k; ++id) {
    int64_t anchor[4];
    for (int a = 0; a < rank; ++a)
      anchor[a] = clamp64(llround(centers[id * stride + channels + a]), 0, dims[a] - 1);
    int64_t aoff = 0;
    for (int a = 0; a < rank; ++a) aoff += anchor[a] * strides[a];
    int64_t seed = -1;
    if (labels[aoff] == (uint32_t)id) {
      seed = aoff;
    } else {
      /* hood = clamp([anchor - S/2, anchor - S/2 + S)), row-major first hit */
      int64_t lo[4], hi[4], cur[4];
      int empty = 0;
      for (int a = 0; a < rank; ++a) {
        lo[a] = clamp64(anchor[a] - grid[a] / 2, 0, dims[a]);
        hi[a] = clamp64(anchor[a] - grid[a] / 2 + grid[a], lo[a], dims[a]) - 1;
        if (hi[a] < lo[a]) empty = 1;
        cur[a] = lo[a];
      }
      while (!empty) {
        int64_t off = 0;
        for (int a = 0; a < rank; ++a) off += cur[a] * strides[a];
        if (labels[off] == (uint32_t)id) {
          seed = off;
          break;
        }
        int a = 0;
        for (; a < rank; ++a) {
          if (++cur[a] <= hi[a]) break;
          cur[a] = lo[a];
        }
        if (a == rank) break;
      }
    }
    if (seed < 0) continue;
    fill_component(labels, rank, dims, strides, seed, (uint32_t)id, visited, &comp, &stack);
    if (comp.n > min_size)
      for (int64_t i = 0; i < comp.n; ++i) markers[comp.v[i]] = 1;
  }
  free(visited);
  free(comp.v);
  free(stack.v);
}

uint32_t orc_sweep(int rank, const int64_t* dims, uint32_t* labels, uint8_t* markers,
                   int64_t min_size, uint32_t k_start) {
  /* connectivity.hpp:182-261 */
  int64_t strides[4], coord[4];
  strides_of(rank, dims, strides);
  const int64_t n = pixel_count(rank, dims);
  uint8_t* visited = (uint8_t*)calloc((size_t)n, 1);
  vec64 comp = {0, 0, 0}, stack = {0, 0, 0};
  uint32_t next_label = k_start;
  for (int64_t off = 0; off < n; ++off) {
    if (markers[off]) continue;
    const uint32_t label = labels[off];
    fill_component(labels, rank, dims, strides, off, label, visited, &comp, &stack);
    if (comp.n > min_size) {
      for (int64_t i = 0; i < comp.n; ++i) {
        labels[comp.v[i]] = next_label;
        markers[comp.v[i]] = 1;
      }
      ++next_label;
      continue;
    }
    int64_t best_before = -1, best_after = -1, best_pending = -1;
    uint32_t label_before = 0, label_after = 0, label_pending = 0;
    for (int64_t i = 0; i < comp.n; ++i) {
      const int64_t o = comp.v[i];
      decode(o, rank, dims, coord);
      for (int a = 0; a < rank; ++a) {
        for (int dir = -1; dir <= 1; dir += 2) {
          const int64_t c = coord[a] + dir;
          if (c < 0 || c >= dims[a]) continue;
          const int64_t adj = o + dir * strides[a];
          if (labels[adj] == label) continue;
          if (markers[adj]) {
            if (adj < off) {
              if (adj > best_before) {
                best_before = adj;
                label_before = labels[adj];
              }
            } else if (best_after < 0 || adj < best_after) {
              best_after = adj;
              label_after = labels[adj];
            }
          } else if (best_pending < 0 || adj < best_pending) {
            best_pending = adj;
            label_pending = labels[adj];
          }
        }
      }
    }
    if (best_before >= 0 || best_after >= 0) {
      const uint32_t target = best_before >= 0 ? label_before : label_after;
      for (int64_t i = 0; i < comp.n; ++i) {
        labels[comp.v[i]] = target;
        markers[comp.v[i]] = 1;
      }
    } else if (best_pending >= 0) {
      for (int64_t i = 0; i < comp.n; ++i) labels[comp.v[i]] = label_pending;
    } else {
      for (int64_t i = 0; i < comp.n; ++i) {
        labels[comp.v[i]] = next_label;
        markers[comp.v[i]] = 1;
      }
      ++next_label;
    }
  }
  free(visited);
  free(comp.v);
  free(stack.v);
  return next_label;
}

uint32_t orc_enforce_connectivity(int rank, const int64_t* dims, const uint32_t* labels_in,
                                  const double* centers, int channels, int64_t k,
                                  const int64_t* grid, uint32_t* labels_out) {
  /* connectivity.hpp:265-273 */
  const int64_t n = pixel_count(rank, dims);
  memcpy(labels_out, labels_in, sizeof(uint32_t) * (size_t)n);
  uint8_t* markers = (uint8_t*)calloc((size_t)n, 1);
  orc_finalize(rank, dims, labels_out, centers, channels, k, grid, markers);
  const uint32_t next =
      orc_sweep(rank, dims, labels_out, markers, orc_size_threshold(rank, grid), (uint32_t)k);
  free(markers);
  return next;
}
