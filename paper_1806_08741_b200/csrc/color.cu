// sRGB -> CIE-Lab (color.hpp:21-66): one thread per pixel, grid-stride.
#include <cmath>

#include "color.cuh"

namespace sslic_b200 {

void srgb_linear_table(double* t) {
  for (int v = 0; v < 256; ++v) {
    const double u = v / 255.0;
    t[v] = u <= 0.04045 ? u / 12.92 : std::pow((u + 0.055) / 1.055, 2.4);
  }
}

namespace {

// integral inputs in [0, 255] (every u8 image, and 8-bit data stored as
// f32/f64) take the host-computed table: bitwise the reference's values
__device__ __forceinline__ double linearize(double v, const double* table) {
  if (v >= 0.0 && v <= 255.0 && v == floor(v)) return table[(int)v];
  const double u = __ddiv_rn(v, 255.0);
  return u <= 0.04045 ? __ddiv_rn(u, 12.92) : pow(__ddiv_rn(__dadd_rn(u, 0.055), 1.055), 2.4);
}

// CIE 1976 pivot (color.hpp:27-31)
__device__ __forceinline__ double pivot(double t) {
  const double eps = 216.0 / 24389.0, kappa = 24389.0 / 27.0;
  return t > eps ? cbrt(t) : __ddiv_rn(__dadd_rn(__dmul_rn(kappa, t), 16.0), 116.0);
}

// ((a r + b g) + c b) in the reference's left-to-right order, no FMA
__device__ __forceinline__ double row(double a, double b, double c, double r, double g,
                                      double bl) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a, r), __dmul_rn(b, g)), __dmul_rn(c, bl));
}

__global__ void k_srgb_to_lab(const void* img, int dtype, int64_t npix, const double* table,
                              double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = linearize(load_value(img, dtype, 3 * i), table);
    const double g = linearize(load_value(img, dtype, 3 * i + 1), table);
    const double b = linearize(load_value(img, dtype, 3 * i + 2), table);
    const double x = row(0.4124564, 0.3575761, 0.1804375, r, g, b);
    const double y = row(0.2126729, 0.7151522, 0.0721750, r, g, b);
    const double z = row(0.0193339, 0.1191920, 0.9503041, r, g, b);
    const double fx = pivot(__ddiv_rn(x, 0.95047));
    const double fy = pivot(__ddiv_rn(y, 1.0));
    const double fz = pivot(__ddiv_rn(z, 1.08883));
    out[3 * i] = __dsub_rn(__dmul_rn(116.0, fy), 16.0);
    out[3 * i + 1] = __dmul_rn(500.0, __dsub_rn(fx, fy));
    out[3 * i + 2] = __dmul_rn(200.0, __dsub_rn(fy, fz));
  }
}

// one thread per voxel; coordinates decoded once, neighbours by stride
__global__ void k_mask_label_contour(Geom g, const void* img, const uint32_t* labels,
                                     double* out, int64_t n) {
  for (int64_t off = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; off < n;
       off += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t l = labels[off];
    bool boundary = false;
    int64_t rem = off;
    for (int a = 0; a < g.rank; ++a) {
      const int64_t c = rem % g.dims[a];
      rem /= g.dims[a];
      if (c > 0 && labels[off - g.strides[a]] != l) boundary = true;
      if (c + 1 < g.dims[a] && labels[off + g.strides[a]] != l) boundary = true;
    }
    for (int ch = 0; ch < g.channels; ++ch)
      out[off * g.channels + ch] = boundary ? 0.0 : load_value(img, g.dtype, off * g.channels + ch);
  }
}

}  // namespace

void mask_label_contour_device(const Geom& g, const void* img, const uint32_t* labels,
                               double* out, cudaStream_t s) {
  int64_t n = 1;
  for (int a = 0; a < g.rank; ++a) n *= g.dims[a];
  if (n <= 0) return;
  const int64_t blocks = (n + 255) / 256;
  k_mask_label_contour<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
      g, img, labels, out, n);
}

void srgb_to_lab_device(const void* img, int dtype, int64_t npix, const double* table,
                        double* out, cudaStream_t s) {
  if (npix <= 0) return;
  const int64_t blocks = (npix + 255) / 256;
  k_srgb_to_lab<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
      img, dtype, npix, table, out);
}

}  // namespace sslic_b200
