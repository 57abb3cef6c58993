// sRGB -> CIE-Lab on the GPU (color.hpp:21-66), SURVEY §8f item 2.
#pragma once

#include "common.cuh"

namespace sslic_b200 {

// Transfer-function table for 8-bit inputs: entry v is the reference's
// srgb_linearize(v / 255.0) evaluated on the host with the same libm pow
// (color.hpp:21-24), so for u8 images the linear values are the reference's
// bit for bit.
void srgb_linear_table(double* table256);

// Lab of npix interleaved RGB pixels (native dtype, values in [0, 255]) into
// out (3 doubles per pixel). fp64, no contraction (the reference builds with
// -ffp-contract=off); integral values use the table, others the device pow;
// cbrt is the device's (<= 1 ulp from the host libm), so Lab agrees with the
// reference to ~1e-13 (bitwise where the cube roots agree).
void srgb_to_lab_device(const void* img, int dtype, int64_t npix, const double* table,
                        double* out, cudaStream_t s);

// mask_label_contour (io.hpp:432-454) on the GPU: out (fp64, c per voxel)
// = 0 where any face neighbour has a different label, else the image value.
// Integer label comparisons and exact value copies: bitwise the reference.
void mask_label_contour_device(const Geom& g, const void* img, const uint32_t* labels,
                               double* out, cudaStream_t s);

}  // namespace sslic_b200
