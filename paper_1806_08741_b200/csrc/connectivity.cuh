// enforce_connectivity (connectivity.hpp:265-273) on the device.
#pragma once

#include "common.cuh"

namespace sslic_b200 {

// labels_in/out: device, N = prod dims (whole image: slab == image).
// centers: device table (k x stride). Returns the next unused label.
// Optional by-products of the final relabel pass (the output files of
// tools/sslic.cpp:104-109,121-125 without another pass over the map):
// max_label: device scalar, atomicMax of the output labels (write_labels'
// "label count", io.hpp:396-412; zero it first); boundary: device bitmask,
// bit i set when voxel i has a face neighbour with a different OUTPUT label
// (mask_label_contour, io.hpp:432-454), ceil(n/32) words, zeroed first.
struct LabelOutputs {
  unsigned* max_label = nullptr;
  uint32_t* boundary = nullptr;
};

uint32_t enforce_connectivity_device(const Geom& g, const uint32_t* labels_in,
                                     const double* centers, uint32_t* labels_out,
                                     cudaStream_t stream, LabelOutputs outs = {});

// The same by-products for a final label map (no connectivity pass).
void label_outputs_device(const Geom& g, const uint32_t* labels, LabelOutputs outs,
                          cudaStream_t stream);

}  // namespace sslic_b200
