// enforce_connectivity (connectivity.hpp:265-273) on the device.
#pragma once

#include "common.cuh"

namespace sslic_b200 {

// labels_in/out: device, N = prod dims (whole image: slab == image).
// centers: device table (k x stride). Returns the next unused label.
uint32_t enforce_connectivity_device(const Geom& g, const uint32_t* labels_in,
                                     const double* centers, uint32_t* labels_out,
                                     cudaStream_t stream);

}  // namespace sslic_b200
