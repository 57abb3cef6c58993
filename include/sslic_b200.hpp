// sslic_b200.hpp — C++ drop-in for users of the reference library.
//
// Include it AFTER the reference headers ("sslic/slic.hpp" and
// "sslic/connectivity.hpp"): it is written against the reference's own types
// (NDImage, SlicParams, ClusterTable, LabelMap, DistanceMap, SlicResult) and
// forwards to the C ABI in sslic_b200.h, so switching a caller from the CPU
// path to the B200 path is a namespace change:
//
//   sslic::SlicResult r = sslic::run_slic(img, params, workers);        // CPU
//   sslic::SlicResult r = sslic::b200::run_slic(img, params, workers);  // B200(s)
//
// (`workers` keeps its reference meaning and caps the GPU count; see
// run_slic below. run_slic_on_device picks one device explicitly.)
//
// Errors are rethrown as the reference's exception classes
// (std::invalid_argument / std::logic_error / std::out_of_range), CUDA
// failures as std::runtime_error. The fp64 NDImage is narrowed losslessly to
// uint8 / uint16 / float32 when every value is representable (so the fast
// fp32-filter kernel applies); otherwise it is passed as fp64. run_slic hands
// the NDImage's storage to the library, which narrows on the device; the
// small helpers (perturb_centers, assign_labels, ...) narrow on the host.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <cmath>
#include <vector>

#include "sslic_b200.h"

namespace sslic {
namespace b200 {

namespace detail {

inline void check(int status) {
  if (status == SSLIC_OK) return;
  const std::string msg = sslic_last_error();
  switch (status) {
    case SSLIC_EINVAL: throw std::invalid_argument(msg);
    case SSLIC_ELOGIC: throw std::logic_error(msg);
    case SSLIC_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error("sslic_b200: " + msg);
  }
}

// Native-dtype copy of an NDImage (image.hpp:236-285), narrowed losslessly.
struct NativeImage {
  sslic_image desc{};
  std::vector<unsigned char> bytes;
};

inline NativeImage narrow(const NDImage& img) {
  NativeImage out;
  const std::vector<double>& d = img.data();
  bool u8 = true, u16 = true, f32 = true;
  for (double v : d) {
    const bool integral = v == static_cast<double>(static_cast<int64_t>(v));
    u8 = u8 && integral && v >= 0.0 && v <= 255.0;
    u16 = u16 && integral && v >= 0.0 && v <= 65535.0;
    f32 = f32 && static_cast<double>(static_cast<float>(v)) == v;
    if (!u16 && !f32) break;
  }
  const int dtype = u8 ? SSLIC_U8 : (u16 ? SSLIC_U16 : (f32 ? SSLIC_F32 : SSLIC_F64));
  const size_t esz = dtype == SSLIC_U8 ? 1 : dtype == SSLIC_U16 ? 2 : dtype == SSLIC_F32 ? 4 : 8;
  out.bytes.resize(d.size() * esz);
  for (size_t i = 0; i < d.size(); ++i) {
    switch (dtype) {
      case SSLIC_U8: out.bytes[i] = static_cast<uint8_t>(d[i]); break;
      case SSLIC_U16: {
        const uint16_t v = static_cast<uint16_t>(d[i]);
        std::memcpy(&out.bytes[i * 2], &v, 2);
        break;
      }
      case SSLIC_F32: {
        const float v = static_cast<float>(d[i]);
        std::memcpy(&out.bytes[i * 4], &v, 4);
        break;
      }
      default: std::memcpy(&out.bytes[i * 8], &d[i], 8);
    }
  }
  out.desc.rank = img.rank();
  for (int a = 0; a < 4; ++a) out.desc.dims[a] = a < img.rank() ? img.dims()[a] : 1;
  out.desc.channels = img.channels();
  out.desc.dtype = dtype;
  out.desc.data = out.bytes.data();
  return out;
}

// The NDImage's own fp64 storage as an image descriptor (no copy).
inline NativeImage view_f64(const NDImage& img) {
  NativeImage out;
  out.desc.rank = img.rank();
  for (int a = 0; a < 4; ++a) out.desc.dims[a] = a < img.rank() ? img.dims()[a] : 1;
  out.desc.channels = img.channels();
  out.desc.dtype = SSLIC_F64;
  out.desc.data = img.data().data();
  return out;
}

inline sslic_params params_of(const SlicParams& p) {
  sslic_params c{};
  for (int a = 0; a < 4; ++a) c.grid[a] = a < p.grid.size() ? p.grid[a] : 1;
  c.weight_m = p.weight_m;
  c.max_iterations = p.max_iterations;
  c.enforce_connectivity = p.enforce_connectivity ? 1 : 0;
  c.has_residual_threshold = p.residual_threshold.has_value() ? 1 : 0;
  c.residual_threshold = p.residual_threshold.value_or(0.0);
  return c;
}

}  // namespace detail

/// run_slic (slic.hpp:384-415) on ONE given device.
inline SlicResult run_slic_on_device(const NDImage& img, const SlicParams& params, int device) {
  params.validate(img.dims());  // same exceptions as the reference, before any copy
  // the fp64 storage goes to the library as is: it narrows uint8 / uint16 /
  // float32 data losslessly on the device (no host pass over the volume)
  detail::NativeImage nimg = detail::view_f64(img);
  const sslic_params p = detail::params_of(params);
  const int iters = params.iterations_for(img.rank());
  std::vector<int64_t> dims(img.dims().begin(), img.dims().end());
  std::vector<int64_t> grid(params.grid.begin(), params.grid.end());
  ClusterTable table(img.channels(), img.rank(),
                     sslic_cluster_count(img.rank(), dims.data(), grid.data()));
  LabelMap labels(img.dims());
  std::vector<double> residuals(iters > 0 ? iters : 1);
  int done = 0;
  detail::check(sslic_run_slic(&nimg.desc, &p, device, labels.data().data(),
                               table.data().data(), residuals.data(), &done));
  residuals.resize(done);
  return SlicResult{std::move(labels), std::move(table), std::move(residuals)};
}

/// run_slic (slic.hpp:384-415) on B200s, same signature as the reference.
/// `workers` keeps its meaning -- the degree of parallelism, >= 1
/// (slic.hpp:386, same std::invalid_argument) -- and caps how many GPUs share
/// the work: a 3-D volume of at least 2^26 voxels is split into
/// min(workers, visible devices, planes) z-slabs, one per GPU, with one NCCL
/// allreduce of the per-cluster partials per iteration
/// (sslic_run_slic_multi); anything smaller runs on device 0. The result is
/// bitwise the same for any count, as the reference's is for any worker
/// count (parallel.hpp:1-8).
inline SlicResult run_slic(const NDImage& img, const SlicParams& params, int workers = 1) {
  params.validate(img.dims());
  if (workers < 1) throw std::invalid_argument("run_slic: workers must be >= 1");
  int n_dev = std::min(workers, sslic_device_count());
  const int64_t n = static_cast<int64_t>(img.pixel_count());
  if (img.rank() != 3 || n < (int64_t(1) << 26)) n_dev = 1;
  if (n_dev > 1) n_dev = static_cast<int>(std::min<int64_t>(n_dev, img.dims()[2]));
  if (n_dev <= 1) return run_slic_on_device(img, params, 0);
  detail::NativeImage nimg = detail::narrow(img);
  const sslic_params p = detail::params_of(params);
  const int iters = params.iterations_for(img.rank());
  std::vector<int64_t> dims(img.dims().begin(), img.dims().end());
  std::vector<int64_t> grid(params.grid.begin(), params.grid.end());
  ClusterTable table(img.channels(), img.rank(),
                     sslic_cluster_count(img.rank(), dims.data(), grid.data()));
  LabelMap labels(img.dims());
  std::vector<double> residuals(iters > 0 ? iters : 1);
  int done = 0;
  detail::check(sslic_run_slic_multi(&nimg.desc, &p, n_dev, nullptr, labels.data().data(),
                                     table.data().data(), residuals.data(), &done));
  residuals.resize(done);
  return SlicResult{std::move(labels), std::move(table), std::move(residuals)};
}

/// enforce_connectivity on ONE given device.
inline LabelMap enforce_connectivity_on_device(const LabelMap& labels, const ClusterTable& table,
                                               const SlicParams& params, int device) {
  std::vector<int64_t> dims(labels.dims().begin(), labels.dims().end());
  std::vector<int64_t> grid(params.grid.begin(), params.grid.end());
  LabelMap out(labels.dims());
  uint32_t next = 0;
  detail::check(sslic_enforce_connectivity(
      labels.rank(), dims.data(), labels.data().data(), table.data().data(), table.channels(),
      table.count(), grid.data(), device, out.data().data(), &next));
  return out;
}

/// enforce_connectivity (connectivity.hpp:265-273) on a B200, same signature:
/// `workers` is accepted for parity (the device pass does the work; the
/// result does not depend on it, as the reference's does not).
inline LabelMap enforce_connectivity(const LabelMap& labels, const ClusterTable& table,
                                     const SlicParams& params, int workers = 1) {
  (void)workers;
  return enforce_connectivity_on_device(labels, table, params, 0);
}

/// perturb_centers (slic.hpp:236-267) on a B200, same signature (`workers`
/// accepted for parity; device 0 does the work).
inline ClusterTable perturb_centers(const NDImage& img, ClusterTable table, int workers = 1) {
  (void)workers;
  detail::NativeImage nimg = detail::narrow(img);
  detail::check(sslic_perturb_centers(&nimg.desc, table.data().data(), table.count(), 0));
  return table;
}

/// One assign_labels pass over the whole image (slic.hpp:275-310), in place.
inline void assign_labels(const NDImage& img, const ClusterTable& table, const SlicParams& params,
                          LabelMap& labels, DistanceMap& dists, int device = 0) {
  detail::NativeImage nimg = detail::narrow(img);
  const sslic_params p = detail::params_of(params);
  detail::check(sslic_assign_pass(&nimg.desc, &p, table.data().data(), table.count(), device,
                                  labels.data().data(), dists.data().data()));
}

/// convert_image_to_lab (color.hpp:54-66) on a B200: fp64 Lab image, same
/// shape; std::invalid_argument unless 3 channels (the C ABI's SSLIC_EINVAL).
inline NDImage convert_image_to_lab(const NDImage& img, int device = 0) {
  detail::NativeImage nimg = detail::narrow(img);
  NDImage out = img;
  detail::check(sslic_convert_image_to_lab(&nimg.desc, device, out.data().data()));
  return out;
}

/// mask_label_contour (io.hpp:432-454) on a B200 (fp64 image out, same
/// shape); std::invalid_argument when the label dims differ.
inline NDImage mask_label_contour(const NDImage& img, const LabelMap& labels, int device = 0) {
  detail::NativeImage nimg = detail::narrow(img);
  const Shape& ld = labels.dims();
  std::vector<std::int64_t> dims(ld.begin(), ld.end());
  NDImage out = img;
  detail::check(sslic_mask_label_contour(&nimg.desc, (int)dims.size(), dims.data(),
                                         labels.data().data(), device, out.data().data()));
  return out;
}

/// read_volume (io.hpp:337-360) for the detached-header format (no PNG):
/// values widened to fp64 exactly as the reference does.
inline NDImage read_volume(const std::string& path) {
  sslic_volume_info info{};
  detail::check(sslic_volume_info_read(path.c_str(), &info));
  if (info.label_map)
    throw std::runtime_error("uint32 volumes are label maps; use read_labels");
  Shape dims;
  std::int64_t n = info.channels;
  for (int a = 0; a < info.rank; ++a) {
    dims.push_back(info.dims[a]);
    n *= info.dims[a];
  }
  const int es = info.dtype == SSLIC_U8 ? 1 : info.dtype == SSLIC_U16 ? 2 : 4;
  std::vector<unsigned char> raw(static_cast<std::size_t>(n * es));
  detail::check(sslic_volume_read(path.c_str(), 0, info.dims[info.rank - 1], raw.data(), -1));
  std::vector<double> v(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) {
    if (info.dtype == SSLIC_U8) v[i] = raw[i];
    else if (info.dtype == SSLIC_U16) v[i] = reinterpret_cast<const std::uint16_t*>(raw.data())[i];
    else v[i] = reinterpret_cast<const float*>(raw.data())[i];
  }
  return NDImage(dims, info.channels, std::move(v));
}

/// write_volume (io.hpp:362-392): "uint8" (rounded, clamped) or "float32".
inline void write_volume(const std::string& path, const NDImage& img,
                         const std::string& type = "float32") {
  const std::int64_t n = img.pixel_count() * img.channels();
  std::vector<unsigned char> raw;
  sslic_image d{};
  d.rank = img.rank();
  for (int a = 0; a < 4; ++a) d.dims[a] = a < img.rank() ? img.dims()[a] : 1;
  d.channels = img.channels();
  if (type == "uint8") {
    raw.resize(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i)
      raw[i] = static_cast<unsigned char>(std::clamp(std::llround(img.data()[i]), 0ll, 255ll));
    d.dtype = SSLIC_U8;
  } else if (type == "float32") {
    raw.resize(static_cast<std::size_t>(n) * 4);
    float* f = reinterpret_cast<float*>(raw.data());
    for (std::int64_t i = 0; i < n; ++i) f[i] = static_cast<float>(img.data()[i]);
    d.dtype = SSLIC_F32;
  } else {
    detail::check(SSLIC_EIO_TYPE);
  }
  d.data = raw.data();
  detail::check(sslic_volume_write(path.c_str(), &d));
}

}  // namespace b200
}  // namespace sslic
