// TEST INFRASTRUCTURE ONLY — C-ABI shim around the UNMODIFIED reference
// headers (/root/reference/proj/include/sslic/*.hpp, included read-only via
// -I by oracle/Makefile; nothing is copied). Built into
// oracle/_ref/libsslic_ref.so and used to (a) pin the C restatement in
// oracle/sslic_oracle.c, (b) generate tests/golden fixtures, and (c) time the
// reference's multi-threaded CPU path for bench.py's cpu_baseline /
// --impl reference arm. io.hpp / sslic.hpp are not included (libpng absent).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <vector>

#include "sslic/bench.hpp"
#include "sslic/color.hpp"
#include "sslic/connectivity.hpp"
#include "sslic/parallel.hpp"
#include "sslic/slic.hpp"
#include "support/oracles.hpp"

using namespace sslic;

namespace {

Shape make_shape(int rank, const int64_t* dims) {
  Shape s;
  for (int a = 0; a < rank; ++a) s.push_back(dims[a]);
  return s;
}

SlicParams make_params(int rank, const int64_t* grid, double m, int iters, int has_thr,
                       double thr) {
  SlicParams p;
  for (int a = 0; a < rank; ++a) p.grid.push_back(grid[a]);
  p.weight_m = m;
  p.max_iterations = iters;
  if (has_thr) p.residual_threshold = thr;
  return p;
}

// Status codes mirror include/sslic_b200.h.
int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::out_of_range&) {
    return -3;
  } catch (const std::logic_error&) {
    return -2;
  } catch (...) {
    return -9;
  }
}

}  // namespace

extern "C" {

int ref_run_slic(int rank, const int64_t* dims, int channels, const double* data,
                 const int64_t* grid, double m, int max_iterations, int has_thr, double thr,
                 int workers, uint32_t* labels_out, double* centers_out, double* residuals_out,
                 int* iters_out) {
  try {
    const Shape shape = make_shape(rank, dims);
    NDImage img(shape, channels,
                std::vector<double>(data, data + pixel_count(shape) * channels));
    const SlicParams params = make_params(rank, grid, m, max_iterations, has_thr, thr);
    const SlicResult r = run_slic(img, params, workers);
    std::memcpy(labels_out, r.labels.data().data(), sizeof(uint32_t) * r.labels.data().size());
    std::memcpy(centers_out, r.centers.data().data(), sizeof(double) * r.centers.data().size());
    for (size_t i = 0; i < r.residuals.size(); ++i) residuals_out[i] = r.residuals[i];
    *iters_out = static_cast<int>(r.residuals.size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_init_perturb(int rank, const int64_t* dims, int channels, const double* data,
                     const int64_t* grid, int perturb, double* centers_out) {
  try {
    const Shape shape = make_shape(rank, dims);
    NDImage img(shape, channels,
                std::vector<double>(data, data + pixel_count(shape) * channels));
    const SlicParams params = make_params(rank, grid, 10.0, 0, 0, 0.0);
    ClusterTable t = init_centers(img, params);
    if (perturb) t = perturb_centers(img, t, 1);
    std::memcpy(centers_out, t.data().data(), sizeof(double) * t.data().size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// One assign_labels pass over every slab of run_slic's decomposition, with
// caller-owned labels/dists (in-out).
int ref_assign_pass(int rank, const int64_t* dims, int channels, const double* data,
                    const int64_t* grid, double m, const double* centers, int64_t k,
                    uint32_t* labels, double* dists) {
  try {
    const Shape shape = make_shape(rank, dims);
    NDImage img(shape, channels,
                std::vector<double>(data, data + pixel_count(shape) * channels));
    const SlicParams params = make_params(rank, grid, m, 0, 0, 0.0);
    ClusterTable table(channels, rank, k);
    std::memcpy(table.data().data(), centers, sizeof(double) * table.data().size());
    LabelMap lm(shape);
    DistanceMap dm(shape);
    std::memcpy(lm.data().data(), labels, sizeof(uint32_t) * lm.data().size());
    std::memcpy(dm.data().data(), dists, sizeof(double) * dm.data().size());
    for (const ImageRegion& slab : decompose(shape, params.grid).slabs)
      assign_labels(img, table, params, lm, dm, slab);
    std::memcpy(labels, lm.data().data(), sizeof(uint32_t) * lm.data().size());
    std::memcpy(dists, dm.data().data(), sizeof(double) * dm.data().size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_enforce_connectivity(int rank, const int64_t* dims, const uint32_t* labels_in,
                             int channels, const double* centers, int64_t k,
                             const int64_t* grid, int workers, uint32_t* labels_out) {
  try {
    const Shape shape = make_shape(rank, dims);
    LabelMap lm(shape);
    std::memcpy(lm.data().data(), labels_in, sizeof(uint32_t) * lm.data().size());
    ClusterTable table(channels, rank, k);
    std::memcpy(table.data().data(), centers, sizeof(double) * table.data().size());
    const SlicParams params = make_params(rank, grid, 10.0, 0, 0, 0.0);
    const LabelMap out = enforce_connectivity(lm, table, params, workers);
    std::memcpy(labels_out, out.data().data(), sizeof(uint32_t) * out.data().size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// Scaling-report analysis (bench.hpp:41-262) on caller-given records: the
// fitted alpha and the CSV / markdown texts (written into buf, NUL-ended).
int ref_scaling_report(int n, const int* workers, const double* times, const int* conn,
                       double* alpha_out, double* speedups_out, double* eff_out, char* csv,
                       int64_t csv_cap, char* md, int64_t md_cap) {
  try {
    std::vector<TimingRecord> recs;
    for (int i = 0; i < n; ++i) recs.push_back(TimingRecord{workers[i], times[i], conn[i] != 0});
    const ScalingReport r = detail::make_report(recs);
    *alpha_out = r.alpha;
    for (int i = 0; i < n; ++i) {
      speedups_out[i] = r.speedups[i];
      eff_out[i] = r.efficiencies[i];
    }
    const std::string c = emit_scaling_csv(r), m = emit_scaling_markdown(r);
    if ((int64_t)c.size() >= csv_cap || (int64_t)m.size() >= md_cap) return -9;
    std::memcpy(csv, c.c_str(), c.size() + 1);
    std::memcpy(md, m.c_str(), m.size() + 1);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

double ref_amdahl_bound(double alpha, int p) { return amdahl_bound(alpha, p); }
double ref_amdahl_efficiency_bound(double alpha, int p) { return amdahl_efficiency_bound(alpha, p); }

// convert_image_to_lab (color.hpp:54-66) on an interleaved 3-channel image.
int ref_convert_to_lab(int rank, const int64_t* dims, const double* rgb, double* lab_out) {
  try {
    const Shape shape = make_shape(rank, dims);
    NDImage img(shape, 3, std::vector<double>(rgb, rgb + pixel_count(shape) * 3));
    const NDImage out = convert_image_to_lab(img);
    std::memcpy(lab_out, out.data().data(), sizeof(double) * out.data().size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// The test-suite randomized image generator (oracles.hpp:302-311) driven by
// mt19937_64, exactly as the reference's corpora draw it. State is kept in an
// opaque handle so a Python script can replay a corpus sequence.
void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }
uint64_t ref_rng_raw(void* rng) { return (*static_cast<std::mt19937_64*>(rng))(); }
int64_t ref_rng_uniform_int(void* rng, int64_t lo, int64_t hi) {
  return std::uniform_int_distribution<std::int64_t>(lo, hi)(*static_cast<std::mt19937_64*>(rng));
}
int ref_rng_uniform_int32(void* rng, int lo, int hi) {
  return std::uniform_int_distribution<int>(lo, hi)(*static_cast<std::mt19937_64*>(rng));
}
// random_image: draws dims then values; returns pixel count, fills dims.
// values_out must hold max_extent^rank * channels doubles.
int64_t ref_random_image(void* rng, int rank, int64_t max_extent, int channels, int64_t* dims_out,
                         double* values_out) {
  auto& g = *static_cast<std::mt19937_64*>(rng);
  const NDImage img = oracle::random_image(g, rank, max_extent, channels);
  for (int a = 0; a < rank; ++a) dims_out[a] = img.dims()[a];
  std::memcpy(values_out, img.data().data(), sizeof(double) * img.data().size());
  return img.pixel_count();
}
void ref_random_grid(void* rng, int rank, const int64_t* dims, int64_t* grid_out) {
  auto& g = *static_cast<std::mt19937_64*>(rng);
  const GridSize gs = oracle::random_grid(g, make_shape(rank, dims));
  for (int a = 0; a < rank; ++a) grid_out[a] = gs[a];
}
double ref_random_weight(void* rng) {
  return oracle::random_weight(*static_cast<std::mt19937_64*>(rng));
}

// Phase-split CPU timing of the metric scope: the public
// functions in run_slic's exact order (slic.hpp:388-412). Returns the wall
// seconds of each of `iterations` rounds of (assign | accumulate |
// reduce_and_update) into iter_seconds[i]; init/perturb time is written to
// *init_seconds. Labels/centres are returned
// so the caller can cross-check.
int ref_time_iterations(int rank, const int64_t* dims, int channels, const double* data,
                        const int64_t* grid, double m, int iterations, int workers,
                        double* init_seconds, double* iter_seconds, uint32_t* labels_out,
                        double* centers_out) {
  try {
    using clk = std::chrono::steady_clock;
    const Shape shape = make_shape(rank, dims);
    NDImage img(shape, channels,
                std::vector<double>(data, data + pixel_count(shape) * channels));
    const SlicParams params = make_params(rank, grid, m, iterations, 0, 0.0);
    auto t0 = clk::now();
    ClusterTable table = perturb_centers(img, init_centers(img, params), workers);
    LabelMap labels(shape);
    DistanceMap dists(shape);
    const SlabDecomposition decomp = decompose(shape, params.grid);
    auto t1 = clk::now();
    auto tprev = t1;
    for (int iter = 0; iter < iterations; ++iter) {
      parallel_for_slabs(decomp, workers, [&](std::int64_t, const ImageRegion& slab) {
        assign_labels(img, table, params, labels, dists, slab);
      });
      std::vector<ClusterAccumulatorMap> partials(decomp.slab_count(),
                                                  ClusterAccumulatorMap(table.stride()));
      parallel_for_slabs(decomp, workers, [&](std::int64_t i, const ImageRegion& slab) {
        partials[i] = accumulate_region(img, labels, slab);
      });
      table = reduce_and_update(table, partials).first;
      const auto tnow = clk::now();
      iter_seconds[iter] = std::chrono::duration<double>(tnow - tprev).count();
      tprev = tnow;
    }
    *init_seconds = std::chrono::duration<double>(t1 - t0).count();
    if (labels_out)
      std::memcpy(labels_out, labels.data().data(), sizeof(uint32_t) * labels.data().size());
    if (centers_out)
      std::memcpy(centers_out, table.data().data(), sizeof(double) * table.data().size());
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

}  // extern "C"
