// TEST INFRASTRUCTURE ONLY — drives include/sslic_b200.hpp (the C++ drop-in
// over the C ABI) side by side with the UNMODIFIED reference headers and
// checks that a caller switching sslic::run_slic -> sslic::b200::run_slic and
// sslic::enforce_connectivity -> sslic::b200::enforce_connectivity gets
// bit-identical results. Built by oracle/Makefile into oracle/_ref/ (it needs
// /root/reference at build time); run by tests/test_gpu_adapter.py.
#include <cstdio>
#include <random>

#include <algorithm>
#include <cmath>

#include "sslic/color.hpp"
#include "sslic/connectivity.hpp"
#include "sslic/slic.hpp"
#include "support/oracles.hpp"
#include "sslic_b200.hpp"

int main() {
  std::mt19937_64 rng(0x55110C);
  int failures = 0, cases = 0;
  for (int i = 0; i < 40; ++i) {
    const int rank = std::uniform_int_distribution<int>(1, 3)(rng);
    const int channels = rng() % 2 == 0 ? 1 : 3;
    sslic::NDImage img = oracle::random_image(rng, rank, 24, channels);
    if (i % 2 == 1)  // integer-valued images exercise the u8 narrowing / fast path
      for (double& v : img.data()) v = static_cast<double>(static_cast<int>(v));
    sslic::SlicParams params;
    params.grid = oracle::random_grid(rng, img.dims());
    params.weight_m = oracle::random_weight(rng);
    const sslic::SlicResult cpu = sslic::run_slic(img, params, 2);
    const sslic::SlicResult gpu = sslic::b200::run_slic(img, params, 2);  // namespace switch only
    const sslic::LabelMap cc_cpu = sslic::enforce_connectivity(cpu.labels, cpu.centers, params, 2);
    const sslic::LabelMap cc_gpu = sslic::b200::enforce_connectivity(gpu.labels, gpu.centers, params, 2);
    const bool ok = cpu.labels == gpu.labels && cpu.centers == gpu.centers && cc_cpu == cc_gpu &&
                    cpu.residuals.size() == gpu.residuals.size();
    if (!ok) {
      std::printf("case %d differs (rank %d, channels %d)\n", i, rank, channels);
      ++failures;
    }
    ++cases;
  }
  // convert_image_to_lab: same shape, Lab within 1e-12 (the two cube roots
  // are each within 1 ulp), invalid_argument for a non-RGB image
  {
    sslic::NDImage rgb = oracle::random_image(rng, 2, 24, 3);
    for (double& v : rgb.data()) v = static_cast<double>(static_cast<int>(v * 255.0 / 256.0));
    const sslic::NDImage a = sslic::convert_image_to_lab(rgb);
    const sslic::NDImage b = sslic::b200::convert_image_to_lab(rgb);
    double worst = 0.0;
    for (std::size_t j = 0; j < a.data().size(); ++j)
      worst = std::max(worst, std::abs(a.data()[j] - b.data()[j]));
    if (!(a.dims() == b.dims()) || !(worst < 1e-12)) {
      std::printf("convert_image_to_lab differs (max %.3g)\n", worst);
      ++failures;
    }
    ++cases;
    try {
      sslic::b200::convert_image_to_lab(sslic::NDImage::zeros(sslic::Shape{2, 2}, 1));
      ++failures;
    } catch (const std::invalid_argument&) {
    }
  }
  // mask_label_contour (io.hpp is not buildable here: no libpng), checked
  // against a direct restatement of its rule on a SLIC label map
  {
    sslic::NDImage img = oracle::random_image(rng, 2, 24, 3);
    sslic::SlicParams params;
    params.grid = oracle::random_grid(rng, img.dims());
    const sslic::SlicResult r = sslic::run_slic(img, params, 2);
    const sslic::NDImage m = sslic::b200::mask_label_contour(img, r.labels);
    const sslic::Shape& d = img.dims();
    bool ok = true;
    for (std::int64_t y = 0; y < d[1]; ++y)
      for (std::int64_t x = 0; x < d[0]; ++x) {
        const std::int64_t o = x + y * d[0];
        const std::uint32_t l = r.labels[o];
        const bool b = (x > 0 && r.labels[o - 1] != l) || (x + 1 < d[0] && r.labels[o + 1] != l) ||
                       (y > 0 && r.labels[o - d[0]] != l) ||
                       (y + 1 < d[1] && r.labels[o + d[0]] != l);
        for (int c = 0; c < 3; ++c)
          ok = ok && m.data()[3 * o + c] == (b ? 0.0 : img.data()[3 * o + c]);
      }
    if (!ok) {
      std::printf("mask_label_contour differs\n");
      ++failures;
    }
    ++cases;
  }
  // exceptions keep the reference's classes
  try {
    sslic::SlicParams bad;
    bad.grid = sslic::GridSize{9, 8};
    sslic::b200::run_slic(sslic::NDImage::zeros(sslic::Shape{8, 8}, 1), bad);
    ++failures;
  } catch (const std::invalid_argument&) {
  }
  try {  // workers keeps its meaning: >= 1 (slic.hpp:386)
    sslic::SlicParams ok;
    ok.grid = sslic::GridSize{4, 4};
    sslic::b200::run_slic(sslic::NDImage::zeros(sslic::Shape{8, 8}, 1), ok, 0);
    ++failures;
  } catch (const std::invalid_argument&) {
  }
  std::printf("adapter: %d cases, %d failures\n", cases, failures);
  return failures ? 1 : 0;
}
