// Drop-in test of include/ib_b200/ib.hpp: the reference's own call pattern
// (tests/coupling_test.cpp, inc/bench/run.hpp), with the reference header
// swapped for the B200 shim, checked against the C oracle (test
// infrastructure: oracle/ib_oracle.h).  Exit 0 = pass, 77 = no CUDA device.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "ib_b200/ib.hpp"
#include "ib_oracle.h"

static int failures = 0;
#define EXPECT(c)                                                \
  do {                                                           \
    if (!(c)) {                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                \
    }                                                            \
  } while (0)

static double max_rel_dev(const std::vector<double>& a, const std::vector<double>& b) {
  double dm = 0, rm = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    dm = std::max(dm, std::abs(a[i] - b[i]));
    rm = std::max(rm, std::abs(b[i]));
  }
  return rm > 0 ? dm / rm : dm;
}

template <std::size_t D>
static or_grid to_or(const ib::StaggeredGrid<D>& g) {
  const ibc_grid& c = g.c_grid();
  or_grid o{};
  o.dim = c.dim;
  o.spacing = c.spacing;
  for (int a = 0; a < 3; ++a) {
    o.extent[a] = c.extent[a];
    o.staggering[a] = c.staggering[a];
    o.periodic[a] = c.periodic[a];
    o.origin[a] = c.origin[a];
  }
  if (c.dim < 3) o.extent[2] = 1;
  if (c.dim < 2) o.extent[1] = 1;
  return o;
}

template <std::size_t D>
static void coupling_case(std::mt19937_64& rng, std::array<int, D> ext, std::array<bool, D> per,
                          std::size_t n) {
  std::uniform_real_distribution<double> u(0.0, 1.0);
  ib::Vec<D> alpha{};
  for (auto& a : alpha) a = u(rng) * 0.999;
  ib::StaggeredGrid<D> grid(ext, 0.5, alpha, per);
  ib::PointSet<D> pts(n);
  std::vector<double> vals(n);
  for (std::size_t i = 0; i < n; ++i) {
    for (std::size_t a = 0; a < D; ++a) {
      const double L = grid.axis_length(a);
      pts[i][a] = per[a] ? (3 * u(rng) - 1) * L : u(rng) * L;
    }
    vals[i] = 2 * u(rng) - 1;
  }
  ib::CosineKernel kern;
  ib::SpreadWorkspace<D> ws(n, grid);
  auto got = ib::spread_fused(pts, std::span<const double>(vals), grid, kern, ws, 8);
  const or_grid og = to_or(grid);
  std::vector<double> want(grid.point_count());
  std::vector<uint32_t> keys(n), perm(n), runs(n);
  size_t q = 0;
  or_spread_fused(&og, pts.front().data(), vals.data(), n, want.data(), keys.data(), perm.data(),
                  runs.data(), &q);
  EXPECT(ws.keys == keys);
  EXPECT(ws.perm == perm);
  EXPECT(ws.run_count == q);
  EXPECT(std::equal(runs.begin(), runs.begin() + q, ws.run_keys.begin()));
  EXPECT(max_rel_dev(got.values, want) <= 1e-12);
  auto serial = ib::spread_serial(pts, std::span<const double>(vals), grid, kern);
  EXPECT(serial.values == got.values);  // one device operator, deterministic
  ib::GridField<D> field(grid);
  for (auto& v : field.values) v = 2 * u(rng) - 1;
  auto e = ib::interpolate(field, pts, kern, 4);
  std::vector<double> ew(n);
  or_interpolate(&og, field.values.data(), pts.front().data(), n, ew.data());
  EXPECT(max_rel_dev(e, ew) <= 1e-12);
}

// run.hpp's MAC vector calls: spread_vector under every algorithm switch
// and interpolate_vector on the three component grids (setup.hpp:16-23).
static void mac_vector_case(std::mt19937_64& rng) {
  std::uniform_real_distribution<double> u(0.0, 1.0);
  const std::array<int, 3> ext = {16, 12, 10};
  const std::array<bool, 3> per = {true, true, true};
  std::array<ib::StaggeredGrid<3>, 3> grids = {
      ib::StaggeredGrid<3>(ext, 0.5, {0.0, 0.5, 0.5}, per),
      ib::StaggeredGrid<3>(ext, 0.5, {0.5, 0.0, 0.5}, per),
      ib::StaggeredGrid<3>(ext, 0.5, {0.5, 0.5, 0.0}, per)};
  const std::size_t n = 900;
  ib::PointSet<3> pts(n);
  std::array<ib::LagrangianValues, 3> force;
  for (auto& f : force) f.resize(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t a = 0; a < 3; ++a) {
      pts[i][a] = u(rng) * grids[0].axis_length(a);
      force[a][i] = 2 * u(rng) - 1;
    }
  ib::CosineKernel kern;
  ib::SpreadWorkspace<3> ws(n, grids[0], 2);
  std::array<std::vector<double>, 3> want;
  for (int c = 0; c < 3; ++c) {
    const or_grid og = to_or(grids[c]);
    want[c].resize(grids[c].point_count());
    or_spread_serial(&og, pts.front().data(), force[c].data(), n, want[c].data());
  }
  for (auto algo : {ib::SpreadAlgorithm::serial, ib::SpreadAlgorithm::fused,
                    ib::SpreadAlgorithm::buffered, ib::SpreadAlgorithm::otf}) {
    auto got = ib::spread_vector<3>(pts, force, std::span<const ib::StaggeredGrid<3>>(grids), kern,
                                    algo, 2, &ws, 8);
    for (int c = 0; c < 3; ++c) EXPECT(max_rel_dev(got[c].values, want[c]) <= 1e-12);
  }
  std::array<ib::GridField<3>, 3> u3 = {ib::GridField<3>(grids[0]), ib::GridField<3>(grids[1]),
                                        ib::GridField<3>(grids[2])};
  for (auto& f : u3)
    for (auto& v : f.values) v = 2 * u(rng) - 1;
  auto e = ib::interpolate_vector<3>(std::span<const ib::GridField<3>>(u3), pts, kern, 8);
  for (int c = 0; c < 3; ++c) {
    const or_grid og = to_or(grids[c]);
    std::vector<double> ew(n);
    or_interpolate(&og, u3[c].values.data(), pts.front().data(), n, ew.data());
    EXPECT(max_rel_dev(e[c], ew) <= 1e-12);
  }
}

int main() {
  try {
    (void)ib::b200::context();
  } catch (const std::exception& ex) {
    std::printf("no CUDA device (%s): skipped\n", ex.what());
    return 77;
  }
  std::mt19937_64 rng(20240611);
  coupling_case<3>(rng, {12, 10, 9}, {true, true, true}, 700);
  coupling_case<3>(rng, {9, 11, 8}, {false, true, false}, 500);
  coupling_case<2>(rng, {13, 7}, {true, false}, 300);
  coupling_case<1>(rng, {17}, {true}, 100);
  coupling_case<3>(rng, {32, 32, 32}, {true, true, true}, 20000);
  mac_vector_case(rng);

  // Reference exceptions (spread.hpp:60-77, grid.hpp:37-60).
  ib::StaggeredGrid<2> g({4, 4}, 1.0, {0.0, 0.0}, {false, false});
  ib::PointSet<2> p(3, ib::Vec<2>{1.0, 1.0});
  std::vector<double> v(2, 1.0);
  bool threw = false;
  try {
    ib::spread_serial(p, std::span<const double>(v), g, ib::CosineKernel{});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    ib::StaggeredGrid<3> big({2000, 2000, 2000}, 1.0, {0, 0, 0}, {true, true, true});
  } catch (const std::length_error&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    ib::SpreadWorkspace<2> ws(5, g);
    std::vector<double> v3(3, 1.0);
    ib::spread_fused(p, std::span<const double>(v3), g, ib::CosineKernel{}, ws, 1);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  // Operation counts (stats.hpp): n * 4^d per operation.
  ib::stats::reset_delta_evaluations();
  ib::interpolate(ib::GridField<2>(g), p, ib::CosineKernel{}, 1);
  EXPECT(ib::stats::delta_evaluations() == 3u * 16u);
  if (failures) {
    std::printf("shim test: %d failure(s)\n", failures);
    return 1;
  }
  std::printf("shim ok\n");
  return 0;
}
