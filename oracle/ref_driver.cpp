// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// against /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libibref.so with the reference's own Release flags
// (-O3 -DNDEBUG -fopenmp, proj/CMakeLists.txt:6-15).  It is used to
//   * pin the C restatement (oracle/ib_oracle.c) against the real thing,
//   * generate tests/golden/ fixtures (tests/golden/make_golden.py),
//   * time the reference CPU path in bench.py (cpu_baseline / --impl reference).
// Nothing in the product library links it.
#include <array>
#include <cmath>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "ib/bench/setup.hpp"
#include "ib/bench/verify.hpp"
#include "ib/ib.hpp"

extern "C" {
typedef struct {
  int dim;
  int extent[3];
  double spacing;
  double staggering[3];
  int periodic[3];
  double origin[3];
} ref_grid;
}

namespace {

// Kernels beyond the reference's CosineKernel, written as the reference's
// tests write their own Kernel types (tests/grid_test.cpp:18-23) and with
// exactly the formulas of oracle/ib_oracle.c or_kernel_phi and the device.
struct Peskin4Kernel {  // Peskin 2002, Eq. 6.27
  double phi(double r) const {
    const double a = std::abs(r);
    if (!(a < 2.0)) return 0.0;
    if (a <= 1.0) return (3.0 - 2.0 * a + std::sqrt(1.0 + 4.0 * a - 4.0 * a * a)) * 0.125;
    return (5.0 - 2.0 * a - std::sqrt(std::fmax(0.0, -7.0 + 12.0 * a - 4.0 * a * a))) * 0.125;
  }
  int support() const { return 4; }
  double radius() const { return 2.0; }
};
struct Roma3Kernel {  // Roma, Peskin & Berger 1999
  double phi(double r) const {
    const double a = std::abs(r);
    if (!(a < 1.5)) return 0.0;
    if (a <= 0.5) return (1.0 + std::sqrt(1.0 - 3.0 * a * a)) / 3.0;
    return (5.0 - 3.0 * a - std::sqrt(1.0 - 3.0 * (1.0 - a) * (1.0 - a))) / 6.0;
  }
  int support() const { return 3; }
  double radius() const { return 1.5; }
};
struct Linear2Kernel {
  double phi(double r) const {
    const double a = std::abs(r);
    return a < 1.0 ? 1.0 - a : 0.0;
  }
  int support() const { return 2; }
  double radius() const { return 1.0; }
};

template <class F>
void with_kernel(int kernel, F&& f) {
  switch (kernel) {
    case 0: f(ib::CosineKernel{}); break;
    case 1: f(Peskin4Kernel{}); break;
    case 2: f(Roma3Kernel{}); break;
    case 3: f(Linear2Kernel{}); break;
    default: throw std::invalid_argument("kernel");
  }
}

template <std::size_t D>
ib::StaggeredGrid<D> make_grid(const ref_grid* g) {
  std::array<int, D> e;
  ib::Vec<D> alpha, origin;
  std::array<bool, D> periodic;
  for (std::size_t a = 0; a < D; ++a) {
    e[a] = g->extent[a];
    alpha[a] = g->staggering[a];
    origin[a] = g->origin[a];
    periodic[a] = g->periodic[a] != 0;
  }
  return ib::StaggeredGrid<D>(e, g->spacing, alpha, periodic, origin);
}

template <std::size_t D>
ib::PointSet<D> make_points(const double* p, std::size_t n) {
  ib::PointSet<D> pts(n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t a = 0; a < D; ++a) pts[i][a] = p[i * D + a];
  return pts;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::length_error&) {
    return 2;
  } catch (...) {
    return 3;
  }
}

template <std::size_t D, class K>
void spread_dk(const K& k, int algo, const ref_grid* gd, const double* pts, const double* vals,
               std::size_t n, int workers, int b, double* out, std::uint32_t* keys,
               std::uint32_t* perm, std::uint32_t* run_keys, std::size_t* q) {
  const auto g = make_grid<D>(gd);
  const auto points = make_points<D>(pts, n);
  std::span<const double> values(vals, n);
  ib::GridField<D> res(g);
  if (algo == 0) {
    res = ib::spread_serial(points, values, g, k);
  } else if (algo == 1 || algo == 2) {
    ib::SpreadWorkspace<D> ws(n, g, algo == 2 ? b : 0);
    res = algo == 1 ? ib::spread_fused(points, values, g, k, ws, workers)
                    : ib::spread_buffered(points, values, g, k, ws, workers);
    if (keys) std::memcpy(keys, ws.keys.data(), n * 4);
    if (perm) std::memcpy(perm, ws.perm.data(), n * 4);
    if (run_keys) std::memcpy(run_keys, ws.run_keys.data(), ws.run_count * 4);
    if (q) *q = ws.run_count;
  } else {
    res = ib::spread_buffered_otf(points, values, g, k, b, workers);
  }
  std::memcpy(out, res.values.data(), res.values.size() * sizeof(double));
}

template <std::size_t D>
void spread_d(int kernel, int algo, const ref_grid* gd, const double* pts, const double* vals,
              std::size_t n, int workers, int b, double* out, std::uint32_t* keys,
              std::uint32_t* perm, std::uint32_t* run_keys, std::size_t* q) {
  with_kernel(kernel, [&](const auto& k) {
    spread_dk<D>(k, algo, gd, pts, vals, n, workers, b, out, keys, perm, run_keys, q);
  });
}

template <std::size_t D>
void interp_d(int kernel, const ref_grid* gd, const double* field, const double* pts,
              std::size_t n, int workers, double* out) {
  const auto g = make_grid<D>(gd);
  ib::GridField<D> f(g);
  std::memcpy(f.values.data(), field, f.values.size() * sizeof(double));
  const auto points = make_points<D>(pts, n);
  with_kernel(kernel, [&](const auto& k) {
    const auto r = ib::interpolate(f, points, k, workers);
    std::memcpy(out, r.data(), n * sizeof(double));
  });
}

template <std::size_t D>
void cell_key_d(const ref_grid* gd, const double* pts, std::size_t n, std::uint32_t* keys) {
  const auto g = make_grid<D>(gd);
  for (std::size_t i = 0; i < n; ++i) {
    ib::Vec<D> x;
    for (std::size_t a = 0; a < D; ++a) x[a] = pts[i * D + a];
    keys[i] = ib::cell_key(ib::cell_index(ib::wrap_position(x, g), g, 4), g);
  }
}

template <std::size_t D>
void time_step_d(const ref_grid* gd, const double* x_star, const double* vals,
                 const double* x_n, const double* field, std::size_t n, int workers, int reps,
                 double* t_spread, double* t_interp) {
  using clock = std::chrono::steady_clock;
  const auto g = make_grid<D>(gd);
  const auto ps = make_points<D>(x_star, n);
  const auto pn = make_points<D>(x_n, n);
  std::span<const double> values(vals, n);
  ib::GridField<D> f(g);
  std::memcpy(f.values.data(), field, f.values.size() * sizeof(double));
  ib::SpreadWorkspace<D> ws(n, g);
  const ib::CosineKernel k;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = clock::now();
    auto out = ib::spread_fused(ps, values, g, k, ws, workers);
    const auto t1 = clock::now();
    auto e = ib::interpolate(f, pn, k, workers);
    const auto t2 = clock::now();
    t_spread[r] = std::chrono::duration<double>(t1 - t0).count();
    t_interp[r] = std::chrono::duration<double>(t2 - t1).count();
    (void)out;
    (void)e;
  }
}

}  // namespace

#define DISPATCH(dim, fn, ...)                      \
  switch (dim) {                                    \
    case 1: fn<1>(__VA_ARGS__); break;              \
    case 2: fn<2>(__VA_ARGS__); break;              \
    case 3: fn<3>(__VA_ARGS__); break;              \
    default: throw std::invalid_argument("dim");    \
  }

extern "C" {

int ref_spread_k(int kernel, int algo, const ref_grid* g, const double* pts, const double* vals,
                 size_t n, int workers, int sweep_width, double* out, uint32_t* keys,
                 uint32_t* perm, uint32_t* run_keys, size_t* q) {
  return guarded([&] {
    DISPATCH(g->dim, spread_d, kernel, algo, g, pts, vals, n, workers, sweep_width, out, keys,
                               perm, run_keys, q);
  });
}

int ref_spread(int algo, const ref_grid* g, const double* pts, const double* vals, size_t n,
               int workers, int sweep_width, double* out, uint32_t* keys, uint32_t* perm,
               uint32_t* run_keys, size_t* q) {
  return ref_spread_k(0, algo, g, pts, vals, n, workers, sweep_width, out, keys, perm, run_keys,
                      q);
}

int ref_interpolate_k(int kernel, const ref_grid* g, const double* field, const double* pts,
                      size_t n, int workers, double* out) {
  return guarded([&] { DISPATCH(g->dim, interp_d, kernel, g, field, pts, n, workers, out); });
}

int ref_interpolate(const ref_grid* g, const double* field, const double* pts, size_t n,
                    int workers, double* out) {
  return ref_interpolate_k(0, g, field, pts, n, workers, out);
}

int ref_cell_keys(const ref_grid* g, const double* pts, size_t n, uint32_t* keys) {
  return guarded([&] { DISPATCH(g->dim, cell_key_d, g, pts, n, keys); });
}

int ref_grid_check(const ref_grid* g) {
  return guarded([&] {
    switch (g->dim) {
      case 1: make_grid<1>(g); break;
      case 2: make_grid<2>(g); break;
      case 3: make_grid<3>(g); break;
      default: throw std::invalid_argument("dim");
    }
  });
}

void ref_key_value_sort(uint32_t* keys, uint32_t* payload, size_t n, int workers) {
  ib::key_value_sort<std::uint32_t>(std::span<ib::SortKey>(keys, n),
                                    std::span<std::uint32_t>(payload, n), workers);
}

size_t ref_segmented_reduce(const uint32_t* keys, const double* values, size_t n, int workers,
                            uint32_t* out_keys, double* out_sums) {
  return ib::segmented_reduce(std::span<const ib::SortKey>(keys, n),
                              std::span<const double>(values, n),
                              std::span<ib::SortKey>(out_keys, n), std::span<double>(out_sums, n),
                              workers);
}

void ref_scatter_points(uint64_t n, double edge, uint64_t seed, double* out) {
  const auto p = ib::bench::scatter_points(n, edge, seed);
  std::memcpy(out, p.data(), n * 3 * sizeof(double));
}

uint64_t ref_delta_evaluations(void) { return ib::stats::delta_evaluations(); }
void ref_reset_delta_evaluations(void) { ib::stats::reset_delta_evaluations(); }

int ref_time_step(const ref_grid* g, const double* x_star, const double* vals,
                  const double* x_n, const double* field, size_t n, int workers, int reps,
                  double* t_spread, double* t_interp) {
  return guarded([&] {
    DISPATCH(g->dim, time_step_d, g, x_star, vals, x_n, field, n, workers, reps, t_spread,
                                  t_interp);
  });
}

// Runs the reference's own verify suite (inc/bench/verify.hpp:396-407);
// returns the number of failing checks.
int ref_run_verification(uint64_t seed, int workers, int cases) {
  ib::bench::VerifyOptions opt;
  opt.seed = seed;
  opt.workers = workers;
  opt.coupling_cases = cases;
  opt.adjointness_instances = cases;
  opt.conservation_instances = cases;
  opt.primitive_cases = 200;
  int fails = 0;
  for (const auto& r : ib::bench::run_verification(opt)) fails += r.pass ? 0 : 1;
  return fails;
}

}  // extern "C"
