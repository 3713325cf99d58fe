// tools/shim_step.cpp -- the bench's end-to-end figure through the C++
// drop-in (include/ib_b200/ib/): one ib::spread_fused at X* and one
// ib::interpolate at X^n per step on config-2-shaped data in std::vector
// (pageable) buffers, the workspace observables (run_count) read every step,
// as a reference caller would.  With `concurrent`, the two calls run on two
// host threads (the reference's threading contract allows concurrent calls on
// disjoint outputs), so the spread's grid copy-out overlaps the
// interpolation's field copy-in.
//   shim_step N n reps [concurrent [heap]]   -> "step_s_median <s> min <s> ..."
//   heap = 1: glibc keeps large blocks on the heap (mallopt), see main().
#include <malloc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <thread>
#include <vector>

#include "ib_b200/ib.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::printf("usage: shim_step N n reps [concurrent]\n");
    return 2;
  }
  ibc_context* probe = nullptr;
  if (ibc_context_create(0, &probe) != IBC_OK) {
    std::printf("no CUDA device\n");
    return 77;
  }
  ibc_context_destroy(probe);
  // Caller-side tuning (glibc): keep large blocks on the heap instead of a
  // fresh mmap per allocation, so the 134 MB GridField each spread returns
  // (spread.hpp:180, by value) reuses pages instead of faulting them in
  // again -- the reference's own callers pay the same construction.
  if (argc > 5 && std::atoi(argv[5]) != 0) {
    mallopt(M_MMAP_THRESHOLD, 1 << 30);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
  }
  const int N = std::atoi(argv[1]);
  const std::size_t n = std::strtoull(argv[2], nullptr, 10);
  const int reps = std::atoi(argv[3]);
  const bool concurrent = argc > 4 && std::atoi(argv[4]) != 0;
  const double edge = 16e-4, h = edge / N;
  const ib::StaggeredGrid<3> g({N, N, N}, h, {0.5, 0.5, 0.0}, {true, true, true});
  // scatter_points (bench/setup.hpp:46-53): mt19937_64, (rng() >> 11) * 2^-53.
  auto unit = [](std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; };
  std::mt19937_64 r1(1), r3(3), r2(2), r4(4);
  ib::PointSet<3> xn(n), xs(n);
  for (auto& p : xn)
    for (auto& c : p) c = unit(r1) * edge;
  for (std::size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) xs[i][a] = xn[i][a] + (2.0 * unit(r3) - 1.0) * 0.1 * h;
  std::vector<double> G(n);
  for (auto& v : G) v = 2.0 * unit(r2) - 1.0;
  ib::GridField<3> e(g);
  for (auto& v : e.values) v = 2.0 * unit(r4) - 1.0;
  ib::SpreadWorkspace<3> ws(n, g);
  const ib::CosineKernel k;
  std::vector<double> t, ts, ti;
  double check = 0.0;
  for (int rep = 0; rep <= reps; ++rep) {
    const auto t0 = std::chrono::steady_clock::now();
    std::size_t q = 0;
    ib::LagrangianValues E;
    double ell_probe = 0.0;
    double t_s = 0.0, t_i = 0.0;
    auto spread = [&] {
      const auto a = std::chrono::steady_clock::now();
      const auto ell = ib::spread_fused(xs, std::span<const double>(G), g, k, ws, 8);
      q = ws.run_count;
      ell_probe = ell.values[ell.values.size() / 3];
      t_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
    };
    auto interp = [&] {
      const auto a = std::chrono::steady_clock::now();
      E = ib::interpolate(e, xn, k, 8);
      t_i = std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
    };
    if (concurrent) {
      std::thread ti(interp);
      spread();
      ti.join();
    } else {
      spread();
      interp();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (rep > 0) {
      t.push_back(std::chrono::duration<double>(t1 - t0).count());
      ts.push_back(t_s);
      ti.push_back(t_i);
    }
    check = ell_probe + E[n / 2] + static_cast<double>(q);
  }
  std::sort(t.begin(), t.end());
  std::sort(ts.begin(), ts.end());
  std::sort(ti.begin(), ti.end());
  std::printf("step_s_median %.9e min %.9e reps %d concurrent %d spread_s %.3e interp_s %.3e check %.17g\n",
              t[t.size() / 2], t[0], reps, concurrent ? 1 : 0, ts[ts.size() / 2], ti[ti.size() / 2],
              check);
  return 0;
}
