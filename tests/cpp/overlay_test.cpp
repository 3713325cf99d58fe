// The reference's own callers, compiled UNMODIFIED against the drop-in
// overlay (include/ib_b200/ib/).  Built twice from this one source:
//  * tests/cpp/build/overlay_test   -I include/ib_b200 -I include -I <ref>/include
//    -> every "ib/<name>.hpp" resolves to the overlay: the B200 path;
//  * oracle/_ref/ref_overlay_test   -I <ref>/include only -> the reference's
//    CPU path (test infrastructure, the comparison target).
// The reference's headers ib/bench/run.hpp and ib/bench/verify.hpp (its step
// loop, run.hpp:59-128, and its oracle / invariant suite, verify.hpp:130-407)
// are the callers; nothing below re-implements them.
//
//   overlay_test verify [seed]                   -> run_verification, one line per check
//   overlay_test bench N n steps algo out.bin    -> run_benchmark, timings + final positions
//   overlay_test step N n reps                   -> scalar spread_fused + interpolate at
//                                                   config-2 shape with std::vector data
// Exit 0 = pass, 1 = a check failed, 77 = no CUDA device (overlay build).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ib/bench/run.hpp"
#include "ib/bench/setup.hpp"
#include "ib/bench/verify.hpp"
#include "ib/ib.hpp"

#ifdef IB_OVERLAY_DEVICE
static bool have_device() {
  ibc_context* c = nullptr;
  if (ibc_context_create(0, &c) != IBC_OK) return false;
  ibc_context_destroy(c);
  return true;
}
#else
static bool have_device() { return true; }
#endif

static int verify(std::uint64_t seed) {
  ib::bench::VerifyOptions opt;
  opt.seed = seed;
  int fails = 0;
  for (const auto& r : ib::bench::run_verification(opt)) {
    std::printf("%s %s %s\n", r.pass ? "PASS" : "FAIL", r.name.c_str(), r.detail.c_str());
    fails += r.pass ? 0 : 1;
  }
  return fails ? 1 : 0;
}

static int bench(int N, std::uint64_t n, int steps, const char* algo, const char* out) {
  ib::bench::BenchmarkConfig cfg;
  cfg.refinement = N;
  cfg.point_count = n;
  cfg.steps = steps;
  cfg.workers = 8;
  const std::string a(algo);
  cfg.algorithm = a == "serial" ? ib::SpreadAlgorithm::serial
                  : a == "buffered" ? ib::SpreadAlgorithm::buffered
                  : a == "otf" ? ib::SpreadAlgorithm::otf
                               : ib::SpreadAlgorithm::fused;
  const auto rep = ib::bench::run_benchmark(cfg);
  std::printf("interpolate mean_s %.9e calls %zu\n", rep.interpolate_timing.mean(),
              rep.interpolate_timing.calls());
  std::printf("spread mean_s %.9e calls %zu\n", rep.spread_timing.mean(), rep.spread_timing.calls());
  std::printf("fingerprint %016llx\n", static_cast<unsigned long long>(rep.physics_fingerprint));
  if (FILE* f = std::fopen(out, "wb")) {
    std::fwrite(rep.final_positions.data(), sizeof(ib::Vec<3>), rep.final_positions.size(), f);
    std::fclose(f);
  }
  return 0;
}

// The bench's scalar pair through the reference API: one
// spread_fused at X* and one interpolate at X^n per step, std::vector
// (pageable) buffers, the workspace observables read back every step.
static int step(int N, std::uint64_t n, int reps) {
  using clock = std::chrono::steady_clock;
  const double edge = 16e-4, h = edge / N;
  const ib::StaggeredGrid<3> g({N, N, N}, h, {0.5, 0.5, 0.0}, {true, true, true});
  const ib::PointSet<3> xn = ib::bench::scatter_points(n, edge, 1);
  ib::PointSet<3> xs = xn;
  const ib::PointSet<3> d = ib::bench::scatter_points(n, 0.2 * h, 3);
  for (std::size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) xs[i][a] += d[i][a] - 0.1 * h;
  std::vector<double> G(n);
  const ib::PointSet<3> gu = ib::bench::scatter_points(n / 3 + 1, 1.0, 2);
  for (std::size_t i = 0; i < n; ++i) G[i] = 2.0 * gu[i / 3][i % 3] - 1.0;
  ib::GridField<3> e(g);
  const ib::PointSet<3> eu = ib::bench::scatter_points(e.values.size() / 3 + 1, 1.0, 4);
  for (std::size_t k = 0; k < e.values.size(); ++k) e.values[k] = 2.0 * eu[k / 3][k % 3] - 1.0;
  ib::SpreadWorkspace<3> ws(n, g);
  const ib::CosineKernel k;
  std::vector<double> t(reps);
  double check = 0.0;
  for (int r = 0; r < reps + 1; ++r) {
    const auto t0 = clock::now();
    const auto ell = ib::spread_fused(xs, std::span<const double>(G), g, k, ws, 8);
    const std::size_t q = ws.run_count;
    const auto E = ib::interpolate(e, xn, k, 8);
    const auto t1 = clock::now();
    if (r > 0) t[r - 1] = std::chrono::duration<double>(t1 - t0).count();
    check = ell.values[12345 % ell.values.size()] + E[n / 2] + static_cast<double>(q);
  }
  std::sort(t.begin(), t.end());
  std::printf("step_s_median %.9e min %.9e reps %d check %.17g\n", t[t.size() / 2], t[0], reps,
              check);
  return 0;
}

int main(int argc, char** argv) {
  if (!have_device()) {
    std::printf("no CUDA device\n");
    return 77;
  }
  const std::string mode = argc > 1 ? argv[1] : "verify";
  try {
    if (mode == "verify") return verify(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
    if (mode == "bench" && argc > 6)
      return bench(std::atoi(argv[2]), std::strtoull(argv[3], nullptr, 10), std::atoi(argv[4]),
                   argv[5], argv[6]);
    if (mode == "step" && argc > 4)
      return step(std::atoi(argv[2]), std::strtoull(argv[3], nullptr, 10), std::atoi(argv[4]));
  } catch (const std::exception& ex) {
    std::printf("exception: %s\n", ex.what());
    return 1;
  }
  std::printf("usage: overlay_test verify [seed] | bench N n steps algo out.bin | step N n reps\n");
  return 2;
}
