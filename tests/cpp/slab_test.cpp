// Multi-rank caller of the C ABI's z-slab path: R ranks, each a
// host thread with its own ibc_context (one process, one device here; across
// processes the same calls take ibc_ipc_* peer pointers), spread their homed
// points into their local slabs, run the peer-memory ghost-plane sum, fill
// their halos and interpolate -- checked against the single-grid device
// operators on the whole grid (<= 1e-12) for periodic and closed global axes.
//   slab_test  -> exit 0 pass, 1 fail, 77 no CUDA device
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "ibcuda.h"

static int failures = 0;
#define CHECK(x)                                                                  \
  do {                                                                            \
    ibc_status s_ = (x);                                                          \
    if (s_ != IBC_OK) {                                                           \
      std::fprintf(stderr, "FAIL %s:%d: %s -> %d %s\n", __FILE__, __LINE__, #x, s_, \
                   ibc_last_error());                                             \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double d = 0, m = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    d = std::max(d, std::abs(a[i] - b[i]));
    m = std::max(m, std::abs(b[i]));
  }
  return m > 0 ? d / m : d;
}

struct Rank {
  ibc_context* ctx = nullptr;
  cudaStream_t stream = nullptr;  // ranks must not share a stream: their handshakes wait on each other
  int z0 = 0, z1 = 0;
  double* d_spread = nullptr;  // local slab: spread output
  double* d_field = nullptr;   // local slab: interpolation input
  uint64_t* d_sig = nullptr;
  std::vector<double> pts, vals;
  std::vector<size_t> idx;  // global index of each local point
  double* d_pts = nullptr;
  double* d_vals = nullptr;
  double* d_E = nullptr;
};

static void run_case(int R, bool periodic) {
  const int nx = 32, ny = 24, nzr = 8, nz = R * nzr;
  const double h = 0.25;
  ibc_grid G{};
  G.dim = 3;
  G.extent[0] = nx; G.extent[1] = ny; G.extent[2] = nz;
  G.spacing = h;
  G.staggering[0] = 0.5; G.staggering[1] = 0.5; G.staggering[2] = 0.0;
  G.periodic[0] = G.periodic[1] = 1;
  G.periodic[2] = periodic ? 1 : 0;
  const size_t plane = (size_t)nx * ny, npts_grid = plane * nz;
  const size_t n = 6000;
  std::mt19937_64 rng(11 + R + (periodic ? 100 : 0));
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::vector<double> X(3 * n), V(n), F(npts_grid);
  for (size_t i = 0; i < n; ++i) {
    X[3 * i] = u(rng) * nx * h;
    X[3 * i + 1] = u(rng) * ny * h;
    // closed axis: keep every home cell (and support) inside [0, nz)
    X[3 * i + 2] = periodic ? (3 * u(rng) - 1) * nz * h : (2.0 + u(rng) * (nz - 4)) * h;
    V[i] = 2 * u(rng) - 1;
  }
  for (auto& f : F) f = 2 * u(rng) - 1;

  // Whole-grid reference on the device, and every point's home plane.
  ibc_context* c0 = nullptr;
  CHECK(ibc_context_create(0, &c0));
  double *dX, *dV, *dOut, *dF, *dE;
  int32_t* dPlanes;
  cudaMalloc(&dX, 24 * n); cudaMalloc(&dV, 8 * n); cudaMalloc(&dOut, 8 * npts_grid);
  cudaMalloc(&dF, 8 * npts_grid); cudaMalloc(&dE, 8 * n); cudaMalloc(&dPlanes, 4 * n);
  cudaMemcpy(dX, X.data(), 24 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dF, F.data(), 8 * npts_grid, cudaMemcpyHostToDevice);
  CHECK(ibc_spread_device(c0, &G, IBC_KERNEL_COSINE4, dX, dV, n, nullptr, dOut));
  CHECK(ibc_interpolate_device(c0, &G, IBC_KERNEL_COSINE4, dF, dX, n, dE));
  CHECK(ibc_home_planes_device(c0, &G, IBC_KERNEL_COSINE4, dX, n, dPlanes));
  CHECK(ibc_context_synchronize(c0));
  std::vector<double> want(npts_grid), wantE(n);
  std::vector<int32_t> planes(n);
  cudaMemcpy(want.data(), dOut, 8 * npts_grid, cudaMemcpyDeviceToHost);
  cudaMemcpy(wantE.data(), dE, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(planes.data(), dPlanes, 4 * n, cudaMemcpyDeviceToHost);

  // Ranks: slabs, homed points, local buffers, links.
  std::vector<Rank> rk(R);
  for (int r = 0; r < R; ++r) {
    Rank& k = rk[r];
    CHECK(ibc_context_create(0, &k.ctx));
    cudaStreamCreateWithFlags(&k.stream, cudaStreamNonBlocking);
    CHECK(ibc_context_set_stream(k.ctx, k.stream));
    k.z0 = r * nzr;
    k.z1 = k.z0 + nzr;
    for (size_t i = 0; i < n; ++i)
      if (planes[i] >= k.z0 && planes[i] < k.z1) {
        k.idx.push_back(i);
        k.pts.insert(k.pts.end(), &X[3 * i], &X[3 * i + 3]);
        k.vals.push_back(V[i]);
      }
    const size_t loc = plane * (nzr + 3), m = k.idx.size();
    CHECK(ibc_device_alloc(k.ctx, 8 * loc, (void**)&k.d_spread));
    CHECK(ibc_device_alloc(k.ctx, 8 * loc, (void**)&k.d_field));
    CHECK(ibc_slab_signals_create(k.ctx, &k.d_sig));
    cudaMalloc(&k.d_pts, 24 * m + 8); cudaMalloc(&k.d_vals, 8 * m + 8); cudaMalloc(&k.d_E, 8 * m + 8);
    cudaMemcpy(k.d_pts, k.pts.data(), 24 * m, cudaMemcpyHostToDevice);
    cudaMemcpy(k.d_vals, k.vals.data(), 8 * m, cudaMemcpyHostToDevice);
    // The field's owned planes in local layout (planes 2 .. nzr + 1).
    cudaMemcpy(k.d_field + 2 * plane, F.data() + (size_t)k.z0 * plane, 8 * plane * nzr,
               cudaMemcpyHostToDevice);
  }
  auto link_of = [&](int r, bool field) {
    ibc_slab_link L{};
    const int dn = (r + R - 1) % R, up = (r + 1) % R;
    L.nloc = nzr;
    L.nloc_down = nzr;
    L.plane = plane;
    L.has_down = periodic || r > 0;
    L.has_up = periodic || r < R - 1;
    L.d_local = field ? rk[r].d_field : rk[r].d_spread;
    L.d_down = field ? rk[dn].d_field : rk[dn].d_spread;
    L.d_up = field ? rk[up].d_field : rk[up].d_spread;
    L.d_sig = rk[r].d_sig;
    L.d_sig_down = rk[dn].d_sig;
    L.d_sig_up = rk[up].d_sig;
    return L;
  };

  // Every rank on its own thread and stream, all at once: spread, ghost sum,
  // halo fill, gather (epochs 1, 2), twice (epochs 3, 4).  Pass 0 runs the
  // local operators alone first: it sizes each context's scratch, since a
  // cudaMalloc waits for the whole device -- including another rank's
  // handshake, which waits for this rank (only ranks sharing a device).
  for (int pass = 0; pass < 2; ++pass) {
  std::vector<std::thread> th;
  for (int r = 0; r < R; ++r)
    th.emplace_back([&, r, pass] {
      Rank& k = rk[r];
      ibc_grid LG = G;
      LG.extent[2] = nzr + 3;
      LG.periodic[2] = 0;
      ibc_slab S{k.z0 - 2, nz, periodic ? 1 : 0};
      const ibc_slab_link Ls = link_of(r, false), Lf = link_of(r, true);
      if (pass == 0) {
        CHECK(ibc_spread_slab_device(k.ctx, &LG, &S, IBC_KERNEL_COSINE4, k.d_pts, k.d_vals,
                                     k.idx.size(), nullptr, k.d_spread));
        CHECK(ibc_interpolate_slab_device(k.ctx, &LG, &S, IBC_KERNEL_COSINE4, k.d_field, k.d_pts,
                                          k.idx.size(), k.d_E));
        CHECK(ibc_context_synchronize(k.ctx));
        return;
      }
      for (int rep = 0; rep < 2; ++rep) {
        CHECK(ibc_spread_slab_device(k.ctx, &LG, &S, IBC_KERNEL_COSINE4, k.d_pts, k.d_vals,
                                     k.idx.size(), nullptr, k.d_spread));
        CHECK(ibc_slab_ghost_sum_device(k.ctx, &Ls, 2 * rep + 1));
        CHECK(ibc_slab_halo_fill_device(k.ctx, &Lf, 2 * rep + 2));
        CHECK(ibc_interpolate_slab_device(k.ctx, &LG, &S, IBC_KERNEL_COSINE4, k.d_field, k.d_pts,
                                          k.idx.size(), k.d_E));
      }
      CHECK(ibc_context_synchronize(k.ctx));
    });
  for (auto& t : th) t.join();
  }

  std::vector<double> got(npts_grid), gotE(n);
  for (int r = 0; r < R; ++r) {
    Rank& k = rk[r];
    int timed_out = 0;
    const ibc_slab_link Ls = link_of(r, false);
    CHECK(ibc_slab_link_error(k.ctx, &Ls, &timed_out));
    if (timed_out) {
      std::fprintf(stderr, "FAIL R=%d rank %d: handshake timed out\n", R, r);
      ++failures;
    }
    cudaMemcpy(got.data() + (size_t)k.z0 * plane, k.d_spread + 2 * plane, 8 * plane * nzr,
               cudaMemcpyDeviceToHost);
    std::vector<double> e(k.idx.size());
    cudaMemcpy(e.data(), k.d_E, 8 * e.size(), cudaMemcpyDeviceToHost);
    for (size_t j = 0; j < e.size(); ++j) gotE[k.idx[j]] = e[j];
  }
  const double ds = max_rel(got, want), di = max_rel(gotE, wantE);
  std::printf("R=%d periodic=%d spread dev %.2e interp dev %.2e\n", R, periodic ? 1 : 0, ds, di);
  std::fflush(stdout);
  if (!(ds <= 1e-12) || !(di <= 1e-12)) ++failures;
  for (auto& k : rk) {
    ibc_device_free(k.ctx, k.d_spread);
    ibc_device_free(k.ctx, k.d_field);
    ibc_device_free(k.ctx, k.d_sig);
    cudaFree(k.d_pts); cudaFree(k.d_vals); cudaFree(k.d_E);
    ibc_context_destroy(k.ctx);
    cudaStreamDestroy(k.stream);
  }
  cudaFree(dX); cudaFree(dV); cudaFree(dOut); cudaFree(dF); cudaFree(dE); cudaFree(dPlanes);
  ibc_context_destroy(c0);
}

int main() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    std::printf("no CUDA device\n");
    return 77;
  }
  for (int R : {1, 2, 3, 4})
    for (bool periodic : {true, false}) {
      if (!periodic && R == 1) continue;
      run_case(R, periodic);
    }
  std::printf(failures ? "slab FAILED\n" : "slab ok\n");
  return failures ? 1 : 0;
}
