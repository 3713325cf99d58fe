// ibc_bucket.cuh -- bucket sort of the Lagrangian points (sm_100a).
//
// Both operators consume the points grouped by home row (cy, cz) -- the
// contiguous ranges of the reference's sorted cell keys that share a row
// (spread.hpp:88-122).  A one-pass counting sort does the grouping:
//   K1 cell key (bit-exact, grid.hpp:121-170) of every point, its bucket --
//      its row (interpolation) or its (row, x cell mod 16) pair (spread; a
//      row's 16 buckets are contiguous, so rows stay contiguous) -- and its
//      arrival rank in the bucket (the bucket-count atomic's return value);
//   K2 single-pass scan of the bucket counts (decoupled look-back) -> the
//      start table, the long-row list, the densest row and fullest bucket;
//   K3 atomic-free scatter to bucket start + rank (interpolation: the 64-byte
//      gather record; spread: the (key << 32 | index) pair).
// Interpolation results do not depend on the order inside a row (each point
// is summed alone, into its own slot), so K1-K3 are all it needs.  The spread
// sums many points into each grid value, so its summation order must not
// depend on the atomics' arrival order:
//   K4 one thread per point ranks its pair by counting over its (row, x bank)
//      bucket (bank mode) or its row (pull mode, rows <= 256 points; longer
//      rows: K4b, one CTA, bitonic sort in shared memory) and writes the
//      64-byte weight record (cell + one sin/cos pair per axis) at start +
//      rank.  Pull mode also writes the sorted pairs -- the reference's
//      stable key-value sort, ws.keys / ws.perm (spread.hpp:33-34); in bank
//      mode they are materialised on request (K4/K4b over the rows, mode 1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"

namespace ibc {
namespace bucket {

constexpr int kThreads = 256;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;                      // buckets per thread, one per row (interp)
constexpr uint32_t kFlagAggregate = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1u;
// Spread sweep, bank mode: target rows per warp and x banks per row (lanes per
// row).  A half-warp holds 16 bank pairs: 2 rows per warp -> 16 banks (x
// mod 16) per row; 4 rows per warp -> two rows interleaved per half, 8 banks
// (x mod 8) each.
constexpr int kRowsPerWarp = 2;
constexpr int kBanks = 32 / kRowsPerWarp;
constexpr int kShortRow = 256;      // rows up to this length are sorted by one warp

// Spread batching mode, decided on the device from the row scan's statistics
// stats[0] = densest row, stats[1] = fullest (row, x bank) bucket, and over
// the rows of >= kBalanceRow points stats[2] = sum of their fullest buckets,
// stats[3] = sum of their lengths: bank mode (lanes own x banks,
// ibc_spread.cuh) for sparse rows; for crowded buckets (>= kClusterBucket
// points), where the pull mode's same-cell shuffle groups serialise; and for
// dense rows whose points spread evenly over the x banks (fullest bucket of a
// row <= kBalance x its mean bucket, summed over the dense rows) -- a lane's
// list is then close to the row's mean, the bank sweep's lanes stay full.
// Measured spreads, bank vs pull (round 2, paired bank loop): W 128^3
// (balance 1.67) 437 vs 460 us, clustered (1.79) 1.91 vs 2.03 ms, severe
// clustering (fullest bucket 297) 10.4 vs 26.9 ms, RBC surfaces (balance
// 2.32: a membrane crossing a row fills a few banks) 422 vs 265 us.
constexpr uint32_t kClusterBucket = 36;
constexpr uint32_t kBalanceRow = 32;
constexpr uint32_t kBalance = 2;  // stats[2] * 16 <= kBalance * stats[3]
// pull_row == kNoBankMode: the bank window does not fit (very long x rows).
constexpr uint32_t kNoBankMode = 0xffffffffu;
__host__ __device__ __forceinline__ bool bank_mode(const uint32_t* stats, uint32_t pull_row) {
  if (pull_row == kNoBankMode) return false;
  if (pull_row == 0xfffffffeu) return true;  // forced (IBC_SPREAD_PATH_BANK)
  return stats[0] <= pull_row || stats[1] >= kClusterBucket ||
         (stats[3] > 0 && (uint64_t)stats[2] * 16u <= (uint64_t)kBalance * stats[3]);
}
constexpr int kLongSortMax = 8192;  // longest row the shared-memory bitonic sort takes
constexpr uint32_t kOutside = 0x80000000u;  // rank flag: home cell outside the grid (K1)

// Cell key of every point (or just its row when full_key == 0), its arrival
// rank in its bucket, and the per-bucket counts.  Buckets: rows (banks == 1,
// interpolation) or (row, x bank) pairs, row * kBanks + (x cell mod kBanks)
// (banks == kBanks, spreading) -- a row's buckets are contiguous, so the
// bucket order is a row order too.
template <int D>
__global__ void __launch_bounds__(kThreads) keys_kernel(DevGrid g, const double* __restrict__ X,
                                                        uint32_t n, int full_key, int banks,
                                                        uint32_t* __restrict__ keys,
                                                        uint32_t* __restrict__ rank,
                                                        uint32_t* __restrict__ count) {
  pdl_wait();
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
  bool inside = true;  // home cell within the extended range [-1, n] on closed axes
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (a == 0 && !full_key) continue;
    double xw;
    int c = cell_of(g, a, __ldg(X + (size_t)i * D + a), &xw);
    if (g.periodic[a]) c = wrap_cell(c, g.n[a]);
    else inside = inside && c >= -1 && c <= g.n[a];
    k += (uint64_t)(int64_t)(c + 1) * g.kstride[a];  // cell_key, grid.hpp:158-170
  }
  const uint32_t key = (uint32_t)k, row = key / g.rowdiv;
  // Points homed outside the extended cells of a closed axis (their keys
  // alias other rows, grid.hpp:158-170) go to an extra last row, flagged in
  // the rank's top bit; the operators skip them.
  const uint32_t bucket = !inside ? g.nrows * (uint32_t)banks
                          : banks > 1 ? row * (uint32_t)banks + ((key - row * g.rowdiv) & (banks - 1))
                                      : row;
  keys[i] = full_key ? key : row;
  rank[i] = atomicAdd(count + bucket, 1u) | (inside ? 0u : kOutside);
}

__device__ __forceinline__ void st_flag(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_flag(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Exclusive scan of count[0..nrows) into start[0..nrows] (start[nrows] = total);
// here "rows" are buckets, `group` (1 or kBanks) consecutive buckets per grid
// row.  status: one zeroed word per chunk; ticket: zeroed
// counter.  Grid rows longer than kShortRow are appended to long_rows (count
// in *nlong) when long_rows != null; maxrow[0] (zeroed, may be null) receives
// the largest grid-row count, maxrow[1] the largest bucket count.
template <int ITEMS>  // buckets per thread: kScanItems (group 1) or group (one grid row per thread)
__global__ void __launch_bounds__(kScanThreads) row_scan_kernel(const uint32_t* __restrict__ count,
                                                                uint32_t* __restrict__ start,
                                                                uint32_t nrows, int group,
                                                                uint32_t* status, uint32_t* ticket,
                                                                uint32_t* __restrict__ long_rows,
                                                                uint32_t* nlong, uint32_t* maxrow) {
  pdl_wait();
  __shared__ uint32_t s_warp[kScanThreads / 32], s_vmax[kScanThreads / 32], s_bmax[kScanThreads / 32];
  __shared__ uint32_t s_balb[kScanThreads / 32], s_baln[kScanThreads / 32];
  __shared__ uint32_t s_chunk, s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_chunk = atomicAdd(ticket, 1u);  // chunks start in ticket order
  __syncthreads();
  const uint32_t chunk = s_chunk;
  const uint32_t r0 = chunk * (uint32_t)(kScanThreads * ITEMS) + (uint32_t)tid * ITEMS;
  uint32_t v[ITEMS], sum = 0, vmax = 0;
  if (ITEMS % 4 == 0 && r0 + ITEMS <= nrows) {  // whole thread range: 16-byte loads
#pragma unroll
    for (int q = 0; q < ITEMS; q += 4) {
      const uint4 w = *reinterpret_cast<const uint4*>(count + r0 + q);
      v[q] = w.x;
      v[q + 1] = w.y;
      v[q + 2] = w.z;
      v[q + 3] = w.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) v[q] = r0 + q < nrows ? count[r0 + q] : 0u;
  }
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    sum += v[q];
    if (group == 1) {
      vmax = max(vmax, v[q]);
      if (long_rows && v[q] > (uint32_t)kShortRow) long_rows[atomicAdd(nlong, 1u)] = r0 + q;
    }
  }
  uint32_t bmax = 0, bal_b = 0, bal_n = 0;
  if (group > 1) {  // the thread's ITEMS == group buckets are one grid row
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) bmax = max(bmax, v[q]);
    vmax = sum;
    if (long_rows && sum > (uint32_t)kShortRow && r0 < nrows)
      long_rows[atomicAdd(nlong, 1u)] = r0 / (uint32_t)group;
    if (sum >= kBalanceRow) {  // dense row: its fullest bucket vs its length
      bal_b = bmax;
      bal_n = sum;
    }
  }
  vmax = __reduce_max_sync(0xffffffffu, vmax);
  bmax = __reduce_max_sync(0xffffffffu, bmax);
  bal_b = __reduce_add_sync(0xffffffffu, bal_b);
  bal_n = __reduce_add_sync(0xffffffffu, bal_n);
  if (lane == 0) {  // per-CTA maxima: one atomic per CTA, not per warp
    s_vmax[warp] = vmax;
    s_bmax[warp] = bmax;
    s_balb[warp] = bal_b;
    s_baln[warp] = bal_n;
  }
  // Block scan of the per-thread sums.
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s_warp[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    s_warp[lane] = wi - w;  // exclusive warp offsets
    const uint32_t total = __shfl_sync(0xffffffffu, wi, 31);
    if (maxrow) {  // densest row, fullest bucket (spread batching mode)
      const uint32_t cm = __reduce_max_sync(0xffffffffu, s_vmax[lane]);
      const uint32_t cb = __reduce_max_sync(0xffffffffu, s_bmax[lane]);
      const uint32_t sb = __reduce_add_sync(0xffffffffu, s_balb[lane]);
      const uint32_t sn = __reduce_add_sync(0xffffffffu, s_baln[lane]);
      if (lane == 0) {
        atomicMax(maxrow, cm);
        if (group > 1) {
          atomicMax(maxrow + 1, cb);
          if (sn) {
            atomicAdd(maxrow + 2, sb);
            atomicAdd(maxrow + 3, sn);
          }
        }
      }
    }
    // Publish the aggregate, then look back 32 chunks per round trip.
    if (lane == 0) st_flag(status + chunk, (chunk == 0 ? kFlagPrefix : kFlagAggregate) | total);
    uint32_t excl = 0;
    if (chunk > 0) {
      int c = (int)chunk - 1;
      while (true) {
        const int cc = c - lane;
        const uint32_t sv = cc >= 0 ? ld_flag(status + cc) : kFlagPrefix;
        const uint32_t ready = __ballot_sync(0xffffffffu, (sv & (kFlagPrefix | kFlagAggregate)) != 0u);
        const uint32_t pref = __ballot_sync(0xffffffffu, (sv & kFlagPrefix) != 0u);
        const int first_pref = pref ? __ffs(pref) - 1 : 32;
        const int first_nr = ~ready ? __ffs(~ready) - 1 : 32;
        if (first_pref < first_nr) {  // every lane up to the prefix is usable
          uint32_t add = lane <= first_pref ? (sv & kValueMask) : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
          excl += add;
          break;
        }
        uint32_t add = lane < first_nr ? (sv & kValueMask) : 0u;  // aggregates only
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
        excl += add;
        c -= first_nr;
      }
      if (lane == 0) st_flag(status + chunk, kFlagPrefix | (excl + total));
    }
    if (lane == 0) s_prefix = excl;
  }
  __syncthreads();
  uint32_t run = s_prefix + s_warp[warp] + x - sum;
  if (ITEMS % 4 == 0 && r0 + ITEMS <= nrows) {  // whole thread range: 16-byte stores
#pragma unroll
    for (int q = 0; q < ITEMS; q += 4) {
      uint4 w;
      w.x = run;
      w.y = w.x + v[q];
      w.z = w.y + v[q + 1];
      w.w = w.z + v[q + 2];
      run = w.w + v[q + 3];
      *reinterpret_cast<uint4*>(start + r0 + q) = w;
    }
    if (r0 + ITEMS == nrows) start[nrows] = run;
    return;
  }
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    if (r0 + q < nrows) {
      start[r0 + q] = run;
      run += v[q];
      if (r0 + q == nrows - 1) start[nrows] = run;
    }
  }
}

// K3, interpolation: each point's 64-byte record at row start + rank --
// {sin/cos(pi u_a / 2) for a = x, y, z; input index, home cx, home cy} -- so
// the gather does no cell or trig math.
// Points homed outside the grid (extra row g.nrows) get a record holding only
// their index: the gather zeroes their outputs (no support point reaches them).
template <int D>
__global__ void __launch_bounds__(kThreads) scatter_interp_kernel(
    DevGrid g, const double* __restrict__ X, const uint32_t* __restrict__ rows,
    const uint32_t* __restrict__ rank, uint32_t n, const uint32_t* __restrict__ start,
    double* __restrict__ rec) {
  pdl_wait();
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const uint32_t rk = __ldg(rank + i);
  if (rk & kOutside) {
    rec[8 * (size_t)(__ldg(start + g.nrows) + (rk & ~kOutside)) + 6] =
        __longlong_as_double((long long)i);
    return;
  }
  const uint32_t slot = __ldg(start + __ldg(rows + i)) + rk;
  double tr[3][2] = {{0.0, 1.0}, {0.0, 1.0}, {0.0, 1.0}};
  int c[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double w;
    c[a] = cell_and_u(axis_of(g, a), g.h, g.inv_h, __ldg(X + (size_t)i * D + a), &w);
    kernel_pair(g.kernel, w, &tr[a][0], &tr[a][1]);
  }
  double* r = rec + 8 * (size_t)slot;
  st_v4(r, tr[0][0], tr[0][1], tr[1][0], tr[1][1]);
  st_v4(r + 4, tr[2][0], tr[2][1], __longlong_as_double(((long long)c[0] << 32) | i),
        __longlong_as_double((long long)(uint32_t)c[1]));
}

// The spread's 64-byte weight record of point i at sorted position o:
//   {G phi_x(k-2-t_x)/h (k = 0..3), sin/cos(pi u_y/2), sin/cos(pi u_z/2)},
// and its home cell along x (wrapped on periodic x).
template <int D>
__device__ __forceinline__ void write_record_from(const DevGrid& g, const double (&x)[3], double gv,
                                                  uint32_t o, double* __restrict__ rec,
                                                  int* __restrict__ rcx) {
  double tr[3][2] = {{0.0, 1.0}, {0.0, 1.0}, {0.0, 1.0}};  // u = 0 on padded axes
  int cx = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double u;
    const int c = cell_and_u(axis_of(g, a), g.h, g.inv_h, x[a], &u);
    if (a == 0) cx = c;
    kernel_pair(g.kernel, u, &tr[a][0], &tr[a][1]);
  }
  const double gq = gv * (0.25 * g.inv_h);
  double* r = rec + 8 * (size_t)o;
  st_v4(r, gq * (1.0 - tr[0][1]), gq * (1.0 + tr[0][0]), gq * (1.0 + tr[0][1]),
        gq * (1.0 - tr[0][0]));
  st_v4(r + 4, tr[1][0], tr[1][1], tr[2][0], tr[2][1]);
  rcx[o] = cx;
}

template <int D>
__device__ __forceinline__ void write_record(const DevGrid& g, const double* __restrict__ X,
                                             const double* __restrict__ G, uint32_t i, uint32_t o,
                                             double* __restrict__ rec, int* __restrict__ rcx) {
  double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int a = 0; a < D; ++a) x[a] = __ldg(X + (size_t)i * D + a);
  write_record_from<D>(g, x, __ldg(G + i), o, rec, rcx);
}

// K3, spread: each point's (key << 32 | index) pair at its (row, x bank)
// bucket slot, start + arrival rank.
__global__ void __launch_bounds__(kThreads) scatter_spread_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ rank, uint32_t n,
    uint32_t rowdiv, uint32_t nrows, const uint32_t* __restrict__ start,
    unsigned long long* __restrict__ bpair) {
  pdl_wait();
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const uint32_t key = __ldg(keys + i), row = key / rowdiv, rk = __ldg(rank + i);
  const uint32_t bucket = (rk & kOutside) ? nrows * (uint32_t)kBanks
                                          : row * (uint32_t)kBanks + ((key - row * rowdiv) & (kBanks - 1));
  bpair[__ldg(start + bucket) + (rk & ~kOutside)] = ((unsigned long long)key << 32) | i;
}

// K4, one thread per bucket slot, ranking its (key, index) pair by counting
// over a contiguous range of pairs (L1 broadcasts: neighbouring lanes share
// it); the arrival order inside a bucket is not deterministic, the ranks are.
//   mode 0, bank mode: range = its (row, x bank) bucket; the weight record
//     goes to bucket start + rank -- records grouped by row and x bank, in
//     (key, index) order inside a bank: all the bank-mode sweep needs;
//   mode 0, pull mode: range = its row (<= kShortRow points, longer rows are
//     K4b's); the pair goes to row start + rank (ws.keys / ws.perm) and the
//     record with it;
//   mode 1 (on request, ensure_observables): the row's sorted pairs only.
template <int D>
__global__ void __launch_bounds__(kThreads) row_sort_kernel(
    const uint32_t* __restrict__ start, uint32_t n, const unsigned long long* __restrict__ bpair,
    uint32_t* __restrict__ skey, uint32_t* __restrict__ sidx, DevGrid g,
    const double* __restrict__ X, const double* __restrict__ G, double* __restrict__ rec,
    int* __restrict__ rcx, const uint32_t* __restrict__ maxrow, uint32_t bank_rows, int mode) {
  pdl_wait();
  const uint32_t o = blockIdx.x * kThreads + threadIdx.x;
  if (o >= n) return;
  const bool banked = mode == 0 && bank_mode(maxrow, bank_rows);
  const unsigned long long me = __ldg(bpair + o);
  const uint32_t k = (uint32_t)(me >> 32), ix = (uint32_t)me;
  // Slots past the grid rows hold the points homed outside (one bucket).
  const bool outside = o >= __ldg(start + (size_t)g.nrows * kBanks);
  const uint32_t row = outside ? g.nrows : k / g.rowdiv;
  const uint32_t b0 = banked && !outside
                          ? row * (uint32_t)kBanks + ((k - row * g.rowdiv) & (kBanks - 1))
                          : row * (uint32_t)kBanks;
  const uint32_t a = __ldg(start + b0);
  const uint32_t len = __ldg(start + b0 + (banked ? 1 : kBanks)) - a;
  if (!banked && len > (uint32_t)kShortRow) return;  // long rows: K4b
  // The point's position and value are gathered before the rank loop so
  // their latency hides behind it.
  double x[3] = {0.0, 0.0, 0.0};
  double gv = 0.0;
  if (mode == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) x[d] = __ldg(X + (size_t)ix * D + d);
    gv = __ldg(G + ix);
  }
  uint32_t rk = 0, j = 0;
  for (; j + 4 <= len; j += 4) {
    unsigned long long c[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) c[u] = __ldg(bpair + a + j + u);
#pragma unroll
    for (int u = 0; u < 4; ++u) rk += c[u] < me ? 1u : 0u;
  }
  for (; j < len; ++j) rk += __ldg(bpair + a + j) < me ? 1u : 0u;
  if (!banked) {
    skey[a + rk] = k;
    sidx[a + rk] = ix;
  }
  if (mode == 0) write_record_from<D>(g, x, gv, a + rk, rec, rcx);
}

// Bitonic sort of m (a power of two) 64-bit words in shared memory, one CTA.
constexpr int kLongThreads = 1024;
__device__ __forceinline__ void cta_bitonic(unsigned long long* sk, uint32_t m) {
  for (uint32_t size = 2; size <= m; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t e = threadIdx.x; e < m; e += kLongThreads) {
        const uint32_t p = e ^ stride;
        if (p > e) {
          const bool up = (e & size) == 0;
          const unsigned long long x = sk[e], y = sk[p];
          if ((x > y) == up) {
            sk[e] = y;
            sk[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// K4b, long rows: one CTA per listed row sorts its (key << 32 | index) pairs
// (all distinct: the index is unique).  Rows up to kLongSortMax: a bitonic
// sort in shared memory.  Longer rows (a fibre along x, a cluster in one row):
// kLongSortMax-chunks sorted the same way, then merged pairwise through
// global memory (`tmp`, n words) -- each element's place in the merged run is
// its index in its own run plus its rank in the partner run (binary search),
// O(len log len) per pass instead of the O(len^2) ranking by counting.
template <int D>
__global__ void __launch_bounds__(kLongThreads) long_row_sort_kernel(
    const uint32_t* __restrict__ start, const uint32_t* __restrict__ long_rows,
    const uint32_t* __restrict__ nlong, const unsigned long long* __restrict__ bpair,
    uint32_t* __restrict__ skey, uint32_t* __restrict__ sidx,
    DevGrid g, const double* __restrict__ X, const double* __restrict__ G,
    double* __restrict__ rec, int* __restrict__ rcx, const uint32_t* __restrict__ maxrow,
    uint32_t bank_rows, int mode, unsigned long long* __restrict__ tmp0,
    unsigned long long* __restrict__ tmp1) {
  pdl_wait();
  extern __shared__ unsigned long long sk[];  // [kLongSortMax] (key << 32 | index)
  if (mode == 0 && bank_mode(maxrow, bank_rows)) return;
  const uint32_t count = *nlong;
  for (uint32_t li = blockIdx.x; li < count; li += gridDim.x) {
    const uint32_t r = long_rows[li];
    const uint32_t a = start[(size_t)r * kBanks], len = start[(size_t)r * kBanks + kBanks] - a;
    const unsigned long long* sorted;
    if (len <= (uint32_t)kLongSortMax) {
      uint32_t m = 1;
      while (m < len) m <<= 1;
      for (uint32_t e = threadIdx.x; e < m; e += kLongThreads) sk[e] = e < len ? bpair[a + e] : ~0ull;
      __syncthreads();
      cta_bitonic(sk, m);
      sorted = sk;
    } else {
      // Sorted chunks into tmp0[a ..], then merge passes tmp0 <-> tmp1.
      for (uint32_t c0 = 0; c0 < len; c0 += kLongSortMax) {
        const uint32_t cl = min((uint32_t)kLongSortMax, len - c0);
        for (uint32_t e = threadIdx.x; e < (uint32_t)kLongSortMax; e += kLongThreads)
          sk[e] = e < cl ? bpair[a + c0 + e] : ~0ull;
        __syncthreads();
        cta_bitonic(sk, kLongSortMax);
        for (uint32_t e = threadIdx.x; e < cl; e += kLongThreads) tmp0[a + c0 + e] = sk[e];
        __syncthreads();
      }
      unsigned long long* src = tmp0 + a;
      unsigned long long* dst = tmp1 + a;
      for (uint32_t w = kLongSortMax; w < len; w <<= 1) {
        for (uint32_t e = threadIdx.x; e < len; e += kLongThreads) {
          const uint32_t run = e / (2 * w), lo = run * 2 * w, mid = min(lo + w, len),
                         hi = min(lo + 2 * w, len);
          const unsigned long long v = src[e];
          // partner run [plo, phi): elements of it below v
          const bool left = e < mid;
          uint32_t plo = left ? mid : lo, phi = left ? hi : mid, lo_b = plo, hi_b = phi;
          while (lo_b < hi_b) {
            const uint32_t mm = (lo_b + hi_b) >> 1;
            if (src[mm] < v) lo_b = mm + 1;
            else hi_b = mm;
          }
          const uint32_t own = e - (left ? lo : mid);
          dst[lo + own + (lo_b - plo)] = v;
        }
        __syncthreads();
        unsigned long long* t = src;
        src = dst;
        dst = t;
      }
      sorted = src;
    }
    for (uint32_t e = threadIdx.x; e < len; e += kLongThreads) {
      const unsigned long long v = sorted[e];
      skey[a + e] = (uint32_t)(v >> 32);
      sidx[a + e] = (uint32_t)v;
      if (mode == 0) write_record<D>(g, X, G, (uint32_t)v, a + e, rec, rcx);
    }
    __syncthreads();
  }
}

}  // namespace bucket
}  // namespace ibc
