// ibc_bucket.cuh -- row bucketing of interpolation points (sm_100a).
//
// The interpolation gather (interpolate.hpp:22-58) needs the points grouped
// by home row (cy, cz) -- each point's result is written to its own input
// slot and summed in a fixed order by one quad of lanes, so the order of the
// points inside a row does not change any result.  That makes a one-pass
// counting bucket sort enough:
//   K1 row keys + per-row counts; the atomic's return value is the point's
//      rank inside its row, kept for K3,
//   K2 single-pass scan of the row counts with decoupled look-back over
//      4096-row chunks -> the row start table the sweep reads,
//   K3 scatter: each point writes its 32-byte record {x, y, z, input index}
//      to row start + rank (no atomics).
// Three kernels instead of a key sort + row table; the spread keeps the
// stable radix sort because its sums (and ws.keys / ws.perm) depend on order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"

namespace ibc {
namespace bucket {

constexpr int kThreads = 256;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kChunk = kScanThreads * kScanItems;  // rows per scan CTA
constexpr uint32_t kFlagAggregate = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1u;

// Row id (cell_key / (n0 + 2)) of every point, its rank in the row, and the
// per-row counts.
template <int D>
__global__ void __launch_bounds__(kThreads) row_keys_kernel(DevGrid g, const double* __restrict__ X,
                                                            uint32_t n, uint32_t* __restrict__ rows,
                                                            uint32_t* __restrict__ rank,
                                                            uint32_t* __restrict__ count) {
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  uint64_t k = 0;
#pragma unroll
  for (int a = 1; a < D; ++a) {
    double xw;
    int c = cell_of(g, a, __ldg(X + (size_t)i * D + a), &xw);
    if (g.periodic[a]) c = wrap_cell(c, g.n[a]);
    k += (uint64_t)(int64_t)(c + 1) * (g.kstride[a] / g.rowdiv);
  }
  const uint32_t row = (uint32_t)k;
  rows[i] = row;
  rank[i] = atomicAdd(count + row, 1u);
}

__device__ __forceinline__ void st_flag(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_flag(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Exclusive scan of count[0..nrows) into start[0..nrows] (start[nrows] = total).
// status: one zeroed word per chunk; ticket: zeroed counter.
__global__ void __launch_bounds__(kScanThreads) row_scan_kernel(uint32_t* __restrict__ count,
                                                                uint32_t* __restrict__ start,
                                                                uint32_t nrows, uint32_t* status,
                                                                uint32_t* ticket) {
  __shared__ uint32_t s_warp[kScanThreads / 32];
  __shared__ uint32_t s_chunk, s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_chunk = atomicAdd(ticket, 1u);  // chunks start in ticket order
  __syncthreads();
  const uint32_t chunk = s_chunk;
  const uint32_t r0 = chunk * (uint32_t)kChunk + (uint32_t)tid * kScanItems;
  uint32_t v[kScanItems], sum = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    v[q] = r0 + q < nrows ? count[r0 + q] : 0u;
    sum += v[q];
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
        // Lanes up to the first prefix (or first not-ready lane) are usable.
        const uint32_t stop_ready = ~ready;  // first not-ready lane
        const int first_pref = pref ? __ffs(pref) - 1 : 32;
        const int first_nr = stop_ready ? __ffs(stop_ready) - 1 : 32;
        if (first_pref < first_nr) {
          uint32_t add = lane <= first_pref ? (sv & kValueMask) : 0u;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) add += __shfl_xor_sync(0xffffffffu, add, o);
          excl += add;
          break;
        }
        uint32_t add = lane < first_nr ? (sv & kValueMask) : 0u;
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
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (r0 + q < nrows) {
      start[r0 + q] = run;
      run += v[q];
      if (r0 + q == nrows - 1) start[nrows] = run;
    }
  }
}

// Each point writes {x, y, z, index} to its row's start + its rank.
__global__ void __launch_bounds__(kThreads) scatter_kernel(const double* __restrict__ X,
                                                           const uint32_t* __restrict__ rows,
                                                           const uint32_t* __restrict__ rank, uint32_t n,
                                                           const uint32_t* __restrict__ start,
                                                           double* __restrict__ rec) {
  const uint32_t i = blockIdx.x * kThreads + threadIdx.x;
  if (i >= n) return;
  const uint32_t slot = __ldg(start + __ldg(rows + i)) + __ldg(rank + i);
  double4 r;
  r.x = __ldg(X + (size_t)i * 3);
  r.y = __ldg(X + (size_t)i * 3 + 1);
  r.z = __ldg(X + (size_t)i * 3 + 2);
  r.w = __longlong_as_double((long long)i);
  reinterpret_cast<double4*>(rec)[slot] = r;
}

}  // namespace bucket
}  // namespace ibc
