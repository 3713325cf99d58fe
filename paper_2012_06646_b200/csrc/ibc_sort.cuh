// ibc_sort.cuh -- stable LSD radix sort of (cell key, point index) on sm_100a.
//
// Replaces ib::key_value_sort<uint32_t> (sort.hpp:17-71).  Same contract:
// stable, so equal keys keep input order and the permutation is unique --
// bit-identical to the reference's ws.keys / ws.perm (spread.hpp:100).
//
// B200 structure:
//  * Keys are < prod(n_a + 2), so only key_bits(grid) bits are sorted, split
//    into P = ceil(bits / 10) balanced digits of <= 10 bits (25 bits at
//    256^3 -> 9/8/8: three passes instead of the reference's four).
//  * Each pass is ONE scatter kernel over 4096-key tiles.  A tile ranks its
//    keys with warp ballots (one __ballot_sync per digit bit builds the
//    equal-digit match mask; rank = popc(mask & lanemask_lt)), and reads its
//    global digit offsets from a table prepared before the pass -- there is
//    no decoupled look-back, so no tile ever waits on another:
//      - the per-tile digit histogram of pass 0 comes from the key kernel
//        (which works tile by tile over the input order),
//      - the per-tile histogram of pass p+1 is accumulated by pass p's
//        scatter (each key knows its output slot, hence its next tile),
//      - a small column scan turns histograms into offsets between passes.
//  * Keys/values leave the tile through shared memory in digit-sorted runs,
//    so the global scatter is coalesced.  The last pass can also gather a
//    32-byte payload per point (coordinates + value or index) into sorted
//    order, so the operators stream contiguous records with TMA bulk copies.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ibc {
namespace sort {

constexpr int kMaxDigitBits = 10;
constexpr int kMaxRadix = 1 << kMaxDigitBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile
constexpr int kWarpSpan = 32 * kItems;    // 512 consecutive keys per warp
constexpr int kMaxPasses = 4;

// Payload gathered by the last pass, one 32-byte record per sorted position.
enum Payload { kPayloadNone = 0, kPayloadSpread = 1, kPayloadInterp = 2 };

struct PassSmem {
  uint32_t whist[kWarps][kMaxRadix];  // per-warp digit counts, then warp offsets
  uint32_t keys[kTile];
  uint32_t vals[kTile];
  uint32_t tile_start[kMaxRadix];
  uint32_t gofs[kMaxRadix];
  uint32_t warp_tmp[kWarps];
};

struct DigitPlan {
  int passes;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
};

inline DigitPlan plan_digits(int key_bits) {
  DigitPlan p{};
  p.passes = (key_bits + kMaxDigitBits - 1) / kMaxDigitBits;
  if (p.passes < 1) p.passes = 1;
  int shift = 0;
  for (int i = 0; i < p.passes; ++i) {
    const int rem = key_bits - shift, left = p.passes - i;
    p.bits[i] = (rem + left - 1) / left;
    p.shift[i] = shift;
    shift += p.bits[i];
  }
  return p;
}

// Exclusive scan of one value per thread over a 256-thread block; *total gets the sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp,
                                                         uint32_t* total = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  uint32_t base = 0, all = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t s = s_warp[w];
    base += (w < warp) ? s : 0u;
    all += s;
  }
  __syncthreads();
  if (total) *total = all;
  return base + x - v;
}

// Column scan between passes: hist[d][t] (digit-major, ntiles per digit) ->
// exclusive prefix over tiles, in place; total[d] = column sum.  One block
// per digit.
__global__ void __launch_bounds__(kThreads) tile_scan(uint32_t* __restrict__ hist,
                                                      uint32_t* __restrict__ total, int ntiles) {
  __shared__ uint32_t s_warp[kWarps];
  uint32_t* col = hist + (size_t)blockIdx.x * ntiles;
  uint32_t carry = 0;
  for (int t0 = 0; t0 < ntiles; t0 += kThreads) {
    const int t = t0 + threadIdx.x;
    const uint32_t v = t < ntiles ? col[t] : 0u;
    uint32_t sum;
    const uint32_t ex = block_exclusive_scan(v, s_warp, &sum);
    if (t < ntiles) col[t] = carry + ex;
    carry += sum;
  }
  if (threadIdx.x == 0) total[blockIdx.x] = carry;
}

// One stable digit pass over tile blockIdx.x.  vals_in == nullptr means the
// identity permutation.  tile_off[d][t]: exclusive prefix of digit d over
// preceding tiles; total[d]: count of digit d.  next_hist (may be null):
// per-tile histogram of the next pass, accumulated over output slots.
template <int PAYLOAD>
__global__ void __launch_bounds__(kThreads) onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
    int bits, const uint32_t* __restrict__ tile_off, const uint32_t* __restrict__ total,
    int ntiles, uint32_t* __restrict__ next_hist, int next_shift, int next_bits,
    const double* __restrict__ pts, const double* __restrict__ gvals, double* __restrict__ rec) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem& S = *reinterpret_cast<PassSmem*>(smem_raw);
  const uint32_t radix = 1u << bits, mask = radix - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t tile = blockIdx.x;
  for (uint32_t i = tid; i < kWarps * radix; i += kThreads) S.whist[i >> bits][i & mask] = 0u;
  // Global digit bases: exclusive scan of the digit totals.
  {
    uint32_t carry = 0;
    for (uint32_t d0 = 0; d0 < radix; d0 += kThreads) {
      const uint32_t d = d0 + tid;
      const uint32_t v = d < radix ? total[d] : 0u;
      uint32_t sum;
      const uint32_t ex = block_exclusive_scan(v, S.warp_tmp, &sum);
      if (d < radix) S.gofs[d] = carry + ex + tile_off[(size_t)d * ntiles + tile];
      carry += sum;
    }
  }
  __syncthreads();
  const uint32_t tile_base = tile * (uint32_t)kTile;
  const uint32_t warp_base = tile_base + (uint32_t)warp * kWarpSpan;

  uint32_t key[kItems], val[kItems], rank[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    if (idx < n) {
      key[j] = __ldg(keys_in + idx);
      val[j] = vals_in ? __ldg(vals_in + idx) : idx;
    } else {
      key[j] = 0u;
      val[j] = 0u;
    }
  }

  // Warp-level stable ranking in (j, lane) == index order.
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    const bool valid = idx < n;
    const uint32_t d = (key[j] >> shift) & mask;
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
    for (int b = 0; b < bits; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    const uint32_t before = __popc(peers & lt_mask);
    uint32_t base = 0;
    if (valid) base = S.whist[warp][d];
    __syncwarp();
    if (valid && before == 0) S.whist[warp][d] = base + __popc(peers);
    __syncwarp();
    rank[j] = base + before;
  }
  __syncthreads();

  // Per digit: warp-exclusive offsets and the tile count; tile-local starts.
  {
    uint32_t carry = 0;
    for (uint32_t d0 = 0; d0 < radix; d0 += kThreads) {
      const uint32_t d = d0 + tid;
      uint32_t c = 0;
      if (d < radix) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const uint32_t x = S.whist[w][d];
          S.whist[w][d] = c;
          c += x;
        }
      }
      uint32_t sum;
      const uint32_t start = carry + block_exclusive_scan(c, S.warp_tmp, &sum);
      carry += sum;
      if (d < radix) {
        S.tile_start[d] = start;
        S.gofs[d] -= start;
      }
    }
  }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    if (idx < n) {
      const uint32_t d = (key[j] >> shift) & mask;
      const uint32_t pos = S.tile_start[d] + S.whist[warp][d] + rank[j];
      S.keys[pos] = key[j];
      S.vals[pos] = val[j];
    }
  }
  __syncthreads();

  const uint32_t tile_n = min((uint32_t)kTile, n - tile_base);
  const uint32_t nmask = (1u << next_bits) - 1u;
  for (uint32_t i = tid; i < tile_n; i += kThreads) {
    const uint32_t k = S.keys[i];
    const uint32_t v = S.vals[i];
    const uint32_t o = S.gofs[(k >> shift) & mask] + i;
    keys_out[o] = k;
    vals_out[o] = v;
    if (next_hist)
      atomicAdd(&next_hist[(size_t)((k >> next_shift) & nmask) * ntiles + o / (uint32_t)kTile], 1u);
    if (PAYLOAD != kPayloadNone) {
      const double* x = pts + (size_t)v * 3;
      double4 r;
      r.x = __ldg(x);
      r.y = __ldg(x + 1);
      r.z = __ldg(x + 2);
      if (PAYLOAD == kPayloadSpread) r.w = __ldg(gvals + v);
      else r.w = __longlong_as_double((long long)v);
      reinterpret_cast<double4*>(rec)[o] = r;
    }
  }
}

}  // namespace sort
}  // namespace ibc
