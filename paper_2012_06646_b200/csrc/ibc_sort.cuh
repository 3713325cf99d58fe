// ibc_sort.cuh -- stable onesweep LSD radix sort of (cell key, point index).
//
// Replaces ib::key_value_sort<uint32_t> (sort.hpp:17-71).  Same contract:
// stable, so equal keys keep input order and the permutation is unique --
// bit-identical to the reference's ws.keys / ws.perm (spread.hpp:100).
//
// Structure (Adinets & Merrill, "Onesweep", 2022), B200-sized:
//  * Keys are < prod(n_a + 2), so only key_bits(grid) bits are sorted, split
//    into P = ceil(bits / 10) balanced digits of <= 10 bits (25 bits at 256^3
//    -> 9/8/8: three passes instead of the reference's four 8-bit passes).
//  * The digit histograms of ALL passes come from one read of the keys,
//    fused into the key-computation kernel (ibc_kernels.cu).
//  * One kernel per digit pass.  Each CTA claims a 4096-key tile through an
//    atomic tile counter (so look-back only ever waits on CTAs that are
//    already resident), ranks its keys with warp ballots (one __ballot_sync
//    per digit bit builds the equal-digit match mask; rank =
//    popc(mask & lanemask_lt)), publishes per-digit tile counts and resolves
//    global offsets by decoupled look-back that polls 32 predecessor tiles
//    per round trip, then writes keys/values in digit-sorted runs through
//    shared memory so the global scatter is coalesced.
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
constexpr int kDigitsPerThread = kMaxRadix / kThreads;
constexpr int kLookback = 32;             // predecessor tiles polled per round trip
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr int kMaxPasses = 4;

// Shared memory of one pass (dynamic: > 48 KB).
struct PassSmem {
  uint32_t whist[kWarps][kMaxRadix];  // per-warp digit counts, then warp offsets
  uint32_t keys[kTile];
  uint32_t vals[kTile];
  uint32_t tile_start[kMaxRadix];
  uint32_t gofs[kMaxRadix];
  uint32_t warp_tmp[kWarps];
  uint32_t tile_id;
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

// The look-back words carry only their own payload (no other data is
// published through them), so relaxed gpu-scope accesses suffice: they are
// served by L2 without the L1 invalidation (CCTL.IVALL) an acquire costs.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// Decoupled look-back for one digit: sum of the counts of all preceding
// tiles.  Polls kLookback predecessors per round trip.
__device__ __forceinline__ uint32_t lookback_digit(const uint32_t* lookback, uint32_t tile,
                                                   uint32_t radix, uint32_t d) {
  uint32_t excl = 0;
  int p = (int)tile - 1;
  while (p >= 0) {
    uint32_t v[kLookback];
#pragma unroll
    for (int j = 0; j < kLookback; ++j)
      v[j] = (p - j >= 0) ? ld_acquire(lookback + (size_t)(p - j) * radix + d) : kFlagInc;
    int consumed = 0;
    bool done = false;
#pragma unroll
    for (int j = 0; j < kLookback; ++j) {
      if (done || consumed != j) continue;
      if (p - j < 0) { done = true; continue; }
      const uint32_t f = v[j] & ~kValueMask;
      if (f == 0u) continue;  // not yet published: re-poll from here
      excl += v[j] & kValueMask;
      ++consumed;
      if (f == kFlagInc) done = true;
    }
    if (done) break;
    p -= consumed;
  }
  return excl;
}

// One stable digit pass.  vals_in == nullptr means the identity permutation.
__global__ void __launch_bounds__(kThreads) onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
    int bits, const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ lookback,
    uint32_t* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem& S = *reinterpret_cast<PassSmem*>(smem_raw);
  const uint32_t radix = 1u << bits, mask = radix - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1u);
  for (uint32_t i = tid; i < kWarps * radix; i += kThreads) S.whist[i >> bits][i & mask] = 0u;
  __syncthreads();
  const uint32_t tile = S.tile_id;
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

  // Digits are owned round-robin by threads: d = tid + 256 * i.
  uint32_t count[kDigitsPerThread];
#pragma unroll
  for (int i = 0; i < kDigitsPerThread; ++i) {
    const uint32_t d = tid + kThreads * i;
    uint32_t c = 0;
    if (d < radix) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t x = S.whist[w][d];
        S.whist[w][d] = c;
        c += x;
      }
      st_release(lookback + (size_t)tile * radix + d, (tile == 0 ? kFlagInc : kFlagAgg) | c);
    }
    count[i] = c;
  }
  uint32_t excl[kDigitsPerThread];
#pragma unroll
  for (int i = 0; i < kDigitsPerThread; ++i) {
    const uint32_t d = tid + kThreads * i;
    excl[i] = 0;
    if (d < radix && tile > 0) {
      excl[i] = lookback_digit(lookback, tile, radix, d);
      st_release(lookback + (size_t)tile * radix + d, kFlagInc | (excl[i] + count[i]));
    }
  }
  // Tile-local exclusive scan over digits (digit-major across the threads).
  uint32_t carry = 0;
#pragma unroll
  for (int i = 0; i < kDigitsPerThread; ++i) {
    const uint32_t d = tid + kThreads * i;
    if ((uint32_t)(kThreads * i) >= radix) break;  // block-uniform
    uint32_t total;
    const uint32_t start = carry + block_exclusive_scan(count[i], S.warp_tmp, &total);
    carry += total;
    if (d < radix) {
      S.tile_start[d] = start;
      S.gofs[d] = digit_base[d] + excl[i] - start;
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
  for (uint32_t i = tid; i < tile_n; i += kThreads) {
    const uint32_t k = S.keys[i];
    const uint32_t o = S.gofs[(k >> shift) & mask] + i;
    keys_out[o] = k;
    vals_out[o] = S.vals[i];
  }
}

// Exclusive scan of each pass's global digit histogram (one block per pass).
__global__ void __launch_bounds__(kThreads) digit_scan(const uint32_t* __restrict__ hist,
                                                       uint32_t* __restrict__ base,
                                                       DigitPlan plan) {
  __shared__ uint32_t s_warp[kWarps];
  const int p = blockIdx.x;
  const uint32_t radix = 1u << plan.bits[p];
  const uint32_t* h = hist + (size_t)p * kMaxRadix;
  uint32_t* b = base + (size_t)p * kMaxRadix;
  uint32_t carry = 0;
  for (uint32_t i0 = 0; i0 < radix; i0 += kThreads) {
    const uint32_t i = i0 + threadIdx.x;
    const uint32_t v = i < radix ? h[i] : 0u;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan(v, s_warp, &total);
    if (i < radix) b[i] = carry + ex;
    carry += total;
  }
}

}  // namespace sort
}  // namespace ibc
