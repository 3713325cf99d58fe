// ibc_sort.cuh -- stable onesweep LSD radix sort of (cell key, point index).
//
// Replaces ib::key_value_sort<uint32_t> (sort.hpp:17-71).  Same contract:
// stable, so equal keys keep input order and the permutation is unique --
// bit-identical to the reference's ws.keys / ws.perm (spread.hpp:100).
//
// Structure (Adinets & Merrill, "Onesweep", 2022), B200-sized:
//  * The per-pass digit histograms of ALL passes come from one read of the
//    keys, fused into the key-computation kernel (ibc_kernels.cu).
//  * One kernel per digit pass.  Each CTA claims a 4096-key tile through an
//    atomic tile counter (tiles are processed in claim order, so the look-back
//    always waits on CTAs that are already resident), ranks its keys with
//    warp ballots (8 __ballot_sync per item build the match mask of equal
//    digits; rank = popc(mask & lanemask_lt)), publishes its per-digit counts
//    and resolves its global offsets by decoupled look-back over preceding
//    tiles, then writes keys/values in digit-sorted runs through shared
//    memory so the global scatter is coalesced.
//  * Only ceil(key_bits / 8) passes run: keys are < prod(n_a + 2), e.g.
//    25 bits for 256^3.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ibc {
namespace sort {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kThreads = 256;  // == kRadix: one thread per digit in the scans
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 keys per tile
constexpr int kWarpSpan = 32 * kItems;    // 512 consecutive keys per warp
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValueMask = (1u << 30) - 1;
constexpr uint32_t kMaxKeys = kValueMask;  // counts are packed in 30 bits

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Exclusive scan of one value per thread over a 256-thread block.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  uint32_t base = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) base += (w < warp) ? s_warp[w] : 0u;
  __syncthreads();
  return base + x - v;
}

// One stable digit pass.  vals_in == nullptr means the identity permutation.
__global__ void __launch_bounds__(kThreads) onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
    const uint32_t* __restrict__ digit_base, uint32_t* __restrict__ lookback,
    uint32_t* __restrict__ tile_counter) {
  __shared__ uint32_t s_whist[kWarps][kRadix];
  __shared__ uint32_t s_keys[kTile];
  __shared__ uint32_t s_vals[kTile];
  __shared__ uint32_t s_tile_start[kRadix];
  __shared__ uint32_t s_gofs[kRadix];
  __shared__ uint32_t s_warp[kWarps];
  __shared__ uint32_t s_tile_id;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile_id = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kWarps * kRadix; i += kThreads) (&s_whist[0][0])[i] = 0u;
  __syncthreads();
  const uint32_t tile = s_tile_id;
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

  // Warp-level stable ranking: items are visited in (j, lane) order, which is
  // index order, and each equal-digit group is counted through the warp's
  // private histogram.
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    const bool valid = idx < n;
    const uint32_t d = (key[j] >> shift) & (kRadix - 1);
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < kRadixBits; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bb = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bb : ~bb;
    }
    const uint32_t before = __popc(peers & lt_mask);
    uint32_t base = 0;
    if (valid) base = s_whist[warp][d];
    __syncwarp();
    if (valid && before == 0) s_whist[warp][d] = base + __popc(peers);
    __syncwarp();
    rank[j] = base + before;
  }
  __syncthreads();

  // Thread t owns digit t: warp-exclusive offsets, tile count, look-back.
  {
    const uint32_t d = (uint32_t)tid;
    uint32_t count = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_whist[w][d];
      s_whist[w][d] = count;
      count += c;
    }
    uint32_t* mine = lookback + (size_t)tile * kRadix + d;
    uint32_t excl = 0;
    if (tile == 0) {
      st_release(mine, kFlagInc | count);
    } else {
      st_release(mine, kFlagAgg | count);
      int p = (int)tile - 1;
      while (true) {
        const uint32_t v = ld_acquire(lookback + (size_t)p * kRadix + d);
        if ((v & ~kValueMask) == 0u) continue;  // predecessor not published yet
        excl += v & kValueMask;
        if (v & kFlagInc) break;
        --p;
      }
      st_release(mine, kFlagInc | (excl + count));
    }
    const uint32_t start = block_exclusive_scan(count, s_warp);
    s_tile_start[d] = start;
    s_gofs[d] = digit_base[d] + excl - start;
  }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    if (idx < n) {
      const uint32_t d = (key[j] >> shift) & (kRadix - 1);
      const uint32_t pos = s_tile_start[d] + s_whist[warp][d] + rank[j];
      s_keys[pos] = key[j];
      s_vals[pos] = val[j];
    }
  }
  __syncthreads();

  const uint32_t tile_n = min((uint32_t)kTile, n - tile_base);
  for (uint32_t i = tid; i < tile_n; i += kThreads) {
    const uint32_t k = s_keys[i];
    const uint32_t d = (k >> shift) & (kRadix - 1);
    const uint32_t o = s_gofs[d] + i;
    keys_out[o] = k;
    vals_out[o] = s_vals[i];
  }
}

// Exclusive scan of each pass's global digit histogram (one block per pass).
__global__ void __launch_bounds__(kThreads) digit_scan(const uint32_t* __restrict__ hist,
                                                       uint32_t* __restrict__ base) {
  __shared__ uint32_t s_warp[kWarps];
  const uint32_t v = hist[blockIdx.x * kRadix + threadIdx.x];
  base[blockIdx.x * kRadix + threadIdx.x] = block_exclusive_scan(v, s_warp);
}

}  // namespace sort
}  // namespace ibc
