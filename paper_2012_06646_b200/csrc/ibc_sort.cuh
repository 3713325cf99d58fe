// ibc_sort.cuh -- stable onesweep LSD radix sort of (cell key, point index).
//
// Replaces ib::key_value_sort<uint32_t> (sort.hpp:17-71).  Same contract:
// stable, so equal keys keep input order and the permutation is unique --
// bit-identical to the reference's ws.keys / ws.perm (spread.hpp:100).
//
// B200 structure:
//  * Keys are < prod(n_a + 2), so only key_bits(grid) bits are sorted, split
//    into P = ceil(bits / 9) balanced digits of <= 9 bits (25 bits at 256^3
//    -> 9/8/8, 17-bit row keys -> 9/8).
//  * The key kernel writes the keys, the global digit counts of EVERY pass
//    and the per-tile digit counts of pass 0.
//  * A pass is a tile-offset scan (per digit, over tiles; digit-major
//    parallel, coalesced over the tile-major count table) and ONE scatter
//    kernel over 2048-key tiles.  A tile ranks its keys with warp match
//    primitives (rank = popc(peers & lanemask_lt) + the warp's running digit
//    count) and scatters them, through shared memory in digit-sorted runs,
//    with coalesced stores; on the way out it counts the next pass's digits
//    per destination tile (warp-aggregated red.add), so no pass re-reads the
//    keys just to histogram them.
//  * The last pass can also gather a 32-byte payload per point (coordinates
//    + value or index) into sorted order, so the operators stream contiguous
//    records with TMA bulk copies.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"

namespace ibc {
namespace sort {

constexpr int kMaxDigitBits = 9;
constexpr int kMaxRadix = 1 << kMaxDigitBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;  // 2048 keys per tile
constexpr int kWarpSpan = 32 * kItems;    // 256 consecutive keys per warp
constexpr int kMaxPasses = 4;

// Payload gathered by the last pass, one 32-byte record per sorted position.
//   kPayloadSpread  {x, y, z, G}          (32 B)
//   kPayloadInterp  {x, y, z, index}      (32 B)
//   kPayloadWeights {G wx[4], sin/cos(pi u_y / 2), sin/cos(pi u_z / 2)} (64 B)
//                   + the home cell along x in rec_cx: everything the
//                   spread sweep needs, computed once per point.
enum Payload { kPayloadNone = 0, kPayloadSpread = 1, kPayloadInterp = 2, kPayloadWeights = 3 };

struct PassSmem {
  uint32_t wcount[kWarps][kMaxRadix];  // per-warp digit counts, then warp offsets
  uint32_t keys[kTile];
  uint32_t vals[kTile];
  uint32_t tstart[kMaxRadix];  // tile-local start of each digit
  uint32_t gofs[kMaxRadix];    // global position of the digit's run minus tstart
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

// Exclusive scan of one value per thread over a kThreads block; *total gets the sum.
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

// Tile offsets of one pass: off[t][d] = base[d] + sum_{t' < t} cnt[t'][d],
// base = exclusive scan of the digit totals gcount.  cnt/off are tile-major
// [ntiles][kMaxRadix].  One CTA per 32 digits: lane <-> digit, warps split the
// tiles (loads batched kUnrollT deep), so every access is a coalesced
// 128-byte row segment and no load waits on another.
constexpr int kUnrollT = 8;

__global__ void __launch_bounds__(kThreads) tile_offsets_kernel(
    const uint32_t* __restrict__ cnt, uint32_t* __restrict__ off, const uint32_t* __restrict__ gcount,
    int radix, int ntiles) {
  __shared__ uint32_t s_part[kWarps][32];
  __shared__ uint32_t s_below[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int d = blockIdx.x * 32 + lane;
  const bool dv = d < radix;
  // Totals of the digits below this CTA's range (warp w sums 64 of them).
  {
    uint32_t below = 0;
    for (int e = warp * 64 + lane; e < blockIdx.x * 32 && e < (warp + 1) * 64; e += 32)
      below += __ldg(gcount + e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
    if (lane == 0) s_below[warp] = below;
  }
  const int chunk = (ntiles + kWarps - 1) / kWarps;
  const int t0 = warp * chunk, t1 = min(ntiles, t0 + chunk);
  const uint32_t* col = cnt + d;
  uint32_t sum = 0;
  if (dv) {
    int t = t0;
    for (; t + kUnrollT <= t1; t += kUnrollT) {
      uint32_t v[kUnrollT];
#pragma unroll
      for (int u = 0; u < kUnrollT; ++u) v[u] = __ldg(col + (size_t)(t + u) * kMaxRadix);
#pragma unroll
      for (int u = 0; u < kUnrollT; ++u) sum += v[u];
    }
    for (; t < t1; ++t) sum += __ldg(col + (size_t)t * kMaxRadix);
  }
  s_part[warp][lane] = sum;
  __syncthreads();
  // base[d] = totals below the CTA + exclusive scan of gcount within it.
  uint32_t x = dv ? __ldg(gcount + d) : 0u, inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t acc = inc - x;
  for (int w = 0; w < kWarps; ++w) acc += s_below[w];
  for (int w = 0; w < warp; ++w) acc += s_part[w][lane];
  if (!dv) return;
  int t = t0;
  for (; t + kUnrollT <= t1; t += kUnrollT) {
    uint32_t v[kUnrollT];
#pragma unroll
    for (int u = 0; u < kUnrollT; ++u) v[u] = __ldg(col + (size_t)(t + u) * kMaxRadix);
#pragma unroll
    for (int u = 0; u < kUnrollT; ++u) {
      off[(size_t)(t + u) * kMaxRadix + d] = acc;
      acc += v[u];
    }
  }
  for (; t < t1; ++t) {
    const uint32_t c = __ldg(col + (size_t)t * kMaxRadix);
    off[(size_t)t * kMaxRadix + d] = acc;
    acc += c;
  }
}

// One stable digit pass over tile blockIdx.x.  vals_in == nullptr means the
// identity permutation.  off[t][d]: global start of digit d's keys of tile t
// (tile_offsets_kernel).  next_cnt (may be null): per-destination-tile digit
// counts of the next pass, accumulated here.
template <int PAYLOAD>
__global__ void __launch_bounds__(kThreads) onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t n, int shift,
    int bits, const uint32_t* __restrict__ off, uint32_t* __restrict__ next_cnt, int next_shift,
    int next_bits, const double* __restrict__ pts, const double* __restrict__ gvals,
    double* __restrict__ rec, DevGrid g, int* __restrict__ rec_cx) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem& S = *reinterpret_cast<PassSmem*>(smem_raw);
  const uint32_t radix = 1u << bits, mask = radix - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t i = tid; i < kWarps * radix; i += kThreads) S.wcount[i >> bits][i & mask] = 0u;
  __syncthreads();
  const uint32_t tile = blockIdx.x;
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
      key[j] = 0xffffffffu;
      val[j] = 0u;
    }
  }

  // Warp-level stable ranking in (j, lane) == input order.
  const uint32_t lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    const bool valid = idx < n;
    const uint32_t d = (key[j] >> shift) & mask;
    const uint32_t peers = __match_any_sync(0xffffffffu, valid ? d : 0xffffffffu);
    const uint32_t before = __popc(peers & lt_mask);
    uint32_t base = 0;
    if (valid) base = S.wcount[warp][d];
    __syncwarp();
    if (valid && before == 0) S.wcount[warp][d] = base + __popc(peers);
    __syncwarp();
    rank[j] = base + before;
  }
  __syncthreads();

  // Per digit: warp-exclusive offsets and the tile-local digit starts.
  constexpr int kDigitsPerThread = kMaxRadix / kThreads;
  uint32_t local = 0, cnt[kDigitsPerThread];
#pragma unroll
  for (int q = 0; q < kDigitsPerThread; ++q) {
    const uint32_t d = (uint32_t)tid * kDigitsPerThread + q;
    uint32_t c = 0;
    if (d < radix) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const uint32_t x = S.wcount[w][d];
        S.wcount[w][d] = c;
        c += x;
      }
    }
    cnt[q] = c;
    local += c;
  }
  uint32_t la = block_exclusive_scan(local, S.warp_tmp);
#pragma unroll
  for (int q = 0; q < kDigitsPerThread; ++q) {
    const uint32_t d = (uint32_t)tid * kDigitsPerThread + q;
    if (d < radix) {
      S.tstart[d] = la;
      S.gofs[d] = __ldg(off + (size_t)tile * kMaxRadix + d) - la;
    }
    la += cnt[q];
  }
  __syncthreads();

#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t idx = warp_base + (uint32_t)(j * 32 + lane);
    if (idx < n) {
      const uint32_t d = (key[j] >> shift) & mask;
      const uint32_t pos = S.tstart[d] + S.wcount[warp][d] + rank[j];
      S.keys[pos] = key[j];
      S.vals[pos] = val[j];
    }
  }
  __syncthreads();

  const uint32_t tile_n = min((uint32_t)kTile, n - tile_base);
  const uint32_t nmask = (1u << next_bits) - 1u;
  for (uint32_t i0 = 0; i0 < tile_n; i0 += kThreads) {
    const uint32_t i = i0 + tid;
    const bool valid = i < tile_n;
    uint32_t k = 0, o = 0;
    if (valid) {
      k = S.keys[i];
      const uint32_t v = S.vals[i];
      o = S.gofs[(k >> shift) & mask] + i;
      keys_out[o] = k;
      vals_out[o] = v;
      if (PAYLOAD == kPayloadWeights) {
        const int D = g.dim;
        const double* x = pts + (size_t)v * D;
        double tr[3][2] = {{0.0, 1.0}, {0.0, 1.0}, {0.0, 1.0}};  // u = 0 on padded axes
        int cx = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          if (a < D) {
            double u;
            const int c = cell_and_u(axis_of(g, a), g.h, g.inv_h, __ldg(x + a), &u);
            if (a == 0) cx = c;
            kernel_pair(g.kernel, u, &tr[a][0], &tr[a][1]);
          }
        }
        const double gq = __ldg(gvals + v) * (0.25 * g.inv_h);
        double4* r4 = reinterpret_cast<double4*>(rec) + 2 * (size_t)o;
        r4[0] = make_double4(gq * (1.0 - tr[0][1]), gq * (1.0 + tr[0][0]), gq * (1.0 + tr[0][1]),
                             gq * (1.0 - tr[0][0]));
        r4[1] = make_double4(tr[1][0], tr[1][1], tr[2][0], tr[2][1]);
        rec_cx[o] = cx;
      } else if (PAYLOAD != kPayloadNone) {
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
    if (next_cnt) {  // warp-aggregated count of (destination tile, next digit)
      const uint32_t slot =
          valid ? (o / (uint32_t)kTile) * kMaxRadix + ((k >> next_shift) & nmask) : 0xffffffffu;
      const uint32_t peers = __match_any_sync(0xffffffffu, slot);
      if (valid && (peers & lt_mask) == 0u) atomicAdd(next_cnt + slot, (uint32_t)__popc(peers));
    }
  }
}

}  // namespace sort
}  // namespace ibc
