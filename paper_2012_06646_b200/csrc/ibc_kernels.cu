// ibc_kernels.cu -- pipelines of the spread / interpolate hot path (sm_100a).
//
// Per operator call:
//   spread, 2-D/3-D grids:  (row, x bank) bucket sort + in-bucket (bank mode)
//     or in-row (pull mode) ranking + weight records (ibc_bucket.cuh) ->
//     write-once sweep (ibc_spread.cuh)
//   interpolation, 3-D grids with nx % 16 == 0: row bucketing
//     (ibc_bucket.cuh) -> TMA-fed gather (ibc_sweep.cuh)
//   general path (1-D grids, rows too long for a shared-memory window, other
//   x extents, IBC_SORT=radix):
//     keys_hist_kernel     wrap -> cell -> 32-bit key + pass-0 digit counts
//                                                          (grid.hpp:121-207)
//     tile_offsets_kernel + onesweep_pass x P  stable key/index radix sort
//                                                          (sort.hpp:17-71)
//     rowstart_kernel      extended-row start table        (reduce.hpp:36-69)
//     prep_records_kernel + spread_tiles_kernel  write-once spread
//                                                          (spread.hpp:165-216)
//     interp_kernel        interpolation gather            (interpolate.hpp:22-58)
//   run keys / q on demand: head_count / block_scan / head_write.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <utility>

#include "ibc_internal.h"
#include "ibc_sort.cuh"
#include "ibc_sweep.cuh"
#include "ibc_bucket.cuh"
#include "ibc_spread.cuh"
#include "ibc_tma.cuh"

namespace ibc {

// Launch with programmatic stream serialization (PDL): the kernel's launch
// overlaps its predecessor's tail; it waits in pdl_wait() (ibc_device.cuh)
// before touching memory.  Works inside CUDA graph capture.
template <typename... KArgs, typename... Args>
static void pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  IBC_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

namespace {

constexpr int kBlock = 256;
constexpr int kSpreadThreads = 256;
constexpr int kMaxPasses = sort::kMaxPasses;
constexpr int kCounters = kMaxPasses + 1;  // tile counters + run count q

__device__ __forceinline__ uint32_t lanemask_le() {
  const int lane = threadIdx.x & 31;
  return lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
}

// ---------------------------------------------------------------- K1
// Cell key of every point (or, with row_only, its extended row id -- all the
// interpolation needs) and the digit histograms of every radix pass.
constexpr int kKeysUnroll = 4;

template <int D>
__device__ __forceinline__ uint32_t key_of(const DevGrid& g, const double* x, bool row_only) {
  uint64_t k = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double xw;
    int c = cell_of(g, a, x[a], &xw);
    if (g.periodic[a]) c = wrap_cell(c, g.n[a]);
    k += (uint64_t)(int64_t)(c + 1) * g.kstride[a];  // cell_key, grid.hpp:158-170
  }
  uint32_t key = (uint32_t)k;
  if (row_only) key /= g.rowdiv;
  return key;
}

// One CTA per 2048-key sort tile (the input order): cell keys of its points,
// their digit counts for EVERY radix pass added to gcount[p][d], and the
// tile's pass-0 digit counts cnt0[tile][d].
constexpr int kKeysThreads = sort::kThreads;

struct KeyDigits {
  int passes;
  int shift[sort::kMaxPasses];
  int bits[sort::kMaxPasses];
};

template <int D>
__global__ void __launch_bounds__(kKeysThreads) keys_hist_kernel(
    DevGrid g, const double* __restrict__ X, uint32_t n, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ gcount, uint32_t* __restrict__ cnt0, KeyDigits kd, int row_only) {
  __shared__ uint32_t sh[sort::kMaxPasses][sort::kMaxRadix];
  for (int t = threadIdx.x; t < sort::kMaxPasses * sort::kMaxRadix; t += blockDim.x)
    (&sh[0][0])[t] = 0u;
  __syncthreads();
  const uint32_t base = blockIdx.x * (uint32_t)sort::kTile;
  constexpr int kPer = sort::kTile / kKeysThreads;  // 8 points per thread
  static_assert(kPer % kKeysUnroll == 0, "tile split");
  for (int j0 = 0; j0 < kPer; j0 += kKeysUnroll) {
    double x[kKeysUnroll][D];
#pragma unroll
    for (int u = 0; u < kKeysUnroll; ++u) {
      const uint32_t i = base + (uint32_t)(j0 + u) * kKeysThreads + threadIdx.x;
#pragma unroll
      for (int a = 0; a < D; ++a) x[u][a] = i < n ? __ldg(X + (size_t)i * D + a) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kKeysUnroll; ++u) {
      const uint32_t i = base + (uint32_t)(j0 + u) * kKeysThreads + threadIdx.x;
      if (i < n) {
        const uint32_t key = key_of<D>(g, x[u], row_only != 0);
        keys[i] = key;
#pragma unroll
        for (int p = 0; p < sort::kMaxPasses; ++p)
          if (p < kd.passes) atomicAdd(&sh[p][(key >> kd.shift[p]) & ((1u << kd.bits[p]) - 1u)], 1u);
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (1 << kd.bits[0]); t += blockDim.x)
    cnt0[(size_t)blockIdx.x * sort::kMaxRadix + t] = sh[0][t];
#pragma unroll
  for (int p = 0; p < sort::kMaxPasses; ++p) {
    if (p >= kd.passes) break;
    const int radix = 1 << kd.bits[p];
    for (int t = threadIdx.x; t < radix; t += blockDim.x) {
      const uint32_t c = sh[p][t];
      if (c) atomicAdd(gcount + p * sort::kMaxRadix + t, c);
    }
  }
}

// ---------------------------------------------------------------- K3
// rowstart[r] = first sorted index whose extended row id is >= r, r in [0, nrows].
__global__ void __launch_bounds__(kBlock) rowstart_kernel(const uint32_t* __restrict__ sk, uint32_t n,
                                                          uint32_t rowdiv, uint32_t nrows,
                                                          uint32_t* __restrict__ rowstart) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    // (min: keys of points homed outside a closed axis can alias past the
    // last row -- keep the writes inside the table.)
    const uint32_t row = min(sk[i] / rowdiv, nrows);
    const uint32_t prow = i == 0 ? 0u : min(sk[i - 1] / rowdiv, nrows);
    for (uint32_t r = i == 0 ? 0u : prow + 1; r <= row; ++r) rowstart[r] = i;
    if (i == n - 1)
      for (uint32_t r = row + 1; r <= nrows; ++r) rowstart[r] = n;
  }
}

// ---------------------------------------------------------------- K4a
// Sorted per-point weight records for the tiled spread:
//   rec[k][r]     = G * phi_x(k-2 - t_x)/h     (k = 0..3)
//   rec[4+k][r]   = phi_y(k-2 - t_y)/h
//   rec[8+k][r]   = phi_z(k-2 - t_z)/h
//   rec_cx[r]     = home cell along x (wrapped on periodic axes)
__global__ void __launch_bounds__(kBlock) prep_records_kernel(DevGrid g, const double* __restrict__ X,
                                                              const double* __restrict__ G,
                                                              const uint32_t* __restrict__ perm,
                                                              uint32_t n, int* __restrict__ rec_cx,
                                                              double* __restrict__ rec) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t i = __ldg(perm + r);
  const int D = g.dim;
  double w[3][4];
  int c0 = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a < D) {
      double xw;
      const int c = cell_of(g, a, __ldg(X + (size_t)i * D + a), &xw);
      kernel_weights(g, displacement(g, a, xw, c), w[a]);
      if (a == 0) c0 = g.periodic[0] ? wrap_cell(c, g.n[0]) : c;
    } else {
      unit_weights(w[a], g.slo);
    }
  }
  const double gv = __ldg(G + i);
  rec_cx[r] = c0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    rec[(size_t)k * n + r] = w[0][k] * gv;
    rec[(size_t)(4 + k) * n + r] = w[1][k];
    rec[(size_t)(8 + k) * n + r] = w[2][k];
  }
}

// ---------------------------------------------------------------- K4b
struct SpreadTiling {
  int tx, ty, tz;     // target tile extents (tx == n0 when rows are whole)
  int ntx, nty, ntz;  // tiles per axis
};

// Write-once spread.  One CTA owns a tile of target rows (all of x, or an x
// chunk) x ty x tz held in shared memory.  Warp w owns target rows w, w+8, ...
// and PULLS, in fixed (sigma_z, sigma_y) order, the sorted points of every
// source row that reaches it; the sorted order makes equal-cell lanes of a
// 32-point batch contiguous, and those are serialized by their rank in the
// cell, so shared-memory accumulation needs no atomics and the summation
// order is fixed (results are bitwise reproducible).  Each grid value is
// written to HBM exactly once, with coalesced stores.
template <typename TO>
__global__ void __launch_bounds__(kSpreadThreads) spread_tiles_kernel(
    DevGrid g, SpreadTiling T, const uint32_t* __restrict__ rowstart,
    const int* __restrict__ rec_cx, const double* __restrict__ rec, uint32_t n,
    TO* __restrict__ out) {
  extern __shared__ double s_acc[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  int b = blockIdx.x;
  const int bx = b % T.ntx;
  b /= T.ntx;
  const int by = b % T.nty;
  const int bz = b / T.nty;
  const int x0 = bx * T.tx, y0 = by * T.ty, z0 = bz * T.tz;
  const int rows = T.ty * T.tz;
  const int cells = rows * T.tx;
  for (int i = tid; i < cells; i += blockDim.x) s_acc[i] = 0.0;
  __syncthreads();

  const double* wy = rec + (size_t)4 * n;
  const double* wz = rec + (size_t)8 * n;
  // Shifts sigma = slo .. slo + s - 1 per axis (kernel.hpp:49-58); record
  // weight index sigma - slo.
  const int slo = g.slo, shi = g.slo + g.support - 1;
  const int szlo = g.dim >= 3 ? slo : 0, szhi = g.dim >= 3 ? shi : 0;
  const int sylo = g.dim >= 2 ? slo : 0, syhi = g.dim >= 2 ? shi : 0;
  const uint32_t le = lanemask_le();

  for (int tr = warp; tr < rows; tr += nwarps) {
    const int ty = y0 + tr % T.ty, tz = z0 + tr / T.ty;
    if (ty >= g.n[1] || tz >= g.n[2]) continue;
    double* acc = s_acc + (size_t)tr * T.tx;
    for (int sz = szlo; sz <= szhi; ++sz) {
      int cz = 0;
      if (g.dim >= 3) {
        cz = tz - sz;
        if (g.periodic[2]) cz = wrap_cell(cz, g.n[2]);
        else if (cz < -1 || cz > g.n[2]) continue;
      }
      for (int sy = sylo; sy <= syhi; ++sy) {
        int cy = 0;
        if (g.dim >= 2) {
          cy = ty - sy;
          if (g.periodic[1]) cy = wrap_cell(cy, g.n[1]);
          else if (cy < -1 || cy > g.n[1]) continue;
        }
        const uint32_t row = (g.dim >= 2 ? (uint32_t)(cy + 1) : 0u) +
                             (g.dim >= 3 ? (uint32_t)(cz + 1) * (uint32_t)(g.n[1] + 2) : 0u);
        const uint32_t rb = __ldg(rowstart + row), re = __ldg(rowstart + row + 1);
        const double* wyc = wy + (size_t)(sy - slo) * n;
        const double* wzc = wz + (size_t)(sz - slo) * n;
        for (uint32_t base = rb; base < re; base += 32) {
          const uint32_t r = base + lane;
          const bool valid = r < re;
          int cx = 0x7fffffff;
          double a = 0.0, gk[4] = {0.0, 0.0, 0.0, 0.0};
          if (valid) {
            cx = __ldg(rec_cx + r);
            a = __ldg(wyc + r) * __ldg(wzc + r);
#pragma unroll
            for (int k = 0; k < 4; ++k) gk[k] = __ldg(rec + (size_t)k * n + r);
          }
          const int pcx = __shfl_up_sync(0xffffffffu, cx, 1);
          const bool head = valid && (lane == 0 || pcx != cx);
          const uint32_t hm = __ballot_sync(0xffffffffu, head);
          const int rank = valid ? lane - (31 - __clz(hm & le)) : 0;
          const int maxrank = __reduce_max_sync(0xffffffffu, (unsigned)rank);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            int xt = cx + k + slo;
            bool ok = valid && k < g.support;
            if (g.periodic[0]) xt = wrap_cell(xt, g.n[0]);
            else ok = ok && xt >= 0 && xt < g.n[0];
            xt -= x0;
            ok = ok && xt >= 0 && xt < T.tx;
            const double v = gk[k] * a;
            for (int rr = 0; rr <= maxrank; ++rr) {
              if (ok && rank == rr) acc[xt] += v;
              __syncwarp();
            }
          }
        }
      }
    }
  }
  __syncthreads();
  const int64_t sy_ = g.n[0], sz_ = (int64_t)g.n[0] * g.n[1];
  for (int i = tid; i < cells; i += blockDim.x) {
    const int tr = i / T.tx, xx = i - tr * T.tx;
    const int ty = y0 + tr % T.ty, tz = z0 + tr / T.ty, x = x0 + xx;
    if (ty < g.n[1] && tz < g.n[2] && x < g.n[0]) out[tz * sz_ + ty * sy_ + x] = (TO)s_acc[i];
  }
}

// ---------------------------------------------------------------- K5
// One thread per point, visited in sorted (cell) order so neighbouring
// threads gather neighbouring grid values; result stored at the point's
// input slot.  Summation order over the 4^d support is the reference's
// colexicographic shift order (interpolate.hpp:42-52).
template <typename TF>
__global__ void __launch_bounds__(kBlock) interp_kernel(DevGrid g, const TF* __restrict__ field,
                                                        const double* __restrict__ X,
                                                        const uint32_t* __restrict__ perm, uint32_t n,
                                                        TF* __restrict__ out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const uint32_t i = perm ? __ldg(perm + r) : r;
  const int D = g.dim;
  constexpr int64_t kInvalid = INT64_MIN / 4;  // support_window.hpp:15-16
  double w[3][4];
  int64_t off[3][4];
  int64_t stride = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (a < D) {
      double xw;
      const int c = cell_of(g, a, __ldg(X + (size_t)i * D + a), &xw);
      kernel_weights(g, displacement(g, a, xw, c), w[a]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int cc = c + k + g.slo;
        if (g.periodic[a]) off[a][k] = stride * wrap_cell(cc, g.n[a]);
        else off[a][k] = (cc < 0 || cc >= g.n[a]) ? kInvalid : stride * cc;
      }
      stride *= g.n[a];
    } else {
      unit_weights(w[a], g.slo);
#pragma unroll
      for (int k = 0; k < 4; ++k) off[a][k] = 0;
    }
  }
  // Weight indices 0 .. s-1; a padded axis contributes only sigma = 0.
  const int s1 = g.support - 1, k0 = -g.slo;
  const int zlo = D >= 3 ? 0 : k0, zhi = D >= 3 ? s1 : k0;
  const int ylo = D >= 2 ? 0 : k0, yhi = D >= 2 ? s1 : k0;
  double acc = 0.0;
#pragma unroll
  for (int kz = 0; kz < 4; ++kz) {
    if (kz < zlo || kz > zhi) continue;
#pragma unroll
    for (int ky = 0; ky < 4; ++ky) {
      if (ky < ylo || ky > yhi) continue;
      const int64_t oyz = off[1][ky] + off[2][kz];
#pragma unroll
      for (int kx = 0; kx < 4; ++kx) {
        const int64_t o = off[0][kx] + oyz;
        if (kx <= s1 && o >= 0) {
          const double wt = (w[0][kx] * w[1][ky]) * w[2][kz];
          acc += wt * (double)__ldg(field + o);
        }
      }
    }
  }
  out[i] = (TF)(acc * g.hd);
}

// ---------------------------------------------------------------- run keys
__global__ void __launch_bounds__(kBlock) head_count_kernel(const uint32_t* __restrict__ sk, uint32_t n,
                                                            uint32_t* __restrict__ counts) {
  __shared__ uint32_t s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool head = i < n && (i == 0 || sk[i] != sk[i - 1]);
  const uint32_t hb = __ballot_sync(0xffffffffu, head);
  if ((threadIdx.x & 31) == 0) atomicAdd(&s, (uint32_t)__popc(hb));
  __syncthreads();
  if (threadIdx.x == 0) counts[blockIdx.x] = s;
}

__global__ void __launch_bounds__(sort::kThreads) block_scan_kernel(uint32_t* counts, uint32_t nb,
                                                                   uint32_t* q_out) {
  __shared__ uint32_t s_warp[sort::kWarps];
  __shared__ uint32_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += sort::kThreads) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < nb ? counts[i] : 0u;
    const uint32_t ex = sort::block_exclusive_scan(v, s_warp);
    const uint32_t carry = s_carry;
    if (i < nb) counts[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == sort::kThreads - 1) s_carry = carry + ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *q_out = s_carry;
}

__global__ void __launch_bounds__(kBlock) head_write_kernel(const uint32_t* __restrict__ sk, uint32_t n,
                                                            const uint32_t* __restrict__ offsets,
                                                            uint32_t* __restrict__ run_keys) {
  __shared__ uint32_t s_w[kBlock / 32];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool head = i < n && (i == 0 || sk[i] != sk[i - 1]);
  const uint32_t hb = __ballot_sync(0xffffffffu, head);
  if (lane == 0) s_w[warp] = __popc(hb);
  __syncthreads();
  uint32_t base = offsets[blockIdx.x];
  for (int w = 0; w < warp; ++w) base += s_w[w];
  if (head) run_keys[base + __popc(hb & ((1u << lane) - 1u))] = sk[i];
}

int bits_for(uint64_t max_key) {
  int bits = 1;
  while (bits < 32 && (max_key >> bits) != 0) ++bits;
  return bits;
}

// Bits of the largest cell key (row_only: of the largest extended row id).
int key_bits(const DevGrid& g, bool row_only) {
  uint64_t ext = 1;
  for (int a = row_only ? 1 : 0; a < g.dim; ++a) ext *= (uint64_t)g.n[a] + 2;
  return bits_for(ext - 1);
}

inline unsigned grid_for(size_t n, int block) { return (unsigned)((n + block - 1) / block); }

size_t sort_smem() { return sizeof(sort::PassSmem); }

// Sort scratch (s.hist): gcount[kMaxPasses][kMaxRadix] | offsets [ntiles][kMaxRadix] |
// per-pass tile counts [kMaxPasses][ntiles][kMaxRadix].
constexpr size_t kOffOff = (size_t)sort::kMaxPasses * sort::kMaxRadix;

// Keys + stable sort.  Leaves s.sorted_keys / s.sorted_perm (and, with a
// payload, s.rec: 32-byte sorted records).  row_only sorts by extended row id
// alone (enough for the interpolation's row grouping).
void sort_points(Context& ctx, const DevGrid& g, const double* d_points, size_t n, PointScratch& s,
                 bool row_only, int payload = sort::kPayloadNone,
                 const double* d_values = nullptr) {
  cudaStream_t st = ctx.stream;
  const sort::DigitPlan plan = sort::plan_digits(key_bits(g, row_only));
  const int ntiles = (int)((n + sort::kTile - 1) / sort::kTile);
  const size_t table = (size_t)ntiles * sort::kMaxRadix;
  uint32_t* gcount = s.hist.p;
  uint32_t* offs = s.hist.p + kOffOff;
  auto cnt = [&](int p) { return s.hist.p + kOffOff + table * (size_t)(1 + p); };
  IBC_CUDA(cudaMemsetAsync(gcount, 0, kOffOff * 4, st));
  if (plan.passes > 1)
    IBC_CUDA(cudaMemsetAsync(cnt(1), 0, table * (size_t)(plan.passes - 1) * 4, st));

  static bool attr_set[64] = {};
  if (!attr_set[ctx.device & 63]) {
    const int sm = (int)sort_smem();
    IBC_CUDA(cudaFuncSetAttribute(sort::onesweep_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    IBC_CUDA(cudaFuncSetAttribute(sort::onesweep_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    IBC_CUDA(cudaFuncSetAttribute(sort::onesweep_pass<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    IBC_CUDA(cudaFuncSetAttribute(sort::onesweep_pass<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    attr_set[ctx.device & 63] = true;
  }

  cudaEvent_t ev = nullptr;
  ctx.prof_begin(kProfKeys, &ev);
  const int ro = row_only ? 1 : 0;
  KeyDigits kd{};
  kd.passes = plan.passes;
  for (int p = 0; p < plan.passes; ++p) {
    kd.shift[p] = plan.shift[p];
    kd.bits[p] = plan.bits[p];
  }
  if (g.dim == 3)
    keys_hist_kernel<3><<<ntiles, kKeysThreads, 0, st>>>(g, d_points, (uint32_t)n, s.keys[0].p,
                                                         gcount, cnt(0), kd, ro);
  else if (g.dim == 2)
    keys_hist_kernel<2><<<ntiles, kKeysThreads, 0, st>>>(g, d_points, (uint32_t)n, s.keys[0].p,
                                                         gcount, cnt(0), kd, ro);
  else
    keys_hist_kernel<1><<<ntiles, kKeysThreads, 0, st>>>(g, d_points, (uint32_t)n, s.keys[0].p,
                                                         gcount, cnt(0), kd, ro);
  ++ctx.launches;
  ctx.prof_end(kProfKeys, ev);

  ctx.prof_begin(kProfSort, &ev);
  int src = 0;
  for (int p = 0; p < plan.passes; ++p) {
    const bool last = p + 1 == plan.passes;
    const int pl = last ? payload : sort::kPayloadNone;
    const int radix = 1 << plan.bits[p];
    sort::tile_offsets_kernel<<<(radix + 31) / 32, sort::kThreads, 0, st>>>(
        cnt(p), offs, gcount + (size_t)p * sort::kMaxRadix, radix, ntiles);
    auto args = [&](auto kern) {
      kern<<<ntiles, sort::kThreads, sort_smem(), st>>>(
          s.keys[src].p, p == 0 ? nullptr : s.vals[src].p, s.keys[src ^ 1].p, s.vals[src ^ 1].p,
          (uint32_t)n, plan.shift[p], plan.bits[p], offs, last ? nullptr : cnt(p + 1),
          last ? 0 : plan.shift[p + 1], last ? 1 : plan.bits[p + 1], d_points, d_values, s.rec.p,
          g, s.rec_cx.p);
    };
    if (pl == sort::kPayloadWeights) args(sort::onesweep_pass<sort::kPayloadWeights>);
    else if (pl == sort::kPayloadSpread) args(sort::onesweep_pass<sort::kPayloadSpread>);
    else if (pl == sort::kPayloadInterp) args(sort::onesweep_pass<sort::kPayloadInterp>);
    else args(sort::onesweep_pass<sort::kPayloadNone>);
    ctx.launches += 2;
    src ^= 1;
  }
  ctx.prof_end(kProfSort, ev);
  IBC_CUDA(cudaGetLastError());
  s.sorted_keys = s.keys[src].p;
  s.sorted_perm = s.vals[src].p;
  s.last_n = n;
  s.run_keys_valid = false;
  s.keys_are_rows = row_only;
  s.obs_pending = false;  // the sorted keys / perm are current
}

void row_table(Context& ctx, const DevGrid& g, size_t n, PointScratch& s) {
  cudaStream_t st = ctx.stream;
  cudaEvent_t ev = nullptr;
  ctx.prof_begin(kProfRows, &ev);
  if (n == 0) {
    IBC_CUDA(cudaMemsetAsync(s.rowstart.p, 0, ((size_t)g.nrows + 1) * 4, st));
  } else {
    rowstart_kernel<<<grid_for(n, kBlock), kBlock, 0, st>>>(
        s.sorted_keys, (uint32_t)n, s.keys_are_rows ? 1u : g.rowdiv, g.nrows, s.rowstart.p);
    ++ctx.launches;
  }
  ctx.prof_end(kProfRows, ev);
}

SpreadTiling choose_tiling(const DevGrid& g) {
  // Target tile: whole x rows when they fit (periodic x then wraps inside the
  // tile), times ty x tz rows, <= 64 KB of doubles in shared memory.
  SpreadTiling T;
  const int n0 = g.n[0];
  T.tx = n0 <= 4096 ? n0 : 2048;
  const int rows_budget = std::max(1, (64 * 1024 / 8) / T.tx);
  int ty = 1, tz = 1;
  if (g.dim >= 3) {
    if (rows_budget >= 16) { ty = 4; tz = 4; }
    else if (rows_budget >= 8) { ty = 4; tz = 2; }
    else if (rows_budget >= 4) { ty = 2; tz = 2; }
    else if (rows_budget >= 2) { ty = 2; tz = 1; }
  } else if (g.dim == 2) {
    ty = std::min(rows_budget, 16);
  }
  ty = std::max(1, std::min(ty, g.n[1]));
  tz = std::max(1, std::min(tz, g.n[2]));
  T.ty = ty;
  T.tz = tz;
  T.ntx = (n0 + T.tx - 1) / T.tx;
  T.nty = (g.n[1] + ty - 1) / ty;
  T.ntz = (g.n[2] + tz - 1) / tz;
  return T;
}

}  // namespace

DevGrid make_devgrid(const ibc_grid& gi, int kernel) {
  DevGrid g{};
  g.dim = gi.dim;
  g.kernel = kernel;
  g.support = kernel_support(kernel);
  g.slo = -(g.support / 2);
  g.half = (g.support % 2 == 0) ? 0.0 : 0.5;
  g.h = gi.spacing;
  g.inv_h = 1.0 / gi.spacing;
  uint64_t ks = 1;
  g.npts = 1;
  for (int a = 0; a < 3; ++a) {
    if (a < gi.dim) {
      g.n[a] = gi.extent[a];
      g.periodic[a] = gi.periodic[a] ? 1 : 0;
      g.alpha[a] = gi.staggering[a];
      g.origin[a] = gi.origin[a];
      g.len[a] = gi.extent[a] * gi.spacing;
      g.kstride[a] = ks;
      ks *= (uint64_t)gi.extent[a] + 2;
      g.npts *= gi.extent[a];
    } else {
      g.n[a] = 1;
      g.periodic[a] = 0;
      g.alpha[a] = 0.0;
      g.origin[a] = 0.0;
      g.len[a] = gi.spacing;
      g.kstride[a] = 0;
    }
  }
  g.rowdiv = (uint32_t)(g.n[0] + 2);
  g.nrows = 1;
  for (int a = 1; a < gi.dim; ++a) g.nrows *= (uint32_t)(g.n[a] + 2);
  g.hd = std::pow(gi.spacing, (double)gi.dim);
  return g;
}

DevGrid make_devgrid(const ibc_grid& gi, const ibc_slab& slab, int kernel) {
  DevGrid g = make_devgrid(gi, kernel);
  const int a = gi.dim - 1;
  g.zslab = 1;
  g.zfirst = slab.z_first;
  g.zg_n = slab.nz_global;
  g.zg_periodic = slab.periodic_global ? 1 : 0;
  g.zg_len = slab.nz_global * gi.spacing;  // axis_length of the global grid (grid.hpp:72)
  g.periodic[a] = 0;
  return g;
}

namespace {
__global__ void __launch_bounds__(kBlock) home_planes_kernel(DevGrid g, const double* __restrict__ X,
                                                             uint32_t n, int* __restrict__ planes) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = g.dim - 1;
  double xw;
  int c = cell_of(g, a, __ldg(X + (size_t)i * g.dim + a), &xw);
  if (g.periodic[a]) c = wrap_cell(c, g.n[a]);
  planes[i] = c;
}
}  // namespace

void home_planes(Context& ctx, const DevGrid& g, const double* d_points, size_t n, int* d_planes) {
  if (n == 0) return;
  home_planes_kernel<<<grid_for(n, kBlock), kBlock, 0, ctx.stream>>>(g, d_points, (uint32_t)n,
                                                                      d_planes);
  ++ctx.launches;
  IBC_CUDA(cudaGetLastError());
}

void PointScratch::reserve_points(size_t n, bool spread) {
  const size_t tiles = (n + sort::kTile - 1) / sort::kTile;
  for (int b = 0; b < 2; ++b) {
    keys[b].ensure(n);
    vals[b].ensure(n);
  }
  hist.ensure(kOffOff + (size_t)(kMaxPasses + 1) * sort::kMaxRadix * std::max<size_t>(tiles, 1));
  base.ensure((size_t)kMaxPasses * sort::kMaxRadix);
  counters.ensure(kCounters);
  rec.ensure(12 * std::max<size_t>(n, 1));  // 12 doubles (V1 weights) or 4 (sorted records)
  if (spread) rec_cx.ensure(n);
  cap = std::max(cap, n);
}

void PointScratch::reserve_rows(size_t nrows) { rowstart.ensure(nrows + 1); }

void PointScratch::release_all() {
  for (int b = 0; b < 2; ++b) {
    keys[b].release();
    vals[b].release();
  }
  hist.release(); base.release(); counters.release(); rowstart.release();
  rec_cx.release(); rec.release(); run_keys.release(); block_counts.release(); rowaux.release();
  bpair.release();
  bpair_tmp.release();
  prim_u32.release();
  prim_bytes.release();
  cap = 0;
}

namespace {
void bucket_points(Context& ctx, const DevGrid& g, const double* d_points, const double* d_values,
                   size_t n, PointScratch& s, bool spread);

// Tiling of the write-once spread sweep (ibc_spread.cuh), 2-D and 3-D grids.
// rows_per_warp = 1: pull mode (wpc warps per CTA, one target row each);
// > 1: bank mode (one warp per CTA, bucket::kRowsPerWarp target rows).
bool sweep_tiling(const DevGrid& g, int sms, uint32_t pull_row, sp::SweepTiling& T,
                  int rows_per_warp) {
  if (g.dim < 2) return false;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int rl = sp::row_len(nx);
  const int slots = g.dim == 3 ? 4 : 1;
  const size_t per_warp = (size_t)rows_per_warp * slots * rl * sizeof(double);
  if (per_warp > 200 * 1024) return false;
  // Warps per CTA: bank mode one (its kernel is __launch_bounds__(32)); pull
  // mode the CTA size (<= 8 warps) that keeps the most warps resident per SM
  // under the window (shared memory) and register (__launch_bounds__(256, 3):
  // 24 warps) limits -- long x rows need small CTAs to fill an SM.
  int wpc = 1;
  if (rows_per_warp == 1) {
    long best = 0;
    for (int w = 8; w >= 1; --w) {
      if ((size_t)w * per_warp > 200 * 1024) continue;
      const long ctas = std::min<long>(32, (227L * 1024) / (long)(w * per_warp));
      const long warps = std::min<long>(24, (long)w * ctas);
      if (warps >= best) {  // ties: smaller CTAs (finer load balance across SMs)
        best = warps;
        wpc = w;
      }
    }
  }
  T.wpc = wpc;
  T.rl = rl;
  T.pull_row = pull_row;
  T.group = bucket::kBanks;
  const int rows_per_cta = wpc * rows_per_warp;
  T.nyg = (ny + rows_per_cta - 1) / rows_per_cta;
  if (g.dim == 3) {
    const long max_warps = rows_per_warp == 1 ? 24 : 16;  // registers / __launch_bounds__
    const long per_sm = std::max<long>(
        1, std::min<long>(std::min<long>(max_warps / wpc, 32), (227L * 1024) / (long)(wpc * per_warp)));
    const long chunks = std::max<long>(1, ((long)sms * per_sm) / T.nyg);
    T.zc = (int)std::max<long>(1, (nz + chunks - 1) / chunks);
    T.nzc = (nz + T.zc - 1) / T.zc;
  } else {
    T.zc = T.nzc = 1;
  }
  return true;
}
}  // namespace

template <typename TO>
void spread_pipeline(Context& ctx, const DevGrid& g, const double* d_points, const double* d_values,
                     size_t n, PointScratch& s, TO* d_out) {
  cudaStream_t st = ctx.stream;
  sp::SweepTiling W, WB;  // pull mode, bank mode
  // Bank-mode row threshold: AUTO -- rows up to kPullRow (and crowded
  // buckets); BANK -- every row; PULL / RADIX -- none.
  const int path = ctx.spread_path;
  const uint32_t pull_row = path == IBC_SPREAD_PATH_BANK ? 0xfffffffeu
                            : (path == IBC_SPREAD_PATH_PULL || path == IBC_SPREAD_PATH_RADIX)
                                ? bucket::kNoBankMode
                                : sp::kPullRow;
  // The sweeps take the 4-point kernels (their records carry one weight pair
  // per axis, ibc_device.cuh kernel_pair); other supports run the generic
  // radix-sort + tiled path.
  const bool sweep = g.support == kSupport && sweep_tiling(g, ctx.sms, pull_row, W, 1);
  if (!sweep_tiling(g, ctx.sms, pull_row, WB, bucket::kRowsPerWarp)) {  // bank window too large
    WB = W;
    W.pull_row = WB.pull_row = bucket::kNoBankMode;
  }
  s.bank_rows = W.pull_row;
  const bool radix = path == IBC_SPREAD_PATH_RADIX;
  if (sweep && !radix) {
    bucket_points(ctx, g, d_points, d_values, n, s, true);
  } else {
    if (n > 0) {
      sort_points(ctx, g, d_points, n, s, false, sweep ? sort::kPayloadWeights : sort::kPayloadNone,
                  d_values);
    } else {
      s.last_n = 0;
      s.sorted_keys = s.keys[0].p;
      s.sorted_perm = s.vals[0].p;
      s.run_keys_valid = false;
      s.keys_are_rows = false;
    }
    row_table(ctx, g, n, s);
    W.group = WB.group = 1;  // one row-start entry per row
  }
  cudaEvent_t ev = nullptr;
  static bool attr_set[64] = {};
  if (!attr_set[ctx.device & 63]) {
    IBC_CUDA(cudaFuncSetAttribute(spread_tiles_kernel<TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  160 * 1024));
    for (const void* k :
         {(const void*)sp::spread_sweep_kernel<2, 0, TO>, (const void*)sp::spread_banks_kernel<2, 0, TO>,
          (const void*)sp::spread_sweep_kernel<3, 0, TO>, (const void*)sp::spread_banks_kernel<3, 0, TO>,
          (const void*)sp::spread_sweep_kernel<3, sp::row_len(64), TO>,
          (const void*)sp::spread_banks_kernel<3, sp::row_len(64), TO>,
          (const void*)sp::spread_sweep_kernel<3, sp::row_len(128), TO>,
          (const void*)sp::spread_banks_kernel<3, sp::row_len(128), TO>,
          (const void*)sp::spread_sweep_kernel<3, sp::row_len(256), TO>,
          (const void*)sp::spread_banks_kernel<3, sp::row_len(256), TO>,
          (const void*)sp::spread_sweep_kernel<3, sp::row_len(512), TO>,
          (const void*)sp::spread_banks_kernel<3, sp::row_len(512), TO>})
      IBC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_set[ctx.device & 63] = true;
  }
  if (sweep) {
    ctx.prof_begin(kProfSpread, &ev);
    const size_t smem = (size_t)W.wpc * (g.dim == 3 ? 4 : 1) * W.rl * sizeof(double);
    const size_t smem_b =
        (size_t)bucket::kRowsPerWarp * WB.wpc * (g.dim == 3 ? 4 : 1) * WB.rl * sizeof(double);
    const unsigned blocks = (unsigned)(W.nyg * W.nzc), blocks_b = (unsigned)(WB.nyg * WB.nzc);
    // Compile-time window row length for the common x extents; both modes
    // are launched when the densest row is only known on the device.
    const uint32_t* maxrow = (!radix) ? s.maxrow : nullptr;
    auto launch = [&](auto bank_k, auto pull_k) {
      if (maxrow && WB.pull_row != bucket::kNoBankMode) {
        pdl_launch(bank_k, blocks_b, 32 * WB.wpc, smem_b, st, g, WB, maxrow, s.rowstart.p, s.rec.p,
                                                      s.rec_cx.p, d_out);
        ++ctx.launches;
      }
      pdl_launch(pull_k, blocks, 32 * W.wpc, smem, st, g, W, maxrow, s.rowstart.p, s.rec.p,
                                               s.rec_cx.p, d_out);
    };
    const int nx = g.n[0];
#define IBC_SWEEP(D, RL) launch(sp::spread_banks_kernel<D, RL, TO>, sp::spread_sweep_kernel<D, RL, TO>)
    if (g.dim == 3) {
      if (nx == 64) IBC_SWEEP(3, sp::row_len(64));
      else if (nx == 128) IBC_SWEEP(3, sp::row_len(128));
      else if (nx == 256) IBC_SWEEP(3, sp::row_len(256));
      else if (nx == 512) IBC_SWEEP(3, sp::row_len(512));
      else IBC_SWEEP(3, 0);
    } else {
      IBC_SWEEP(2, 0);
    }
#undef IBC_SWEEP
    ++ctx.launches;
    ctx.prof_end(kProfSpread, ev);
  } else {
    if (n > 0) {
      ctx.prof_begin(kProfPrep, &ev);
      prep_records_kernel<<<grid_for(n, kBlock), kBlock, 0, st>>>(
          g, d_points, d_values, s.sorted_perm, (uint32_t)n, s.rec_cx.p, s.rec.p);
      ++ctx.launches;
      ctx.prof_end(kProfPrep, ev);
    }
    const SpreadTiling T = choose_tiling(g);
    const size_t smem = (size_t)T.tx * T.ty * T.tz * sizeof(double);
    ctx.prof_begin(kProfSpread, &ev);
    const unsigned blocks = (unsigned)((size_t)T.ntx * T.nty * T.ntz);
    spread_tiles_kernel<TO><<<blocks, kSpreadThreads, smem, st>>>(g, T, s.rowstart.p, s.rec_cx.p,
                                                                  s.rec.p, (uint32_t)n, d_out);
    ++ctx.launches;
    ctx.prof_end(kProfSpread, ev);
  }
  IBC_CUDA(cudaGetLastError());
  ++ctx.spread_calls;
}
namespace {
__global__ void __launch_bounds__(kBlock) widen_kernel(const float* __restrict__ in, size_t m,
                                                       double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)kBlock + threadIdx.x; i < m; i += (size_t)gridDim.x * kBlock)
    out[i] = (double)__ldg(in + i);
}
}  // namespace

const double* widen(Context& ctx, const float* d_in, size_t m, DevBuf<double>& buf) {
  buf.ensure(m);
  if (m) {
    const unsigned blocks = (unsigned)std::min<size_t>((m + kBlock - 1) / kBlock, (size_t)ctx.sms * 8);
    widen_kernel<<<blocks, kBlock, 0, ctx.stream>>>(d_in, m, buf.p);
    ++ctx.launches;
    IBC_CUDA(cudaGetLastError());
  }
  return buf.p;
}

template void spread_pipeline<double>(Context&, const DevGrid&, const double*, const double*, size_t,
                                      PointScratch&, double*);
template void spread_pipeline<float>(Context&, const DevGrid&, const double*, const double*, size_t,
                                     PointScratch&, float*);

namespace {

// Tiling of the TMA interpolation sweep (3-D, nx % 16 == 0, nx <= 4096).
// elem: bytes per field value (8, or 4 in the FP32 storage mode).
bool interp_tma_tiling(const DevGrid& g, size_t n, int sms, sw::InterpTiling& T, int elem = 8) {
  if (g.dim != 3) return false;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  if (nx % 16 != 0 || nx > 4096) return false;
  const uint32_t pitch = (uint32_t)((nx * elem + 1023) & ~1023);
  // Pick TY (home rows per CTA) minimising the bytes one SM streams, with at
  // least 3 planes in flight (slots >= 7) when possible and one CTA per SM.
  double best = 1e300;
  bool found = false;
  for (int ty = 1; ty <= std::min(ny, 32); ++ty) {
    const int nty = (ny + ty - 1) / ty;
    const int ghosts = g.periodic[1] ? 0 : (nty == 1 ? 2 : 1);
    const int fr = ty + 3 + ghosts;
    const long chunks = std::max<long>(1, sms / nty);
    int zc = (int)std::max<long>(4, (nz + chunks - 1) / chunks);
    zc = std::min(zc, nz);
    const int hmax = zc + 2;
    // Records staged per step: 0.9 x the mean points per step, 64..1024 (a
    // step's overflow is read from global memory; smaller stages leave room
    // for taller tiles -- less field re-read -- and a deeper ring).
    const double mean = (double)n * (ty + ghosts) / ((double)(ny + 2) * (nz + 2));
    int cap = (int)std::min(1024.0, std::max(64.0, 0.9 * mean));
    cap = (cap + 31) & ~31;
    const uint32_t stride = (uint32_t)(((size_t)fr * pitch + (size_t)cap * 64 + 1023) & ~size_t(1023));
    const size_t budget = 226 * 1024 - 16 * sw::kMaxSlots - 12 * (size_t)hmax - 1024;
    const int slots = (int)std::min<size_t>(sw::kMaxSlots, budget / stride);
    if (slots < 5) continue;
    const long ctas = (long)nty * ((nz + zc - 1) / zc);
    const long waves = (ctas + sms - 1) / sms;
    double cost = (double)waves * (zc + 3) * fr;
    if (slots < 7) cost *= 1.0 + 0.15 * (7 - slots);  // shallow ring: exposed TMA latency
    if (cost < best) {
      best = cost;
      found = true;
      T.ty = ty;
      T.frmax = fr;
      T.slots = slots;
      T.nty = nty;
      T.zc = zc;
      T.nzc = (nz + zc - 1) / zc;
      T.rec_cap = cap;
      T.hmax = hmax;
      T.slot_stride = stride;
    }
  }
  if (!found) return false;
  T.pitch = pitch;
  T.slot_bytes = (uint32_t)T.frmax * pitch;
  T.box_ok = (nx * elem) % 1024 == 0 ? 1 : 0;  // box rows land at the slot pitch (1024-byte multiple)
  return true;
}

size_t interp_tma_smem(const sw::InterpTiling& T) {
  return 16 * sw::kMaxSlots + 12 * (size_t)T.hmax + 1024 + (size_t)T.slots * T.slot_stride;
}

}  // namespace

namespace tma {
bool encode_rows_map(CUtensorMap* map, const void* field, int elem, int nx, int ny, int nz,
                     int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        !p)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  if (reinterpret_cast<uintptr_t>(field) % 16 != 0) return false;
  const cuuint64_t e = (cuuint64_t)elem;
  const cuuint64_t dims[4] = {16, (cuuint64_t)(nx / 16), (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t strides[3] = {16 * e, (cuuint64_t)nx * e, (cuuint64_t)nx * ny * e};
  const cuuint32_t box[4] = {16, (cuuint32_t)(nx / 16), (cuuint32_t)box_rows, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(map, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
            const_cast<void*>(field), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tma

namespace {
// K3 over the spread buckets.
void launch_scatter_spread(Context& ctx, const DevGrid& g, size_t n, PointScratch& s) {
  pdl_launch(bucket::scatter_spread_kernel, grid_for(n, bucket::kThreads), bucket::kThreads, 0, ctx.stream, 
      s.keys[1].p, s.vals[1].p, (uint32_t)n, g.rowdiv, g.nrows, s.rowstart.p, s.bpair.p);
  ++ctx.launches;
}

// K4 / K4b over the spread buckets: mode 0 inside the spread (pull mode:
// sorted pairs + records), mode 1 on request (sorted pairs only).
void launch_row_sorts(Context& ctx, const DevGrid& g, const double* d_points,
                      const double* d_values, size_t n, PointScratch& s, int mode) {
  cudaStream_t st = ctx.stream;
  const uint32_t* maxrow = s.maxrow;
  uint32_t* nlong = const_cast<uint32_t*>(maxrow) - 1;
  const uint32_t* long_rows = maxrow + 4;
  static bool attr_set[64] = {};
  const size_t lsm = (size_t)bucket::kLongSortMax * 8;
  if (!attr_set[ctx.device & 63]) {
    IBC_CUDA(cudaFuncSetAttribute(bucket::long_row_sort_kernel<2>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    IBC_CUDA(cudaFuncSetAttribute(bucket::long_row_sort_kernel<3>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm));
    attr_set[ctx.device & 63] = true;
  }
  auto sorts = [&](auto short_k, auto long_k) {
    pdl_launch(short_k, grid_for(n, bucket::kThreads), bucket::kThreads, 0, st, 
        s.rowstart.p, (uint32_t)n, s.bpair.p, s.keys[0].p, s.vals[0].p, g, d_points, d_values,
        s.rec.p, s.rec_cx.p, maxrow, s.bank_rows, mode);
    pdl_launch(long_k, (unsigned)ctx.sms, bucket::kLongThreads, lsm, st, s.rowstart.p, long_rows, nlong, s.bpair.p,
                                                   s.keys[0].p, s.vals[0].p, g, d_points,
                                                   d_values, s.rec.p, s.rec_cx.p, maxrow,
                                                   s.bank_rows, mode, s.bpair_tmp.p,
                                                   s.bpair_tmp.p + s.bpair_tmp_half);
  };
  if (g.dim == 3) sorts(bucket::row_sort_kernel<3>, bucket::long_row_sort_kernel<3>);
  else sorts(bucket::row_sort_kernel<2>, bucket::long_row_sort_kernel<2>);
  ctx.launches += 2;
}

// Bucket sort (ibc_bucket.cuh).  Interpolation: records grouped by row.
// Spread: points bucketed by (row, x bank); in bank mode the weight records
// are written straight into the buckets, in pull mode K4 puts them in the
// rows' key order.  The stable (key, index) order the reference exposes as
// ws.keys / ws.perm is materialised on request (ensure_observables).
void bucket_points(Context& ctx, const DevGrid& g, const double* d_points, const double* d_values,
                   size_t n, PointScratch& s, bool spread) {
  cudaStream_t st = ctx.stream;
  const uint32_t nrows = g.nrows + 1;  // + the row of points homed outside (K1)
  const int group = spread ? bucket::kBanks : 1;     // buckets per grid row
  const uint32_t nb = nrows * (uint32_t)group;       // buckets
  const uint32_t chunk = bucket::kScanThreads * (spread ? bucket::kBanks : bucket::kScanItems);
  const uint32_t nchunks = (nb + chunk - 1) / chunk;
  s.rowaux.ensure((size_t)nb + nchunks + 8 + nrows);
  s.rowstart.ensure((size_t)nb + 1);
  uint32_t* count = s.rowaux.p;
  uint32_t* status = count + nb;
  uint32_t* ticket = status + nchunks;
  uint32_t* nlong = ticket + 1;
  uint32_t* maxrow = nlong + 1;     // [densest row, fullest bucket]
  uint32_t* long_rows = maxrow + 4;
  IBC_CUDA(cudaMemsetAsync(count, 0, ((size_t)nb + nchunks + 6) * 4, st));
  s.maxrow = spread ? maxrow : nullptr;  // (zeroed above; set by the row scan)
  if (n == 0) {
    IBC_CUDA(cudaMemsetAsync(s.rowstart.p, 0, ((size_t)nb + 1) * 4, st));
    if (spread) {
      s.last_n = 0;
      s.obs_pending = false;
    }
    return;
  }
  cudaEvent_t ev = nullptr;
  ctx.prof_begin(kProfKeys, &ev);
  const unsigned blocks = grid_for(n, bucket::kThreads);
  const int full = spread ? 1 : 0;
  // Input-order keys and ranks: buffers 1 for the spread (buffers 0 receive
  // the sorted keys / permutation), 0 for interpolation.
  uint32_t* ikeys = s.keys[spread ? 1 : 0].p;
  uint32_t* irank = s.vals[spread ? 1 : 0].p;
  if (g.dim == 3)
    pdl_launch(bucket::keys_kernel<3>, blocks, bucket::kThreads, 0, st, g, d_points, (uint32_t)n, full, group,
                                                               ikeys, irank, count);
  else if (g.dim == 2)
    pdl_launch(bucket::keys_kernel<2>, blocks, bucket::kThreads, 0, st, g, d_points, (uint32_t)n, full, group,
                                                               ikeys, irank, count);
  else
    pdl_launch(bucket::keys_kernel<1>, blocks, bucket::kThreads, 0, st, g, d_points, (uint32_t)n, full, group,
                                                               ikeys, irank, count);
  ctx.prof_end(kProfKeys, ev);
  ctx.prof_begin(kProfSort, &ev);
  if (spread)
    pdl_launch(bucket::row_scan_kernel<bucket::kBanks>, nchunks, bucket::kScanThreads, 0, st, 
        count, s.rowstart.p, nb, group, status, ticket, long_rows, nlong, maxrow);
  else
    pdl_launch(bucket::row_scan_kernel<bucket::kScanItems>, nchunks, bucket::kScanThreads, 0, st, 
        count, s.rowstart.p, nb, group, status, ticket, nullptr, nlong, maxrow);
  ctx.launches += 2;
  if (!spread) {
    if (g.dim == 3)
      pdl_launch(bucket::scatter_interp_kernel<3>, blocks, bucket::kThreads, 0, st, 
          g, d_points, s.keys[0].p, s.vals[0].p, (uint32_t)n, s.rowstart.p, s.rec.p);
    else
      pdl_launch(bucket::scatter_interp_kernel<2>, blocks, bucket::kThreads, 0, st, 
          g, d_points, s.keys[0].p, s.vals[0].p, (uint32_t)n, s.rowstart.p, s.rec.p);
    ctx.launches += 1;
    s.last_n = 0;  // interpolation leaves no observable sort
  } else {
    s.bpair.ensure(n);
    // merge space of the very long rows (long_row_sort_kernel): 2 x n words
    s.bpair_tmp.ensure(2 * n);
    s.bpair_tmp_half = n;
    launch_scatter_spread(ctx, g, n, s);
    // Records: in (row, x bank) buckets (bank mode) or the rows' key order
    // (pull mode, K4b for the long rows; it exits at once in bank mode).
    launch_row_sorts(ctx, g, d_points, d_values, n, s, 0);
    s.sorted_keys = s.keys[0].p;
    s.sorted_perm = s.vals[0].p;
    s.last_n = n;
    s.obs_pending = true;
    s.obs_grid = g;
    s.run_keys_valid = false;
    s.keys_are_rows = false;
  }
  ctx.prof_end(kProfSort, ev);
  IBC_CUDA(cudaGetLastError());
}

}  // namespace

// Interpolation binning -- everything that depends on the points and the
// grid but not on the field, so one binning serves any number of fields at
// the same points (the reference's step interpolates twice at X^n,
// run.hpp:94-115): TMA path -- row bucket sort + 64-byte records (points
// homed outside the grid get their index in the extra row, zeroed by the
// gather); generic path -- the stable radix sort (permutation).
InterpPlan interp_bin(Context& ctx, const DevGrid& g, const double* d_points, size_t n,
                      PointScratch& s, bool allow_tma) {
  InterpPlan P;
  if (n == 0) return P;
  P.tma = allow_tma && g.support == kSupport && interp_tma_tiling(g, n, ctx.sms, P.T);
  if (P.tma) bucket_points(ctx, g, d_points, nullptr, n, s, false);
  else sort_points(ctx, g, d_points, n, s, false, sort::kPayloadNone);
  return P;
}

// The gather over a binning (d_points is read again on the generic path).
// The binning plans the TMA tiling for 8-byte values; FP32 fields retile
// (half the plane bytes: a 4-byte tiling exists whenever the 8-byte one does).
template <typename TF>
void interp_gather(Context& ctx, const DevGrid& g, const InterpPlan& P, const TF* d_field,
                   const double* d_points, size_t n, PointScratch& s, TF* d_out) {
  if (n == 0) return;
  cudaStream_t st = ctx.stream;
  cudaEvent_t ev = nullptr;
  if (P.tma) {
    sw::InterpTiling T = P.T;
    if (sizeof(TF) != 8 && !interp_tma_tiling(g, n, ctx.sms, T, (int)sizeof(TF)))
      throw ArgError{"no shared-memory tiling for this field"};
    CUtensorMap map, map_box;
    if (!tma::encode_rows_map(&map, d_field, (int)sizeof(TF), g.n[0], g.n[1], g.n[2]) ||
        !tma::encode_rows_map(&map_box, d_field, (int)sizeof(TF), g.n[0], g.n[1], g.n[2], T.frmax))
      throw ArgError{"field must be 16-byte aligned device memory"};
    const size_t smem = interp_tma_smem(T);
    static bool attr_set[64] = {};
    if (!attr_set[ctx.device & 63]) {
      IBC_CUDA(cudaFuncSetAttribute(sw::interp_tma_kernel<TF>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr_set[ctx.device & 63] = true;
    }
    ctx.prof_begin(kProfInterp, &ev);
    pdl_launch(sw::interp_tma_kernel<TF>, (unsigned)(T.nty * T.nzc), sw::kIThreads, smem, st, g, T,
               map, map_box, (const uint32_t*)s.rowstart.p, (const double*)s.rec.p, d_out);
  } else {
    // Generic gather (1-D/2-D grids, x extents the TMA rows do not take,
    // other supports): one thread per point in sorted order.
    ctx.prof_begin(kProfInterp, &ev);
    interp_kernel<TF><<<grid_for(n, kBlock), kBlock, 0, st>>>(g, d_field, d_points, s.sorted_perm,
                                                              (uint32_t)n, d_out);
  }
  ++ctx.launches;
  ctx.prof_end(kProfInterp, ev);
  IBC_CUDA(cudaGetLastError());
  ++ctx.interp_calls;
}

template <typename TF>
void interp_pipeline(Context& ctx, const DevGrid& g, const TF* d_field, const double* d_points,
                     size_t n, PointScratch& s, TF* d_out) {
  if (n == 0) return;
  // The TMA tensor maps need a 16-byte aligned field.
  const bool aligned = reinterpret_cast<uintptr_t>(d_field) % 16 == 0;
  const InterpPlan P = interp_bin(ctx, g, d_points, n, s, aligned);
  interp_gather(ctx, g, P, d_field, d_points, n, s, d_out);
}
template void interp_gather<double>(Context&, const DevGrid&, const InterpPlan&, const double*,
                                    const double*, size_t, PointScratch&, double*);
template void interp_gather<float>(Context&, const DevGrid&, const InterpPlan&, const float*,
                                   const double*, size_t, PointScratch&, float*);
template void interp_pipeline<double>(Context&, const DevGrid&, const double*, const double*, size_t,
                                      PointScratch&, double*);
template void interp_pipeline<float>(Context&, const DevGrid&, const float*, const double*, size_t,
                                     PointScratch&, float*);

// ws.run_keys and ws.run_count (= q) on the device, computed on demand from
// the sorted keys (reduce.hpp:36-69); cached until the next sort.
void ensure_observables(Context& ctx, PointScratch& s) {
  if (!s.obs_pending || !s.last_n) return;
  launch_row_sorts(ctx, s.obs_grid, nullptr, nullptr, s.last_n, s, 1);
  IBC_CUDA(cudaGetLastError());
  s.obs_pending = false;
  s.run_keys_valid = false;
}

size_t compute_run_keys(Context& ctx, PointScratch& s) {
  const size_t n = s.last_n;
  if (n == 0) return 0;
  ensure_observables(ctx, s);
  cudaStream_t st = ctx.stream;
  if (!s.run_keys_valid) {
    const unsigned nb = grid_for(n, kBlock);
    s.block_counts.ensure(nb);
    s.run_keys.ensure(n);
    head_count_kernel<<<nb, kBlock, 0, st>>>(s.sorted_keys, (uint32_t)n, s.block_counts.p);
    block_scan_kernel<<<1, sort::kThreads, 0, st>>>(s.block_counts.p, nb, s.counters.p + kMaxPasses);
    head_write_kernel<<<nb, kBlock, 0, st>>>(s.sorted_keys, (uint32_t)n, s.block_counts.p,
                                             s.run_keys.p);
    ctx.launches += 3;
    IBC_CUDA(cudaGetLastError());
    s.run_keys_valid = true;
  }
  uint32_t q = 0;
  IBC_CUDA(cudaMemcpyAsync(&q, s.counters.p + kMaxPasses, 4, cudaMemcpyDeviceToHost, st));
  IBC_CUDA(cudaStreamSynchronize(st));
  return q;
}

size_t read_run_count(Context& ctx, PointScratch& s) { return compute_run_keys(ctx, s); }

// ---------------------------------------------------------------- primitives
// ib::key_value_sort (sort.hpp:16-71), ib::count_unique (reduce.hpp:57-69)
// and ib::segmented_reduce(_rows) (reduce.hpp:80-145) on the device, for
// callers of the reference's primitive API (the operators above never call
// them: their sort and reduction are fused into the bucket sort and sweeps).
namespace {

// Digit histograms of every pass over raw 32-bit keys (keys_hist_kernel
// without the cell arithmetic).
__global__ void __launch_bounds__(kKeysThreads) raw_hist_kernel(const uint32_t* __restrict__ keys,
                                                                uint32_t n, uint32_t* __restrict__ gcount,
                                                                uint32_t* __restrict__ cnt0, KeyDigits kd) {
  __shared__ uint32_t sh[sort::kMaxPasses][sort::kMaxRadix];
  for (int t = threadIdx.x; t < sort::kMaxPasses * sort::kMaxRadix; t += blockDim.x)
    (&sh[0][0])[t] = 0u;
  __syncthreads();
  const uint32_t base = blockIdx.x * (uint32_t)sort::kTile;
  for (int j = 0; j < sort::kTile / kKeysThreads; ++j) {
    const uint32_t i = base + (uint32_t)j * kKeysThreads + threadIdx.x;
    if (i < n) {
      const uint32_t key = __ldg(keys + i);
#pragma unroll
      for (int p = 0; p < sort::kMaxPasses; ++p)
        if (p < kd.passes) atomicAdd(&sh[p][(key >> kd.shift[p]) & ((1u << kd.bits[p]) - 1u)], 1u);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (1 << kd.bits[0]); t += blockDim.x)
    cnt0[(size_t)blockIdx.x * sort::kMaxRadix + t] = sh[0][t];
#pragma unroll
  for (int p = 0; p < sort::kMaxPasses; ++p) {
    if (p >= kd.passes) break;
    for (int t = threadIdx.x; t < (1 << kd.bits[p]); t += blockDim.x) {
      const uint32_t c = sh[p][t];
      if (c) atomicAdd(gcount + p * sort::kMaxRadix + t, c);
    }
  }
}

// out[i] = in[perm[i]] for elements of `bytes` bytes (4-byte words when the
// size allows).
__global__ void __launch_bounds__(kBlock) gather_payload_kernel(const unsigned char* __restrict__ in,
                                                                unsigned char* __restrict__ out,
                                                                const uint32_t* __restrict__ perm,
                                                                size_t n, size_t bytes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t src = (size_t)__ldg(perm + i) * bytes, dst = i * bytes;
  if (bytes % 4 == 0) {
    for (size_t b = 0; b < bytes; b += 4)
      *reinterpret_cast<uint32_t*>(out + dst + b) = *reinterpret_cast<const uint32_t*>(in + src + b);
  } else {
    for (size_t b = 0; b < bytes; ++b) out[dst + b] = in[src + b];
  }
}

// Run heads -> run keys and run start positions (head_write_kernel + starts),
// plus an "unsorted" flag if any key decreases.
__global__ void __launch_bounds__(kBlock) head_start_kernel(const uint32_t* __restrict__ sk, uint32_t n,
                                                            const uint32_t* __restrict__ offsets,
                                                            uint32_t* __restrict__ run_keys,
                                                            uint32_t* __restrict__ run_start,
                                                            uint32_t* __restrict__ unsorted) {
  __shared__ uint32_t s_w[kBlock / 32];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool head = i < n && (i == 0 || sk[i] != sk[i - 1]);
  if (i < n && i > 0 && sk[i] < sk[i - 1]) atomicOr(unsorted, 1u);
  const uint32_t hb = __ballot_sync(0xffffffffu, head);
  if (lane == 0) s_w[warp] = __popc(hb);
  __syncthreads();
  uint32_t base = offsets[blockIdx.x];
  for (int w = 0; w < warp; ++w) base += s_w[w];
  if (head) {
    const uint32_t r = base + __popc(hb & ((1u << lane) - 1u));
    run_keys[r] = sk[i];
    run_start[r] = i;
  }
}

// One thread per (run, column): the left fold of the run's rows in index
// order -- segmented_reduce_rows at workers == 1 (reduce.hpp:80-137), so the
// sums are the reference's bit for bit at one worker.
__global__ void __launch_bounds__(kBlock) run_fold_kernel(const double* __restrict__ values,
                                                          size_t width, const uint32_t* __restrict__ run_start,
                                                          const uint32_t* __restrict__ qp, uint32_t n,
                                                          double* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t q = *qp;
  if (t >= (size_t)q * width) return;
  const size_t r = t / width, k = t - r * width;
  const uint32_t b = __ldg(run_start + r), e = r + 1 < q ? __ldg(run_start + r + 1) : n;
  double acc = __ldg(values + (size_t)b * width + k);
  for (uint32_t i = b + 1; i < e; ++i) acc += __ldg(values + (size_t)i * width + k);
  out[r * width + k] = acc;
}

}  // namespace

void sort_keys_device(Context& ctx, uint32_t* d_keys, void* d_payload, size_t bytes, size_t n,
                      PointScratch& s) {
  if (n < 2) return;
  cudaStream_t st = ctx.stream;
  s.reserve_points(n, false);
  const sort::DigitPlan plan = sort::plan_digits(32);
  const int ntiles = (int)((n + sort::kTile - 1) / sort::kTile);
  const size_t table = (size_t)ntiles * sort::kMaxRadix;
  uint32_t* gcount = s.hist.p;
  uint32_t* offs = s.hist.p + kOffOff;
  auto cnt = [&](int p) { return s.hist.p + kOffOff + table * (size_t)(1 + p); };
  IBC_CUDA(cudaMemsetAsync(gcount, 0, kOffOff * 4, st));
  IBC_CUDA(cudaMemsetAsync(cnt(1), 0, table * (size_t)(plan.passes - 1) * 4, st));
  static bool attr_set[64] = {};
  if (!attr_set[ctx.device & 63]) {
    IBC_CUDA(cudaFuncSetAttribute(sort::onesweep_pass<sort::kPayloadNone>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sort_smem()));
    attr_set[ctx.device & 63] = true;
  }
  KeyDigits kd{};
  kd.passes = plan.passes;
  for (int p = 0; p < plan.passes; ++p) {
    kd.shift[p] = plan.shift[p];
    kd.bits[p] = plan.bits[p];
  }
  raw_hist_kernel<<<ntiles, kKeysThreads, 0, st>>>(d_keys, (uint32_t)n, gcount, cnt(0), kd);
  ++ctx.launches;
  // A 4-byte payload rides along as the sort's value; any other is gathered
  // through the permutation afterwards.
  const bool word = bytes == 4 && d_payload;
  const uint32_t* first_vals = word ? static_cast<const uint32_t*>(d_payload) : nullptr;
  const uint32_t* src_k = d_keys;
  int dst = 0;
  for (int p = 0; p < plan.passes; ++p) {
    const bool last = p + 1 == plan.passes;
    const int radix = 1 << plan.bits[p];
    sort::tile_offsets_kernel<<<(radix + 31) / 32, sort::kThreads, 0, st>>>(
        cnt(p), offs, gcount + (size_t)p * sort::kMaxRadix, radix, ntiles);
    sort::onesweep_pass<sort::kPayloadNone><<<ntiles, sort::kThreads, sort_smem(), st>>>(
        src_k, p == 0 ? first_vals : s.vals[dst ^ 1].p, s.keys[dst].p, s.vals[dst].p, (uint32_t)n,
        plan.shift[p], plan.bits[p], offs, last ? nullptr : cnt(p + 1), last ? 0 : plan.shift[p + 1],
        last ? 1 : plan.bits[p + 1], nullptr, nullptr, nullptr, DevGrid{}, nullptr);
    ctx.launches += 2;
    src_k = s.keys[dst].p;
    dst ^= 1;
  }
  const int fin = dst ^ 1;  // buffers of the last pass
  IBC_CUDA(cudaMemcpyAsync(d_keys, s.keys[fin].p, n * 4, cudaMemcpyDeviceToDevice, st));
  if (word) {
    IBC_CUDA(cudaMemcpyAsync(d_payload, s.vals[fin].p, n * 4, cudaMemcpyDeviceToDevice, st));
  } else if (d_payload && bytes) {
    s.prim_bytes.ensure(n * bytes);
    gather_payload_kernel<<<grid_for(n, kBlock), kBlock, 0, st>>>(
        static_cast<const unsigned char*>(d_payload), s.prim_bytes.p, s.vals[fin].p, n, bytes);
    ++ctx.launches;
    IBC_CUDA(cudaMemcpyAsync(d_payload, s.prim_bytes.p, n * bytes, cudaMemcpyDeviceToDevice, st));
  }
  IBC_CUDA(cudaGetLastError());
  s.last_n = 0;  // the scratch no longer holds a spread's observables
  s.obs_pending = false;
}

size_t runs_device(Context& ctx, const uint32_t* d_keys, size_t n, PointScratch& s,
                   uint32_t* d_run_keys, const double* d_values, size_t width, double* d_out,
                   bool* unsorted) {
  if (unsorted) *unsorted = false;
  if (n == 0) return 0;
  cudaStream_t st = ctx.stream;
  s.counters.ensure(kCounters + 2);
  uint32_t* qp = s.counters.p + kMaxPasses;
  uint32_t* flag = qp + 1;
  const unsigned nb = grid_for(n, kBlock);
  s.block_counts.ensure(nb);
  s.prim_u32.ensure(2 * n);
  uint32_t* rk = d_run_keys ? d_run_keys : s.prim_u32.p;
  uint32_t* starts = s.prim_u32.p + n;
  IBC_CUDA(cudaMemsetAsync(flag, 0, 4, st));
  head_count_kernel<<<nb, kBlock, 0, st>>>(d_keys, (uint32_t)n, s.block_counts.p);
  block_scan_kernel<<<1, sort::kThreads, 0, st>>>(s.block_counts.p, nb, qp);
  head_start_kernel<<<nb, kBlock, 0, st>>>(d_keys, (uint32_t)n, s.block_counts.p, rk, starts, flag);
  ctx.launches += 3;
  if (d_values && d_out && width) {
    // q <= n runs: launch for n * width threads, idle past q * width.
    run_fold_kernel<<<grid_for(n * width, kBlock), kBlock, 0, st>>>(d_values, width, starts, qp,
                                                                    (uint32_t)n, d_out);
    ++ctx.launches;
  }
  IBC_CUDA(cudaGetLastError());
  uint32_t h[2] = {0, 0};
  IBC_CUDA(cudaMemcpyAsync(h, qp, 8, cudaMemcpyDeviceToHost, st));
  IBC_CUDA(cudaStreamSynchronize(st));
  if (unsorted) *unsorted = h[1] != 0;
  return h[0];
}

}  // namespace ibc
