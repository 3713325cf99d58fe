// ibc_zsweep.cuh -- z-sweep spread and interpolation kernels (3-D grids).
//
// Both operators walk a CTA's column of the grid -- all of x, TY rows of y,
// a chunk of ZC planes of z -- one plane at a time, holding a rolling window
// of 4 planes in shared memory (the kernel's support is 4 planes deep).
// Rows are whole, so periodic x wraps inside the window through a 3-cell
// left / 2-cell right pad that is folded back when a plane is written.
// Only the y direction has a halo (3 rows); z and x are exact.
//
// Spread (spread.hpp:165-216, Alg. 4): the points of source plane s are
// staged row by row (rows are contiguous in the key-sorted order) into
// registers -- one point per lane, its 3 x 4 delta weights computed once --
// and pushed into the window planes s-2..s+1.  Conflict freedom without
// atomics: (1) four sigma_y phases separated by __syncthreads, so distinct
// source rows always hit distinct target rows; (2) a source row is owned by
// one warp, whose lanes visit sigma_x in lock-step (distinct cells -> distinct
// targets); (3) points sharing a cell are adjacent lanes and are serialized
// by their rank in the cell.  Summation order is fixed, so results are
// bitwise reproducible.  A plane leaves the window only once complete and is
// written to HBM exactly once, with coalesced stores.
//
// Interpolation (interpolate.hpp:22-58, Alg. 3): the same column walk with a
// window of FIELD planes; each point is gathered exactly once from shared
// memory, rows of the window arrive by cp.async.bulk (TMA bulk copies)
// signalled on an mbarrier.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"

namespace ibc {
namespace zs {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRows = 32;  // source/field rows per tile (ty + 5 <= 32)
constexpr int kPadL = 4;      // padded x index = x + kPadL (16-byte aligned row body)
constexpr int kPadR = 2;
constexpr int kBatches = 2;   // point batches a warp keeps in registers per group

struct Tiling {
  int ty, zc, nty, nzc, nxp;  // nxp = n0 + kPadL + kPadR (even)
};

// Debug timeline (clock64 per step and phase, CTA `trace_block`, thread 0).
__device__ long long g_trace[2][64][8];
__device__ int g_trace_block = -1;
#define ZS_TRACE(which, step, slot)                                               \
  do {                                                                            \
    if ((int)blockIdx.x == g_trace_block && threadIdx.x == 0 && (step) >= 0 &&   \
        (step) < 64)                                                              \
      g_trace[which][step][slot] = clock64();                                     \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t lanemask_le() {
  const int lane = threadIdx.x & 31;
  return lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
}

__device__ __forceinline__ uint32_t row_id(const DevGrid& g, int cyw, int czw) {
  return (uint32_t)(cyw + 1) + (uint32_t)(czw + 1) * (uint32_t)(g.n[1] + 2);
}

// One staged spread point held by a lane.
struct SrcPoint {
  int cx, cyu, rank, run_after;  // run_after: following lanes in the same cell (heads only)
  bool valid;
  double gx[4], wy[4], wz[4];
};

constexpr int kSThreads = 128;  // spread CTA: 4 warps, small window -> 6 CTAs / SM
constexpr int kSWarps = kSThreads / 32;

// Fold the periodic x pad of one window row and store it (x in [0, nx)).
__device__ __forceinline__ double folded(const double* row, int x, int nx, bool periodic) {
  double v = row[x];
  if (periodic) {
    if (nx >= 4) {
      if (x < 2) v += row[x + nx];
      if (x >= nx - 3) v += row[x - nx];
    } else {
      for (int p = x - nx; p >= -3; p -= nx) v += row[p];
      for (int p = x + nx; p <= nx + 1; p += nx) v += row[p];
    }
  }
  return v;
}

// ------------------------------------------------------------------ spread
constexpr int kStages = 3;        // TMA ring depth (work items in flight)
constexpr int kCap = 256;         // sorted points per work item (32 B records)
constexpr int kMaxSteps = 72;     // z-steps per CTA (zc + 4)

struct SpreadSmem {
  double4 ring[kStages][kCap];               // sorted records {x, y, z, G}
  uint64_t bar[kStages];
  uint32_t rs[kMaxSteps][kMaxRows];          // per step, per source row: sorted range start
  uint32_t pref[kMaxSteps][kMaxRows + 1];    // per step: prefix of row lengths
  uint32_t item0[kMaxSteps + 1];             // first work item of each step
};

__device__ __forceinline__ int find_row(const uint32_t* pref, int nrows, uint32_t p) {
  int j = 0;
  while (j + 1 < nrows && pref[j + 1] <= p) ++j;
  return j;
}

__global__ void __launch_bounds__(kSThreads) spread_zsweep_kernel(
    DevGrid g, Tiling T, const uint32_t* __restrict__ rowstart, const double* __restrict__ rec,
    double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SpreadSmem& S = *reinterpret_cast<SpreadSmem*>(smem_raw);
  double* win = reinterpret_cast<double*>(smem_raw + sizeof(SpreadSmem));  // [4][ty][nxp] + dummies

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int by = blockIdx.x % T.nty, bz = blockIdx.x / T.nty;
  const int y0 = by * T.ty, y1 = min(y0 + T.ty, ny);
  const int z0 = bz * T.zc, z1 = min(z0 + T.zc, nz);
  const int rows = y1 - y0;
  const int srows = rows + 3;            // unwrapped source rows y0-1 .. y1+1
  const int nsteps = (z1 + 1) - (z0 - 1) + 1;  // source planes z0-1 .. z1+1
  const int plane = T.ty * T.nxp;
  double* dummy = win + 4 * plane + tid;  // sink for lanes with nothing to add
  const uint32_t le = lanemask_le();
  const bool px = g.periodic[0] != 0;
  const bool vec = (nx & 1) == 0;

  for (int i = tid; i < 4 * plane + kSThreads; i += kSThreads) win[i] = 0.0;
  // Prologue: sorted ranges of every (step, source row) of this CTA.
  for (int e = tid; e < nsteps * srows; e += kSThreads) {
    const int st = e / srows, j = e - st * srows;
    const int s = z0 - 1 + st, cyu = y0 - 1 + j;
    uint32_t rb = 0, len = 0;
    const bool zok = g.periodic[2] || (s >= -1 && s <= nz);
    const bool yok = g.periodic[1] || (cyu >= -1 && cyu <= ny);
    if (zok && yok) {
      const int cyw = g.periodic[1] ? wrap_cell(cyu, ny) : cyu;
      const int szw = g.periodic[2] ? wrap_cell(s, nz) : s;
      const uint32_t rid = row_id(g, cyw, szw);
      rb = __ldg(rowstart + rid);
      len = __ldg(rowstart + rid + 1) - rb;
    }
    S.rs[st][j] = rb;
    S.pref[st][j + 1] = len;  // lengths for now
  }
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&S.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid < nsteps) {
    uint32_t acc = 0;
    S.pref[tid][0] = 0;
    for (int j = 0; j < srows; ++j) {
      acc += S.pref[tid][j + 1];
      S.pref[tid][j + 1] = acc;
    }
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t it = 0;
    for (int st = 0; st < nsteps; ++st) {
      S.item0[st] = it;
      it += (S.pref[st][srows] + kCap - 1) / kCap;
    }
    S.item0[nsteps] = it;
  }
  __syncthreads();
  const uint32_t nitems = S.item0[nsteps];

  // Producer (thread 0): TMA bulk copies of work item k into ring slot k % kStages.
  auto issue = [&](uint32_t k) {
    if (k >= nitems) return;
    int st = 0;
    while (st + 1 < nsteps && S.item0[st + 1] <= k) ++st;
    const uint32_t a = (k - S.item0[st]) * kCap;
    const uint32_t b = min(a + (uint32_t)kCap, S.pref[st][srows]);
    const int slot = (int)(k % kStages);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&S.bar[slot], (b - a) * 32u);
    uint32_t run_src = 0, run_dst = 0, run_len = 0;
    for (int j = 0; j < srows; ++j) {
      const uint32_t pa = max(S.pref[st][j], a), pb = min(S.pref[st][j + 1], b);
      if (pa >= pb) continue;
      const uint32_t src = S.rs[st][j] + (pa - S.pref[st][j]);
      if (run_len && run_src + run_len == src) {
        run_len += pb - pa;
      } else {
        if (run_len)
          bulk_g2s(&S.ring[slot][run_dst], rec + (size_t)run_src * 4, run_len * 32u, &S.bar[slot]);
        run_src = src;
        run_dst = pa - a;
        run_len = pb - pa;
      }
    }
    if (run_len) bulk_g2s(&S.ring[slot][run_dst], rec + (size_t)run_src * 4, run_len * 32u, &S.bar[slot]);
  };
  if (tid == 0)
    for (uint32_t k = 0; k < (uint32_t)kStages; ++k) issue(k);

  uint32_t item = 0;
  for (int st = 0; st <= nsteps; ++st) {
    const int s = z0 - 1 + st;
    // (a) Target plane s-3 is complete (its last source plane was s-1): fold
    //     the periodic x pad back, write it to HBM once, clear the slot for
    //     plane s+1.  Each element is read and cleared by one thread.
    const int t = s - 3;
    if (t >= z0 && t < z1) {
      double* wp = win + (t & 3) * plane;
      if (vec && nx >= 4) {
        const int half = nx >> 1;
        for (int r = 0; r < rows; ++r) {
          double* row = wp + r * T.nxp + kPadL;
          double* orow = out + ((size_t)t * ny + (size_t)(y0 + r)) * nx;
          for (int i = tid; i < half; i += kSThreads) {
            const int x = 2 * i;
            double2 v = *reinterpret_cast<double2*>(row + x);
            *reinterpret_cast<double2*>(row + x) = make_double2(0.0, 0.0);
            if (px) {
              if (x < 2) {
                v.x += row[x + nx];
                v.y += row[x + 1 + nx];
                row[x + nx] = 0.0;
                row[x + 1 + nx] = 0.0;
              }
              if (x + 1 >= nx - 3) {
                if (x >= nx - 3) { v.x += row[x - nx]; row[x - nx] = 0.0; }
                v.y += row[x + 1 - nx];
                row[x + 1 - nx] = 0.0;
              }
            }
            *reinterpret_cast<double2*>(orow + x) = v;
          }
          if (!px && tid < kPadL + kPadR) {  // closed x: pads only collect dropped targets
            const int pi = tid < kPadL ? tid - kPadL : nx + (tid - kPadL);
            row[pi] = 0.0;
          }
        }
      } else {
        __syncthreads();
        for (int r = 0; r < rows; ++r) {
          const double* row = wp + r * T.nxp + kPadL;
          double* orow = out + ((size_t)t * ny + (size_t)(y0 + r)) * nx;
          for (int x = tid; x < nx; x += kSThreads) orow[x] = folded(row, x, nx, px);
        }
        __syncthreads();
        for (int i = tid; i < plane; i += kSThreads) wp[i] = 0.0;
      }
    }
    if (st == nsteps) break;
    __syncthreads();
    ZS_TRACE(0, st, 0);

    const uint32_t* pref = S.pref[st];
    const uint32_t total = pref[srows];
    for (uint32_t c = 0; c * kCap < total; ++c, ++item) {
      const int slot = (int)(item % kStages);
      mbar_wait(&S.bar[slot], (item / kStages) & 1u);
      ZS_TRACE(0, st, 1);
      const uint32_t a = c * kCap, cnt = min((uint32_t)kCap, total - a);
      // Row-aligned split of [a, a + cnt) among the warps (same on every thread).
      int lo = 0, hi = 0, groups = 0;
      {
        int wl[kSWarps + 1];
        const int jf = find_row(pref, srows, a);
        const int jl = find_row(pref, srows, a + cnt - 1);
        int j = jf;
        for (int w = 0; w <= kSWarps; ++w) {
          const uint32_t target = a + (uint32_t)(((uint64_t)cnt * w) / kSWarps);
          while (j <= jl && max(pref[j], a) < target) ++j;
          wl[w] = (w == kSWarps) ? (int)cnt
                                 : (int)min(cnt, max(pref[min(j, jl + 1)], a) - a);
          if (w == 0) wl[0] = 0;
        }
        for (int w = 0; w < kSWarps; ++w) groups = max(groups, (wl[w + 1] - wl[w] + 31) / 32);
        lo = wl[warp];
        hi = wl[warp + 1];
      }
      for (int gi = 0; gi < groups; ++gi) {
        // (b) One point per lane from the ring: cell, weights, in-cell rank.
        const int pl = lo + gi * 32 + lane;
        const bool valid = pl < hi;
        int cx = 0, cyu = y0;
        uint32_t key = 0xffffffffu;
        double gx[4], wy[4], wz[4];
        if (valid) {
          const double4 r = S.ring[slot][pl];
          const int j = find_row(pref, srows, a + (uint32_t)pl);
          cyu = y0 - 1 + j;
          const double xx[3] = {r.x, r.y, r.z};
          double w[3][4];
          int c3[3];
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            double xw;
            c3[ax] = cell_of(g, ax, xx[ax], &xw);
            cosine_weights(displacement(g, ax, xw, c3[ax]), g.inv_h, w[ax]);
          }
          cx = px ? wrap_cell(c3[0], nx) : c3[0];
          key = cell_key(g, c3);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            gx[k] = w[0][k] * r.w;
            wy[k] = w[1][k];
            wz[k] = w[2][k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) gx[k] = wy[k] = wz[k] = 0.0;
        }
        const uint32_t pkey = __shfl_up_sync(0xffffffffu, key, 1);
        const bool head = valid && (lane == 0 || pkey != key);
        const uint32_t hm = __ballot_sync(0xffffffffu, head);
        const uint32_t vm = __ballot_sync(0xffffffffu, valid);
        const int rank = valid ? lane - (31 - __clz(hm & le)) : 1;
        const uint32_t later = hm & ~le;
        const int next = later ? __ffs(later) - 1 : __popc(vm);
        const int run_after = head ? next - lane - 1 : 0;
        const int maxrank = __reduce_max_sync(0xffffffffu, (unsigned)run_after);
        ZS_TRACE(0, st, 2);
        // (c) Four sigma_y phases: distinct source rows hit distinct target rows.
#pragma unroll 1
        for (int sy = -2; sy <= 1; ++sy) {
          const int ty = cyu + sy;
          const bool inrow = valid && ty >= y0 && ty < y1;
          if (__ballot_sync(0xffffffffu, inrow) != 0u) {
            const bool yok = inrow && rank == 0;
            const int rowoff = yok ? (ty - y0) * T.nxp + cx + (kPadL - 2) : 0;
            const double wyv = sy == -2 ? wy[0] : sy == -1 ? wy[1] : sy == 0 ? wy[2] : wy[3];
#pragma unroll
            for (int sz = -2; sz <= 1; ++sz) {
              const int tz = s + sz;
              if (tz < z0 || tz >= z1) continue;  // warp-uniform
              double* base = win + (tz & 3) * plane + rowoff;
              const double a2 = wyv * wz[sz + 2];
              if (maxrank == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  double* dst = yok ? base + k : dummy;
                  *dst += gx[k] * a2;
                  __syncwarp();
                }
              } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  double v = gx[k] * a2;
                  for (int jj = 1; jj <= maxrank; ++jj) {
                    const double w2 = __shfl_down_sync(0xffffffffu, v, jj);
                    if (jj <= run_after) v += w2;
                  }
                  double* dst = yok ? base + k : dummy;
                  *dst += v;
                  __syncwarp();
                }
              }
            }
          }
          __syncthreads();
          ZS_TRACE(0, st, 5 + sy);
        }
      }
      // The slot is free: prefetch work item item + kStages into it.
      if (tid == 0) issue(item + kStages);
    }
  }
}

// ------------------------------------------------------------------ interpolation
// Skewed row layout (see spread_rows_kernel): padded x index xi -> xi + xi/16,
// so the gathers of points ~16 cells apart fall on distinct banks.
__device__ __forceinline__ int iskew(int xi) { return xi + (xi >> 4); }

constexpr int kIThreads = 256;
constexpr int kMaxPlaneVals = 16;  // field values per thread per plane prefetch

__global__ void __launch_bounds__(kIThreads) interp_zsweep_kernel(
    DevGrid g, Tiling T, const uint32_t* __restrict__ rowstart, const double* __restrict__ rec,
    const double* __restrict__ field, double* __restrict__ out) {
  extern __shared__ __align__(16) double fwin[];  // [4][frows][nxp] (skewed rows)
  const int tid = threadIdx.x;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int by = blockIdx.x % T.nty, bz = blockIdx.x / T.nty;
  const int y0 = by * T.ty, y1 = min(y0 + T.ty, ny);
  const int z0 = bz * T.zc, z1 = min(z0 + T.zc, nz);
  // Home rows/planes: ghost cells (-1, n) belong to the boundary tiles on
  // non-periodic axes.
  const int hy0 = (!g.periodic[1] && y0 == 0) ? -1 : y0;
  const int hy1 = (!g.periodic[1] && y1 == ny) ? ny + 1 : y1;
  const int hz0 = (!g.periodic[2] && z0 == 0) ? -1 : z0;
  const int hz1 = (!g.periodic[2] && z1 == nz) ? nz + 1 : z1;
  const int frows = (hy1 - hy0) + 3;  // field rows hy0-2 .. hy1
  const int rowlen = nx + kPadL + kPadR;  // padded x extent
  const int plane = frows * T.nxp;
  const int pvals = frows * rowlen;

  // Field plane t (unwrapped) -> registers (coalesced loads), then -> window.
  double pre[kMaxPlaneVals];
  auto fetch_plane = [&](int t) {
    const bool zin = g.periodic[2] || (t >= 0 && t < nz);
    const int tw = g.periodic[2] ? wrap_cell(t, nz) : t;
#pragma unroll
    for (int k = 0; k < kMaxPlaneVals; ++k) {
      const int e = tid + k * kIThreads;
      double v = 0.0;
      if (e < pvals && zin) {
        const int r = e / rowlen, xi = e - r * rowlen;
        const int yu = hy0 - 2 + r, x = xi - kPadL;
        const bool yin = g.periodic[1] || (yu >= 0 && yu < ny);
        const bool xin = g.periodic[0] || (x >= 0 && x < nx);
        if (yin && xin) {
          const int yw = g.periodic[1] ? wrap_cell(yu, ny) : yu;
          const int xw = g.periodic[0] ? wrap_cell(x, nx) : x;
          v = __ldg(field + ((size_t)tw * ny + yw) * nx + xw);
        }
      }
      pre[k] = v;
    }
  };
  auto store_plane = [&](int t) {
    double* wp = fwin + (t & 3) * plane;
#pragma unroll
    for (int k = 0; k < kMaxPlaneVals; ++k) {
      const int e = tid + k * kIThreads;
      if (e < pvals) {
        const int r = e / rowlen, xi = e - r * rowlen;
        wp[r * T.nxp + iskew(xi)] = pre[k];
      }
    }
  };

  for (int t = hz0 - 2; t <= hz0 + 1; ++t) {
    fetch_plane(t);
    store_plane(t);
  }
  __syncthreads();

  for (int s = hz0; s < hz1; ++s) {
    const int step = s - hz0;
    ZS_TRACE(1, step, 0);
    if (s + 2 < hz1 + 1) fetch_plane(s + 2);  // in flight during this step's gathers
    // Points homed in plane s, rows [hy0, hy1): one contiguous sorted range.
    const int szw = g.periodic[2] ? wrap_cell(s, nz) : s;
    const uint32_t rb = __ldg(rowstart + row_id(g, hy0, szw));
    const uint32_t re = __ldg(rowstart + row_id(g, hy1 - 1, szw) + 1);
    for (uint32_t r = rb + tid; r < re; r += kIThreads) {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(rec) + 2 * (size_t)r);
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(rec) + 2 * (size_t)r + 1);
      const uint32_t i = (uint32_t)__double_as_longlong(q1.y);
      const double xx[3] = {q0.x, q0.y, q1.x};
      double w[3][4];
      int c[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double xw;
        c[a] = cell_of(g, a, xx[a], &xw);
        cosine_weights(displacement(g, a, xw, c[a]), g.inv_h, w[a]);
      }
      const int cx = g.periodic[0] ? wrap_cell(c[0], nx) : c[0];
      const int cy = g.periodic[1] ? wrap_cell(c[1], ny) : c[1];
      double part[4];
#pragma unroll
      for (int kz = 0; kz < 4; ++kz) {
        const double* pz = fwin + ((s + kz - 2) & 3) * plane;
        double acc = 0.0;
#pragma unroll
        for (int ky = 0; ky < 4; ++ky) {
          const double* prow = pz + (cy - hy0 + ky) * T.nxp;
#pragma unroll
          for (int kx = 0; kx < 4; ++kx) {
            const double wt = (w[0][kx] * w[1][ky]) * w[2][kz];
            acc += wt * prow[iskew(cx + kx + (kPadL - 2))];
          }
        }
        part[kz] = acc;
      }
      out[i] = ((part[0] + part[1]) + (part[2] + part[3])) * g.hd;
    }
    ZS_TRACE(1, step, 1);
    if (s + 1 < hz1) {
      __syncthreads();  // everyone is done with plane s-2
      store_plane(s + 2);
      __syncthreads();
    }
    ZS_TRACE(1, step, 2);
  }
}

}  // namespace zs
}  // namespace ibc
