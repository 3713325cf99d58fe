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
__global__ void __launch_bounds__(kSThreads) spread_zsweep_kernel(
    DevGrid g, Tiling T, const uint32_t* __restrict__ rowstart,
    const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ perm,
    const double* __restrict__ X, const double* __restrict__ G, double* __restrict__ out) {
  extern __shared__ __align__(16) double win[];  // [4][ty][nxp], then one dummy slot per thread
  __shared__ uint32_t s_rb[kMaxRows];
  __shared__ uint32_t s_pref[kMaxRows + 1];
  __shared__ int s_wlo[kSWarps + 1];
  __shared__ int s_groups;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int by = blockIdx.x % T.nty, bz = blockIdx.x / T.nty;
  const int y0 = by * T.ty, y1 = min(y0 + T.ty, ny);
  const int z0 = bz * T.zc, z1 = min(z0 + T.zc, nz);
  const int rows = y1 - y0;
  const int srows = rows + 3;  // unwrapped source rows y0-1 .. y1+1
  const int plane = T.ty * T.nxp;
  double* dummy = win + 4 * plane + tid;  // sink for lanes with nothing to add
  const uint32_t le = lanemask_le();
  const bool px = g.periodic[0] != 0;
  const bool vec = (nx & 1) == 0;  // double2 write-back (row bodies are 16-byte aligned)
  for (int i = tid; i < 4 * plane + kSThreads; i += kSThreads) win[i] = 0.0;

  for (int s = z0 - 1; s <= z1 + 2; ++s) {
    const int step = s - (z0 - 1);
    ZS_TRACE(0, step, 0);
    // (a) Target plane s-3 is complete (its last source plane was s-1):
    //     fold the periodic x pad back and write it to HBM once.
    const int t = s - 3;
    const bool flush = t >= z0 && t < z1;
    if (flush) {
      const double* wp = win + (t & 3) * plane;
      if (vec) {
        const int half = nx >> 1;
        for (int i = tid; i < rows * half; i += kSThreads) {
          const int r = i / half, x = 2 * (i - r * half);
          const double* row = wp + r * T.nxp + kPadL;
          double2 v = *reinterpret_cast<const double2*>(row + x);
          if (px) {
            v.x = folded(row, x, nx, true);
            v.y = folded(row, x + 1, nx, true);
          }
          *reinterpret_cast<double2*>(out + ((size_t)t * ny + (size_t)(y0 + r)) * nx + x) = v;
        }
      } else {
        for (int r = 0; r < rows; ++r) {
          const double* row = wp + r * T.nxp + kPadL;
          double* orow = out + ((size_t)t * ny + (size_t)(y0 + r)) * nx;
          for (int x = tid; x < nx; x += kSThreads) orow[x] = folded(row, x, nx, px);
        }
      }
    }
    ZS_TRACE(0, step, 1);
    // Source-row table of plane s (warp 0).
    const bool src_plane = g.periodic[2] ? true : (s >= -1 && s <= nz);
    const bool sweep = s <= z1 + 1 && src_plane;
    if (warp == 0) {
      uint32_t len = 0, rb = 0;
      if (sweep && lane < srows) {
        const int cyu = y0 - 1 + lane;
        int cyw = cyu;
        bool ok = true;
        if (g.periodic[1]) cyw = wrap_cell(cyu, ny);
        else ok = cyu >= -1 && cyu <= ny;
        if (ok) {
          const int szw = g.periodic[2] ? wrap_cell(s, nz) : s;
          const uint32_t rid = row_id(g, cyw, szw);
          rb = __ldg(rowstart + rid);
          len = __ldg(rowstart + rid + 1) - rb;
        }
      }
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - len;
      if (lane < kMaxRows) {
        s_rb[lane] = rb;
        s_pref[lane] = excl;
      }
      if (lane == 0) s_pref[kMaxRows] = total;
      // Row-aligned chunks: warp w owns rows [wlo[w], wlo[w+1]); a row is
      // never split across warps.
      int lo = srows;
      for (int w = 0; w <= kSWarps; ++w) {
        const uint32_t target = (uint32_t)(((uint64_t)total * w) / kSWarps);
        const uint32_t m = __ballot_sync(0xffffffffu, lane < srows && excl >= target);
        const int j = (w == kSWarps || m == 0u) ? srows : __ffs(m) - 1;
        if (lane == w) lo = j;
      }
      if (lane <= kSWarps) s_wlo[lane] = lo;
      __syncwarp();
      int gcount = 0;
      if (lane < kSWarps) {
        const int a = s_wlo[lane], b = s_wlo[lane + 1];
        const uint32_t pts = (b > a) ? (s_pref[b] - s_pref[a]) : 0u;
        gcount = (int)((pts + 32 * kBatches - 1) / (32 * kBatches));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gcount = max(gcount, __shfl_down_sync(0xffffffffu, gcount, o));
      if (lane == 0) s_groups = gcount;
    }
    __syncthreads();
    ZS_TRACE(0, step, 2);
    // (b) The flushed slot becomes plane s+1's slot: clear it.
    if (flush) {
      double2* wp = reinterpret_cast<double2*>(win + (t & 3) * plane);
      for (int i = tid; i < (plane >> 1); i += kSThreads) wp[i] = make_double2(0.0, 0.0);
    }
    const int groups = s_groups;
    const int wlo = s_wlo[warp], whi = s_wlo[warp + 1];
    const uint32_t pbeg = s_pref[wlo], pend = s_pref[whi];
    __syncthreads();
    ZS_TRACE(0, step, 3);
    if (groups == 0) continue;  // the next table build happens after a barrier

    for (int gi = 0; gi < groups; ++gi) {
      // (c) Stage up to kBatches x 32 points of this warp's rows into registers.
      SrcPoint P[kBatches];
      int maxrank[kBatches];
#pragma unroll
      for (int b = 0; b < kBatches; ++b) {
        const uint32_t p = pbeg + (uint32_t)(gi * kBatches + b) * 32u + (uint32_t)lane;
        SrcPoint& q = P[b];
        q.valid = p < pend;
        q.cx = 0;
        q.cyu = y0;
        uint32_t key = 0xffffffffu;
        if (q.valid) {
          int j = wlo;
          while (j + 1 < whi && s_pref[j + 1] <= p) ++j;
          const uint32_t r = s_rb[j] + (p - s_pref[j]);
          key = __ldg(skeys + r);
          const uint32_t i = __ldg(perm + r);
          q.cyu = y0 - 1 + j;
          double w[3][4];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            double xw;
            const int c = cell_of(g, a, __ldg(X + (size_t)i * 3 + a), &xw);
            cosine_weights(displacement(g, a, xw, c), g.inv_h, w[a]);
            if (a == 0) q.cx = px ? wrap_cell(c, nx) : c;
          }
          const double gv = __ldg(G + i);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            q.gx[k] = w[0][k] * gv;
            q.wy[k] = w[1][k];
            q.wz[k] = w[2][k];
          }
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) q.gx[k] = q.wy[k] = q.wz[k] = 0.0;
        }
        // Points sharing a cell are adjacent lanes (keys are sorted): the
        // head lane adds its followers' contributions before touching memory.
        const uint32_t pkey = __shfl_up_sync(0xffffffffu, key, 1);
        const bool head = q.valid && (lane == 0 || pkey != key);
        const uint32_t hm = __ballot_sync(0xffffffffu, head);
        const uint32_t vm = __ballot_sync(0xffffffffu, q.valid);
        q.rank = q.valid ? lane - (31 - __clz(hm & le)) : 1;
        const uint32_t later = hm & ~le;
        const int next = later ? __ffs(later) - 1 : __popc(vm);
        q.run_after = (head ? next - lane - 1 : 0);
        maxrank[b] = __reduce_max_sync(0xffffffffu, (unsigned)q.run_after);
      }
      ZS_TRACE(0, step, 4);
      // (d) Four sigma_y phases; within a phase distinct source rows hit
      //     distinct target rows.
#pragma unroll
      for (int sy = -2; sy <= 1; ++sy) {
#pragma unroll
        for (int b = 0; b < kBatches; ++b) {
          const SrcPoint& q = P[b];
          const int ty = q.cyu + sy;
          const bool yok = q.valid && q.rank == 0 && ty >= y0 && ty < y1;
          if (__ballot_sync(0xffffffffu, q.valid && ty >= y0 && ty < y1) == 0u) continue;
          const int rowoff = yok ? (ty - y0) * T.nxp + q.cx + (kPadL - 2) : 0;
#pragma unroll
          for (int sz = -2; sz <= 1; ++sz) {
            const int tz = s + sz;
            if (tz < z0 || tz >= z1) continue;  // warp-uniform
            double* base = win + (tz & 3) * plane + rowoff;
            const double a = q.wy[sy + 2] * q.wz[sz + 2];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              double v = q.gx[k] * a;
              for (int j = 1; j <= maxrank[b]; ++j) {
                const double w = __shfl_down_sync(0xffffffffu, v, j);
                if (j <= q.run_after) v += w;
              }
              double* dst = yok ? base + k : dummy;
              *dst += v;
              __syncwarp();
            }
          }
        }
        __syncthreads();
        ZS_TRACE(0, step, 5 + (sy + 2 < 3 ? sy + 2 : 2));
      }
    }
  }
}

// ------------------------------------------------------------------ interpolation
__global__ void __launch_bounds__(kThreads) interp_zsweep_kernel(
    DevGrid g, Tiling T, const uint32_t* __restrict__ rowstart, const uint32_t* __restrict__ perm,
    const double* __restrict__ X, const double* __restrict__ field, double* __restrict__ out,
    int use_bulk) {
  extern __shared__ __align__(16) double fwin[];  // [4][frows][nxp]
  __shared__ __align__(8) uint64_t s_bar[4];

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
  const int plane = frows * T.nxp;

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&s_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t parity = 0;  // bit i: phase parity of s_bar[i]

  // Fill window slot for field plane t (unwrapped): row bodies by TMA bulk
  // copy (or plain loads), zero rows outside closed axes.
  auto load_plane = [&](int t) {
    double* wp = fwin + (t & 3) * plane;
    const bool zin = g.periodic[2] || (t >= 0 && t < nz);
    const int tw = g.periodic[2] ? wrap_cell(t, nz) : t;
    if (use_bulk && zin && tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint32_t bytes = 0;
      for (int r = 0; r < frows; ++r) {
        const int yu = hy0 - 2 + r;
        if (g.periodic[1] || (yu >= 0 && yu < ny)) bytes += (uint32_t)nx * 8u;
      }
      mbar_expect_tx(&s_bar[t & 3], bytes);
      for (int r = 0; r < frows; ++r) {
        const int yu = hy0 - 2 + r;
        if (!(g.periodic[1] || (yu >= 0 && yu < ny))) continue;
        const int yw = g.periodic[1] ? wrap_cell(yu, ny) : yu;
        bulk_g2s(wp + r * T.nxp + kPadL, field + ((size_t)tw * ny + yw) * nx, (uint32_t)nx * 8u,
                 &s_bar[t & 3]);
      }
    }
    // Everything the bulk copies do not write: all of each row without TMA,
    // else only the x pads (zero here; periodic pads are copied from the
    // row body once it has landed, see fill_pads).
    const int total = frows * T.nxp;
    for (int e = tid; e < total; e += kThreads) {
      const int r = e / T.nxp, xi = e - r * T.nxp;
      const int yu = hy0 - 2 + r;
      const bool yin = g.periodic[1] || (yu >= 0 && yu < ny);
      const int x = xi - kPadL;
      const bool body = x >= 0 && x < nx;
      if (use_bulk && zin && yin && (body || g.periodic[0])) continue;  // TMA / fill_pads
      double v = 0.0;
      if (!use_bulk && zin && yin) {
        const int yw = g.periodic[1] ? wrap_cell(yu, ny) : yu;
        const double* src = field + ((size_t)tw * ny + yw) * nx;
        if (body) v = __ldg(src + x);
        else if (g.periodic[0]) v = __ldg(src + wrap_cell(x, nx));
      }
      wp[e] = v;
    }
  };
  // Periodic x pads of bulk-copied rows, from the landed row bodies.
  auto fill_pads = [&](int t) {
    const bool zin = g.periodic[2] || (t >= 0 && t < nz);
    if (!(use_bulk && zin && g.periodic[0])) return;
    double* wp = fwin + (t & 3) * plane;
    const int npad = kPadL + (T.nxp - kPadL - nx);
    for (int e = tid; e < frows * npad; e += kThreads) {
      const int r = e / npad, j = e - r * npad;
      const int yu = hy0 - 2 + r;
      if (!(g.periodic[1] || (yu >= 0 && yu < ny))) continue;
      const int xi = j < kPadL ? j : nx + j;  // padded index
      double* row = wp + r * T.nxp;
      row[xi] = row[kPadL + wrap_cell(xi - kPadL, nx)];
    }
  };
  auto wait_plane = [&](int t) {
    const bool zin = g.periodic[2] || (t >= 0 && t < nz);
    if (use_bulk && zin) {
      mbar_wait(&s_bar[t & 3], (parity >> (t & 3)) & 1u);
      parity ^= 1u << (t & 3);
    }
  };

  for (int t = hz0 - 2; t <= hz0 + 1; ++t) load_plane(t);
  for (int t = hz0 - 2; t <= hz0 + 1; ++t) wait_plane(t);
  for (int t = hz0 - 2; t <= hz0 + 1; ++t) fill_pads(t);
  __syncthreads();

  for (int s = hz0; s < hz1; ++s) {
    const int step = s - hz0;
    ZS_TRACE(1, step, 0);
    // Points homed in plane s, rows [hy0, hy1): one contiguous sorted range.
    const int szw = g.periodic[2] ? wrap_cell(s, nz) : s;
    const uint32_t rb = __ldg(rowstart + row_id(g, hy0, szw));
    const uint32_t re = __ldg(rowstart + row_id(g, hy1 - 1, szw) + 1);
    for (uint32_t r = rb + tid; r < re; r += kThreads) {
      const uint32_t i = __ldg(perm + r);
      double w[3][4];
      int c[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double xw;
        c[a] = cell_of(g, a, __ldg(X + (size_t)i * 3 + a), &xw);
        cosine_weights(displacement(g, a, xw, c[a]), g.inv_h, w[a]);
      }
      const int cx = g.periodic[0] ? wrap_cell(c[0], nx) : c[0];
      const int cy = g.periodic[1] ? wrap_cell(c[1], ny) : c[1];
      double acc = 0.0;
#pragma unroll
      for (int kz = 0; kz < 4; ++kz) {
        const double* pz = fwin + ((s + kz - 2) & 3) * plane;
#pragma unroll
        for (int ky = 0; ky < 4; ++ky) {
          const double* prow = pz + (cy - hy0 + ky) * T.nxp + cx + (kPadL - 2);
#pragma unroll
          for (int kx = 0; kx < 4; ++kx) {
            const double wt = (w[0][kx] * w[1][ky]) * w[2][kz];
            acc += wt * prow[kx];
          }
        }
      }
      out[i] = acc * g.hd;
    }
    ZS_TRACE(1, step, 1);
    if (s + 1 < hz1) {
      __syncthreads();  // everyone is done with plane s-2
      ZS_TRACE(1, step, 2);
      load_plane(s + 2);
      ZS_TRACE(1, step, 3);
      wait_plane(s + 2);
      fill_pads(s + 2);
      ZS_TRACE(1, step, 4);
      __syncthreads();
      ZS_TRACE(1, step, 5);
    }
  }
}

}  // namespace zs
}  // namespace ibc
