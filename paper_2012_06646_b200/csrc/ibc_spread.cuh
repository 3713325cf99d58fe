// ibc_spread.cuh -- write-once spreading sweeps (sm_100a), 2-D and 3-D grids.
//
// Replaces ib::spread_fused (spread.hpp:165-216, Alg. 4): the same operator
// l_m = sum_sigma sum_{p in cell(m - sigma)} w_sigma(t_p) G_p, with every grid
// value written to HBM exactly once and no global atomics.
//
// Inputs: each point's 64-byte weight record -- G * phi_x(k-2-t_x)/h for
// k = 0..3 and sin/cos(pi u / 2) of the y and z displacements -- and its
// home cell along x, grouped by home row (ibc_bucket.cuh / ibc_sort.cuh), and
// the start table of those groups.
//
// Warps own target rows of a z-chunk [z0, z1) and sweep the source planes
// z0-1 .. z1+1.  A warp's private shared-memory window holds its rows in the
// four target planes a source plane reaches (s-2 .. s+1), padded by 4 cells
// left and 2 right for the periodic fold.  For source plane s the warp takes
// the points of the four source rows that reach each target row (cy = ty+2 ..
// ty-1) and adds their 16 contributions (4 x x 4 z) per lane.  When plane s is
// done, target plane s-2 is complete: the warp folds the periodic x pad,
// stores the row once (coalesced) and clears the slot for plane s+2.  No CTA
// barrier anywhere: warps are independent.
//
// Two ways to keep a lane's read-modify-writes from colliding, picked on the
// device from the densest row (bucket::bank_mode):
//  * bank mode (spread_banks_kernel): a target row per half-warp; lane b owns
//    x cells = b mod 16 and walks that bank's records (records sit in
//    (row, x bank) buckets), so one instruction's adds hit 16 distinct bank
//    pairs -- conflict-free and collision-free by construction;
//  * pull mode (spread_sweep_kernel): a target row per warp, 32 consecutive
//    records per batch; lanes with the same home cx are summed into their
//    group's lowest lane by shuffles, which adds alone.
// Either way the summation order is fixed by the data: bitwise reproducible.
// Sums are FP64 throughout; TO (double, or float for the FP32 storage mode)
// is only the type of the single store per grid value.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"
#include "ibc_bucket.cuh"  // bank_mode

namespace ibc {
namespace sp {

constexpr int kPadL = 4;  // padded x index xi = x + kPadL
constexpr uint32_t kPullRow = 64;  // densest row above which batches pull instead of bank mode
// Bank-mode lists at least this long (per lane and source plane) take the
// paired loop of plane_banks.
constexpr uint32_t kPairMin = 12;
constexpr int kPadR = 2;

struct SweepTiling {
  int wpc;       // warps (target rows) per CTA
  int nyg;       // CTAs along y
  int zc, nzc;   // z-chunk length, chunks
  int rl;        // doubles per window row (padded, even)
  int group;     // row start table entries per grid row (kBanks: bucket sort; 1: radix path)
  uint32_t pull_row;  // bucket::bank_mode threshold (kNoBankMode: pull mode only)
};

// Doubles per window row for nx: padded, even (16-byte aligned rows).
__host__ __device__ constexpr int row_len(int nx) {
  return (nx + kPadL + kPadR) + ((nx + kPadL + kPadR) & 1);
}

// Bank mode: one source plane for the kRowsPerWarp target rows of a warp,
// GS = kBanks lanes per row.  Lane b of a row's group owns x bank b (x cell
// mod kBanks, up to a fixed shift) and walks that bank's records of the row's
// four source rows in order (records sit in (row, x bank) buckets,
// ibc_bucket.cuh K1-K3; bstart is the bucket start table).  A half-warp
// holds 16 / kBanks rows whose windows are interleaved element by element
// (stride ES = 16 / kBanks), so within a half the cells of one instruction's
// adds hit distinct bank pairs -- and distinct addresses, even across the kx
// phases of one point: conflict-free, no collision test.  Lane gb + j (j <
// 4, gb = the group's first lane) holds source row j's length len and row id
// rid for the group's target row.
// The paired loop of plane_banks for long lists, kept out of line so the
// short-list loop of config-2-like densities is compiled as before.
template <int D, int RL, int R>
__device__ __noinline__ void plane_banks_paired(double* __restrict__ W, uint32_t lo0, uint32_t lo1,
                                                uint32_t lo2, uint32_t lo3, uint32_t c0, uint32_t c1,
                                                uint32_t c2, uint32_t cnt, uint32_t kmax,
                                                const double* __restrict__ rec,
                                                const int* __restrict__ rcx, double q) {
  constexpr int ES = 16 / bucket::kBanks;
  const uint32_t lo[4] = {lo0, lo1, lo2, lo3};
  const uint32_t c[3] = {c0, c1, c2};
  auto pos = [&](uint32_t k) {
    const int j = (k >= c[0]) + (k >= c[1]) + (k >= c[2]);
    return (j == 0 ? lo[0] : j == 1 ? lo[1] : j == 2 ? lo[2] : lo[3]) + k;
  };
  // y / z weights of a record: phi(sigma_y - t_y)/h for its source row j
  // (j = 0..3 -> (1-c), (1+s), (1+c), (1-s) over 4h) times the four z weights.
  auto weights = [&](const double4& gbr, int j, double a[4]) {
    const double vy = (j & 1) ? gbr.x : gbr.y;
    const double wq = q * fma((j == 0 || j == 3) ? -q : q, vy, q);  // wy * q
    if (D == 3) {
      a[0] = fma(-wq, gbr.w, wq);
      a[1] = fma(wq, gbr.z, wq);
      a[2] = fma(wq, gbr.w, wq);
      a[3] = fma(-wq, gbr.z, wq);
    } else {
      a[0] = a[1] = a[3] = 0.0;
      a[2] = wq / q;
    }
  };
  {
    // Long lists (dense rows): records k and k + 1 of a lane in one pass,
    // their read-modify-write chains interleaved.  Both sit in the lane's
    // bank, so their 4-cell x windows are disjoint unless the home cells are
    // equal -- then the pair is summed in registers and added once.
    double4 a1 = make_double4(0.0, 0.0, 0.0, 0.0), b1 = a1, a2 = a1, b2 = a1;
    int x1 = 0, x2 = 0;
    auto load = [&](uint32_t k, double4& ga_, double4& gb_, int& cx_) {
      if (k < cnt) {
        const uint32_t p = pos(k);
        ga_ = ld_v4_nc(rec + 8 * (size_t)p);
        gb_ = ld_v4_nc(rec + 8 * (size_t)p + 4);
        cx_ = __ldg(rcx + p);
      }
    };
    load(0, a1, b1, x1);
    load(1, a2, b2, x2);
    for (uint32_t k = 0; k < kmax; k += 2) {
      const bool v1 = k < cnt;
      bool v2 = k + 1 < cnt;
      double4 na1 = a1, nb1 = b1, na2 = a2, nb2 = b2;  // the next pair, in flight
      int nx1 = x1, nx2 = x2;
      load(k + 2, na1, nb1, nx1);
      load(k + 3, na2, nb2, nx2);
      double w1[4], w2[4];
      weights(b1, (k >= c[0]) + (k >= c[1]) + (k >= c[2]), w1);
      weights(b2, (k + 1 >= c[0]) + (k + 1 >= c[1]) + (k + 1 >= c[2]), w2);
      const double g1[4] = {a1.x, a1.y, a1.z, a1.w};
      const double g2[4] = {a2.x, a2.y, a2.z, a2.w};
      const bool merge = v2 && x2 == x1;
      double* wa1 = W + ES * (x1 + (kPadL - 2));
      double* wa2 = W + ES * (x2 + (kPadL - 2));
      if (merge) v2 = false;
#pragma unroll
      for (int kx = 0; kx < 4; ++kx) {
        double l1[4], l2[4];
#pragma unroll
        for (int kz = 0; kz < 4; ++kz) {
          const int o = ((R + kz + 2) & 3) * (ES * RL) + ES * kx;
          l1[kz] = v1 ? wa1[o] : 0.0;
          l2[kz] = v2 ? wa2[o] : 0.0;
        }
#pragma unroll
        for (int kz = 0; kz < 4; ++kz) {
          const int o = ((R + kz + 2) & 3) * (ES * RL) + ES * kx;
          double t1 = g1[kx] * w1[kz];
          if (merge) t1 = fma(g2[kx], w2[kz], t1);
          if (v1) wa1[o] = l1[kz] + t1;
          if (v2) wa2[o] = l2[kz] + g2[kx] * w2[kz];
        }
        __syncwarp();
      }
      a1 = na1;
      b1 = nb1;
      x1 = nx1;
      a2 = na2;
      b2 = nb2;
      x2 = nx2;
    }
    return;
  }
}

template <int D, int RL, int R>
__device__ __forceinline__ void plane_banks(double* __restrict__ W, const int so[4], uint32_t len,
                                           uint32_t rid, const uint32_t* __restrict__ bstart,
                                           const double* __restrict__ rec,
                                           const int* __restrict__ rcx, double q) {
  constexpr int GS = bucket::kBanks, ES = 16 / GS;
  const int lane = threadIdx.x & 31, bank = lane & (GS - 1), gb = lane & ~(GS - 1);
  uint32_t lo[4], c[4], cnt = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t lenj = __shfl_sync(0xffffffffu, len, gb + j);
    const uint32_t ridj = __shfl_sync(0xffffffffu, rid, gb + j);
    uint32_t b0 = 0, b1 = 0;  // this lane's (row, bank) bucket of source row j
    if (lenj) {
      const uint32_t* t = bstart + (size_t)ridj * GS + bank;
      b0 = __ldg(t);
      b1 = __ldg(t + 1);
    }
    lo[j] = b0 - cnt;  // record slot of this lane's k-th record = lo[j] + k
    cnt += b1 - b0;
    c[j] = cnt;
  }
  const uint32_t kmax = __reduce_max_sync(0xffffffffu, cnt);
  auto pos = [&](uint32_t k) {
    const int j = (k >= c[0]) + (k >= c[1]) + (k >= c[2]);
    return (j == 0 ? lo[0] : j == 1 ? lo[1] : j == 2 ? lo[2] : lo[3]) + k;
  };
  if (R >= 0 && kmax >= kPairMin) {
    plane_banks_paired<D, RL, R>(W, lo[0], lo[1], lo[2], lo[3], c[0], c[1], c[2], cnt, kmax, rec, rcx,
                                 q);
    return;
  }
  // Records are prefetched one iteration ahead (the loop is latency-bound).
  double4 ga = make_double4(0.0, 0.0, 0.0, 0.0), gb4 = ga;
  int cx = 0;
  if (cnt > 0) {
    const uint32_t p = pos(0);
    ga = ld_v4_nc(rec + 8 * (size_t)p);
    gb4 = ld_v4_nc(rec + 8 * (size_t)p + 4);
    cx = __ldg(rcx + p);
  }
  for (uint32_t k = 0; k < kmax; ++k) {
    const bool valid = k < cnt;
    const int j = (k >= c[0]) + (k >= c[1]) + (k >= c[2]);
    double4 na = ga, nb = gb4;
    int ncx = cx;
    if (k + 1 < cnt) {
      const uint32_t p = pos(k + 1);
      na = ld_v4_nc(rec + 8 * (size_t)p);
      nb = ld_v4_nc(rec + 8 * (size_t)p + 4);
      ncx = __ldg(rcx + p);
    }
    // phi(sigma_y - t_y)/h: j = 0..3 -> (1-c), (1+s), (1+c), (1-s) over 4h.
    const double vy = (j & 1) ? gb4.x : gb4.y;
    const double wq = q * fma((j == 0 || j == 3) ? -q : q, vy, q);  // wy * q
    double a[4];
    if (D == 3) {
      a[0] = fma(-wq, gb4.w, wq);
      a[1] = fma(wq, gb4.z, wq);
      a[2] = fma(wq, gb4.w, wq);
      a[3] = fma(-wq, gb4.z, wq);
    } else {
      a[0] = a[1] = a[3] = 0.0;
      a[2] = wq / q;
    }
    const double gk[4] = {ga.x, ga.y, ga.z, ga.w};
    double* wa = W + ES * (cx + (kPadL - 2));
#pragma unroll
    for (int kx = 0; kx < 4; ++kx) {
      if (valid) {
        if (R >= 0) {  // interior plane: slot offsets are immediates
#pragma unroll
          for (int kz = 0; kz < 4; ++kz) wa[((R + kz + 2) & 3) * (ES * RL) + ES * kx] += gk[kx] * a[kz];
        } else {
#pragma unroll
          for (int kz = 0; kz < 4; ++kz)
            if (so[kz] >= 0) wa[ES * (so[kz] + kx)] += gk[kx] * a[kz];
        }
      }
      __syncwarp();
    }
    ga = na;
    gb4 = nb;
    cx = ncx;
  }
}

template <int D, int RL, int R>
__device__ __forceinline__ void plane_batches_pull(double* __restrict__ W, const int so[4], uint32_t e0,
                                              uint32_t e1, uint32_t e2, uint32_t total,
                                              uint32_t rstart,
                                              const double* __restrict__ rec,
                                              const int* __restrict__ rcx, double q, int nx) {
  const int lane = threadIdx.x & 31;
  for (uint32_t base = 0; base < total; base += 32) {
    const uint32_t p = base + (uint32_t)lane;
    bool valid = p < total;
    const int j = (p >= e0) + (p >= e1) + (p >= e2);
    const uint32_t rs = __shfl_sync(0xffffffffu, rstart, j & 3) + p;
    int cx = -0x40000000 - lane;  // distinct per idle lane: never matched
    double2 g01 = make_double2(0.0, 0.0), g23 = g01, tr = g01, tz2 = g01;
    if (valid) {
      const uint32_t r = rs;  // record slot = sorted position
      const double4 ga = ld_v4_nc(rec + 8 * (size_t)r), gb = ld_v4_nc(rec + 8 * (size_t)r + 4);
      g01 = make_double2(ga.x, ga.y);
      g23 = make_double2(ga.z, ga.w);
      tr = make_double2(gb.x, gb.y);
      tz2 = make_double2(gb.z, gb.w);
      cx = __ldg(rcx + r);
      if (cx < -1 || cx > nx) {  // homed outside a closed x axis (radix path): no target
        valid = false;
        cx = -0x40000000 - lane;
      }
    }
    // phi(sigma_y - t_y)/h: j = 0..3 -> (1-c), (1+s), (1+c), (1-s) over 4h.
    const double vy = (j & 1) ? tr.x : tr.y;
    const double wq = q * fma((j == 0 || j == 3) ? -q : q, vy, q);  // wy * q
    double a[4];
    if (D == 3) {
      a[0] = fma(-wq, tz2.y, wq);
      a[1] = fma(wq, tz2.x, wq);
      a[2] = fma(wq, tz2.y, wq);
      a[3] = fma(-wq, tz2.x, wq);
    } else {
      a[0] = a[1] = a[3] = 0.0;
      a[2] = wq / q;
    }
    double gk[4] = {g01.x, g01.y, g23.x, g23.y};
    // Lanes with the same home cx (same cell, or another source row) hit the
    // same 16 targets of this warp's row: the lowest such lane sums the
    // group's contributions in lane (= sequence) order and adds alone.
    const uint32_t peers = __match_any_sync(0xffffffffu, cx);  // every lane takes part
    const int gmax = (int)__reduce_max_sync(0xffffffffu, (uint32_t)__popc(peers));
    const bool lead = valid && (peers & ((1u << lane) - 1u)) == 0u;
    double v[4][4];
#pragma unroll
    for (int kx = 0; kx < 4; ++kx)
#pragma unroll
      for (int kz = 0; kz < 4; ++kz) v[kx][kz] = gk[kx] * a[kz];
    if (gmax > 1) {
      uint32_t rest = lead ? peers & (peers - 1u) : 0u;  // members after the leader
      for (int it = 1; it < gmax; ++it) {
        const int src = rest ? __ffs(rest) - 1 : lane;
        double ma[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) ma[k] = __shfl_sync(0xffffffffu, a[k], src);
#pragma unroll
        for (int kx = 0; kx < 4; ++kx) {  // one member weight at a time (register pressure)
          const double mg = __shfl_sync(0xffffffffu, gk[kx], src);
          if (rest) {
#pragma unroll
            for (int kz = 0; kz < 4; ++kz) v[kx][kz] = fma(mg, ma[kz], v[kx][kz]);
          }
        }
        if (rest) rest &= rest - 1u;
      }
    }
    const int xb = cx + (kPadL - 2);
#pragma unroll
    for (int kx = 0; kx < 4; ++kx) {
      if (lead) {
        double* wa = W + (xb + kx);
        if (R >= 0) {
#pragma unroll
          for (int kz = 0; kz < 4; ++kz) wa[((R + kz + 2) & 3) * RL] += v[kx][kz];
        } else {
#pragma unroll
          for (int kz = 0; kz < 4; ++kz)
            if (so[kz] >= 0) wa[so[kz]] += v[kx][kz];
        }
      }
      __syncwarp();
    }
  }
}

// Pull mode (dense or clustered rows, or records not bank-ordered): one warp
// per target row, batches of 32 consecutive records of the four source rows;
// lanes with the same home cx are summed into their group leader by shuffles.
// Launched next to the bank-mode kernel; the one that does not match the
// densest row seen by the row scan (*maxrow) returns at once.
template <int D, int RL, typename TO>
__global__ void __launch_bounds__(256, 3) spread_sweep_kernel(DevGrid g, SweepTiling T,
                                                           const uint32_t* __restrict__ maxrow,
                                                           const uint32_t* __restrict__ rowstart,
                                                           const double* __restrict__ rec,
                                                           const int* __restrict__ rcx,
                                                           TO* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) double win[];
  if (maxrow && bucket::bank_mode(maxrow, T.pull_row)) return;  // bank mode
  constexpr int kSlots = D == 3 ? 4 : 1;
  const int rl = RL > 0 ? RL : T.rl;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = g.n[0], ny = g.n[1], nz = D == 3 ? g.n[2] : 1;
  const int yg = blockIdx.x % T.nyg, zi = blockIdx.x / T.nyg;
  const int ty = yg * T.wpc + warp;
  if (ty >= ny) return;  // warp-uniform; the kernel has no CTA barriers
  const int z0 = D == 3 ? zi * T.zc : 0;
  const int z1 = D == 3 ? min(z0 + T.zc, nz) : 1;
  double* W = win + (size_t)warp * kSlots * rl;
  for (int i = lane; i < kSlots * rl; i += 32) W[i] = 0.0;
  __syncwarp();

  const bool px = g.periodic[0] != 0, py = g.periodic[1] != 0;
  const bool pz = D == 3 && g.periodic[2] != 0;
  const double q = 0.25 * g.inv_h;
  const int s_lo = D == 3 ? z0 - 1 : 0, s_hi = D == 3 ? z1 + 1 : 0;

  // Lane j < 4: sorted range of source row cy = ty + 2 - j (sigma_y = j - 2)
  // of source plane s; the next plane's ranges are loaded while this one runs.
  auto ranges = [&](int s, uint32_t& rb, uint32_t& len, uint32_t& rid) {
    rb = 0;
    len = 0;
    rid = 0;
    const bool zok = D != 3 || pz || (s >= -1 && s <= nz);
    if (lane < 4 && zok && s <= s_hi) {
      const int szw = D == 3 ? (pz ? wrap_cell(s, nz) : s) : 0;
      int cy = ty + 2 - lane;
      bool ok = true;
      if (py) cy = wrap_cell(cy, ny);
      else ok = cy >= -1 && cy <= ny;
      if (ok) {
        rid = (uint32_t)(cy + 1) + (D == 3 ? (uint32_t)(szw + 1) * (uint32_t)(ny + 2) : 0u);
        rb = __ldg(rowstart + (size_t)rid * T.group);  // row = T.group buckets
        len = __ldg(rowstart + (size_t)rid * T.group + T.group);  // the end: len = end - rb at use
      }
    }
  };
  uint32_t rb_n, len_n, rid_n;
  ranges(s_lo, rb_n, len_n, rid_n);

  for (int s = s_lo; s <= s_hi; ++s) {
    const uint32_t rb = rb_n, len = len_n - rb_n;  // (loaded during the previous plane)
    ranges(s + 1, rb_n, len_n, rid_n);
    {
      // Window slot offset of target plane s + kz - 2 (-1: outside [z0, z1)).
      int so[4];
#pragma unroll
      for (int kz = 0; kz < 4; ++kz) {
        const int tz = s + kz - 2;
        so[kz] = D == 3 ? ((tz >= z0 && tz < z1) ? (tz & 3) * rl : -1) : (kz == 2 ? 0 : -1);
      }
      const bool interior = D == 3 && s - 2 >= z0 && s + 1 < z1;
      {
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t e0 = __shfl_sync(0xffffffffu, incl, 0), e1 = __shfl_sync(0xffffffffu, incl, 1);
        const uint32_t e2 = __shfl_sync(0xffffffffu, incl, 2), total = __shfl_sync(0xffffffffu, incl, 3);
        const uint32_t rstart = rb - (incl - len);  // sorted index = rstart_j + p
        // Interior planes with a compile-time row length take the static
        // path: slot offsets are immediates, no per-add range checks.
        if (RL > 0 && interior) {
          switch (s & 3) {
            case 0: plane_batches_pull<D, RL, 0>(W, so, e0, e1, e2, total, rstart, rec, rcx, q, nx); break;
            case 1: plane_batches_pull<D, RL, 1>(W, so, e0, e1, e2, total, rstart, rec, rcx, q, nx); break;
            case 2: plane_batches_pull<D, RL, 2>(W, so, e0, e1, e2, total, rstart, rec, rcx, q, nx); break;
            default: plane_batches_pull<D, RL, 3>(W, so, e0, e1, e2, total, rstart, rec, rcx, q, nx); break;
          }
        } else {
          plane_batches_pull<D, RL, -1>(W, so, e0, e1, e2, total, rstart, rec, rcx, q, nx);
        }
      }
    }
    // Target plane s - 2 has all its sources: fold, store once, clear.
    const int t = D == 3 ? s - 2 : 0;
    if (t >= z0 && t < z1) {
      double* Wr = W + (D == 3 ? (t & 3) * rl : 0);
      TO* orow = out + ((size_t)t * ny + ty) * nx;
      if (px && nx < 8) {
        for (int x = lane; x < nx; x += 32) {
          double v = Wr[(x + kPadL)];
          for (int qx = x - nx; qx >= -kPadL; qx -= nx) v += Wr[(qx + kPadL)];
          for (int qx = x + nx; qx < nx + kPadR; qx += nx) v += Wr[(qx + kPadL)];
          orow[x] = (TO)v;
        }
      } else {
        for (int x = lane; x < nx; x += 32) {
          double v = Wr[(x + kPadL)];
          if (px) {  // pads x' = -4..-1 fold onto nx-4.., x' = nx, nx+1 onto 0, 1
            if (x >= nx - kPadL) v += Wr[(x - nx + kPadL)];
            if (x < kPadR) v += Wr[(x + nx + kPadL)];
          }
          orow[x] = (TO)v;
        }
      }
      __syncwarp();
      double2* Z = reinterpret_cast<double2*>(Wr);
      for (int i = lane; i < rl / 2; i += 32) Z[i] = make_double2(0.0, 0.0);
      __syncwarp();
    }
  }
}


// Bank mode (bucket::bank_mode): one warp per kRowsPerWarp target rows of a
// z-chunk, z-sweep as above, plane_banks per source plane.  Window per
// half-warp: its 16 / kBanks rows interleaved, four slots.
template <int D, int RL, typename TO>
__global__ void __launch_bounds__(32) spread_banks_kernel(DevGrid g, SweepTiling T,
                                                          const uint32_t* __restrict__ maxrow,
                                                          const uint32_t* __restrict__ bstart,
                                                          const double* __restrict__ rec,
                                                          const int* __restrict__ rcx,
                                                          TO* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) double win[];
  if (!bucket::bank_mode(maxrow, T.pull_row)) return;  // pull mode
  constexpr int kSlots = D == 3 ? 4 : 1;
  constexpr int GS = bucket::kBanks, ES = 16 / GS, RPW = bucket::kRowsPerWarp;
  const int rl = RL > 0 ? RL : T.rl;
  const int lane = threadIdx.x & 31, hl = lane & 15, h = lane >> 4;
  const int grp = lane / GS, bank = lane & (GS - 1), sub = grp & (ES - 1);
  const int nx = g.n[0], ny = g.n[1], nz = D == 3 ? g.n[2] : 1;
  const int yg = blockIdx.x % T.nyg, zi = blockIdx.x / T.nyg;
  const int ty = RPW * yg + grp;  // this group's target row
  const bool row_ok = ty < ny;
  const int z0 = D == 3 ? zi * T.zc : 0;
  const int z1 = D == 3 ? min(z0 + T.zc, nz) : 1;
  const size_t half_win = (size_t)kSlots * ES * rl;  // doubles per half-warp window
  double* Wh = win + (size_t)h * half_win;
  double* W = Wh + sub;  // this group's row, element stride ES
  for (int i = lane; i < 2 * (int)half_win; i += 32) win[i] = 0.0;
  __syncwarp();

  const bool px = g.periodic[0] != 0, py = g.periodic[1] != 0;
  const bool pz = D == 3 && g.periodic[2] != 0;
  const double q = 0.25 * g.inv_h;
  const int s_lo = D == 3 ? z0 - 1 : 0, s_hi = D == 3 ? z1 + 1 : 0;

  // Lane gb + j (j < 4): sorted range of source row cy = ty + 2 - j of
  // source plane s for the group's row; the next plane's load while this runs.
  auto ranges = [&](int s, uint32_t& rb, uint32_t& len, uint32_t& rid) {
    rb = 0;
    len = 0;
    rid = 0;
    const bool zok = D != 3 || pz || (s >= -1 && s <= nz);
    if (bank < 4 && row_ok && zok && s <= s_hi) {
      const int szw = D == 3 ? (pz ? wrap_cell(s, nz) : s) : 0;
      int cy = ty + 2 - bank;
      bool ok = true;
      if (py) cy = wrap_cell(cy, ny);
      else ok = cy >= -1 && cy <= ny;
      if (ok) {
        rid = (uint32_t)(cy + 1) + (D == 3 ? (uint32_t)(szw + 1) * (uint32_t)(ny + 2) : 0u);
        rb = __ldg(bstart + (size_t)rid * GS);  // a row's kBanks buckets
        len = __ldg(bstart + (size_t)rid * GS + GS);  // the end: len = end - rb at use
      }
    }
  };
  uint32_t rb_n, len_n, rid_n;
  ranges(s_lo, rb_n, len_n, rid_n);

  for (int s = s_lo; s <= s_hi; ++s) {
    const uint32_t len = len_n - rb_n, rid = rid_n;  // (loaded during the previous plane)
    ranges(s + 1, rb_n, len_n, rid_n);
    int so[4];
#pragma unroll
    for (int kz = 0; kz < 4; ++kz) {
      const int tz = s + kz - 2;
      so[kz] = D == 3 ? ((tz >= z0 && tz < z1) ? (tz & 3) * rl : -1) : (kz == 2 ? 0 : -1);
    }
    const bool interior = D == 3 && s - 2 >= z0 && s + 1 < z1;
    if (RL > 0 && interior) {
      switch (s & 3) {
        case 0: plane_banks<D, RL, 0>(W, so, len, rid, bstart, rec, rcx, q); break;
        case 1: plane_banks<D, RL, 1>(W, so, len, rid, bstart, rec, rcx, q); break;
        case 2: plane_banks<D, RL, 2>(W, so, len, rid, bstart, rec, rcx, q); break;
        default: plane_banks<D, RL, 3>(W, so, len, rid, bstart, rec, rcx, q); break;
      }
    } else {
      plane_banks<D, RL, -1>(W, so, len, rid, bstart, rec, rcx, q);
    }
    // Target plane s - 2 has all its sources: fold, store once, clear.
    const int t = D == 3 ? s - 2 : 0;
    if (t >= z0 && t < z1) {
      const size_t slot = D == 3 ? (size_t)(t & 3) * ES * rl : 0;
      const double* Wr = W + slot;
      if (row_ok) {
        TO* orow = out + ((size_t)t * ny + ty) * nx;
        if (px && nx < 8) {
          for (int x = bank; x < nx; x += GS) {
            double v = Wr[ES * (x + kPadL)];
            for (int qx = x - nx; qx >= -kPadL; qx -= nx) v += Wr[ES * (qx + kPadL)];
            for (int qx = x + nx; qx < nx + kPadR; qx += nx) v += Wr[ES * (qx + kPadL)];
            orow[x] = (TO)v;
          }
        } else {
          for (int x = bank; x < nx; x += GS) {
            double v = Wr[ES * (x + kPadL)];
            if (px) {  // pads x' = -4..-1 fold onto nx-4.., x' = nx, nx+1 onto 0, 1
              if (x >= nx - kPadL) v += Wr[ES * (x - nx + kPadL)];
              if (x < kPadR) v += Wr[ES * (x + nx + kPadL)];
            }
            orow[x] = (TO)v;
          }
        }
      }
      __syncwarp();
      double2* Z = reinterpret_cast<double2*>(Wh + slot);
      for (int i = hl; i < ES * rl / 2; i += 16) Z[i] = make_double2(0.0, 0.0);
      __syncwarp();
    }
  }
}

}  // namespace sp
}  // namespace ibc
