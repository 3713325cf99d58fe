// ibc_sweep.cuh -- 3-D interpolation gather fed by TMA (sm_100a).
//
// Replaces the per-point loop of ib::interpolate (interpolate.hpp:22-58,
// Alg. 3).  Points arrive grouped by their home row (cy, cz) (ibc_bucket.cuh),
// each as a 64-byte record {sin/cos(pi u_a / 2) per axis, input index, home
// cx, home cy}: cells and trig are computed once, by the bucketing pass.
//
// A CTA (one per SM) owns TY home rows [y0, y0 + TY) of a z-chunk [z0, z1)
// and sweeps its home planes in order.  The field planes a home plane s needs
// (s-2 .. s+1, rows y0-2 .. y0+TY) live in a ring of `slots` shared-memory
// slots.  A dedicated producer warp fills slot i % slots with field plane i --
// one TMA tensor load per plane (unswizzled rows; per field row where the
// rows wrap around a periodic y boundary), plus one bulk copy of the point
// records of the step that plane completes -- and signals a `full` mbarrier.
// Periodic rows/planes are wrapped by the producer; non-periodic ones fall
// outside the tensor and arrive zero-filled, exactly the reference's skipped
// `invalid_offset` terms.  Consumer warps release a plane on its `empty`
// mbarrier after the last step that reads it; there is no CTA-wide barrier
// in the sweep, so warps drift across steps and the TMA engine streams
// slots - 4 planes ahead of the slowest warp.
//
// Gather layout: four lanes per point, lane k reading x = cx + k - 2 of every
// (y, z) window row; the quad's partial sums are combined with two
// xor-shuffles.  Groups of 8 points are dealt round-robin to the consumer
// warps across steps, so no warp is systematically the last one.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"
#include "ibc_tma.cuh"

namespace ibc {
namespace sw {

constexpr int kIConsumers = 16;                    // consumer warps
constexpr int kIThreads = 32 * (kIConsumers + 1);  // + 1 producer warp
constexpr int kMaxSlots = 16;


__device__ __forceinline__ uint32_t row_id(const DevGrid& g, int cyw, int czw) {
  return (uint32_t)(cyw + 1) + (uint32_t)(czw + 1) * (uint32_t)(g.n[1] + 2);
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// TF: the field / output element type (double, or float for the FP32
// storage mode: planes half the size in shared memory, FP64 arithmetic).
template <typename TF>
__global__ void __launch_bounds__(kIThreads, 1) interp_tma_kernel(
    DevGrid g, InterpTiling T, const __grid_constant__ CUtensorMap tmap_row,
    const __grid_constant__ CUtensorMap tmap_box, const uint32_t* __restrict__ rowstart,
    const double* __restrict__ rec, TF* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // Layout: full[kMaxSlots] | empty[kMaxSlots] | step table [3][hmax] |
  // ring of 1024-aligned slots (field rows of one plane + records of one step).
  const uint32_t raw = tma::smem_u32(smem_raw);
  const uint32_t full0 = raw, empty0 = raw + 8u * kMaxSlots;
  uint32_t* rs = reinterpret_cast<uint32_t*>(smem_raw + 16 * kMaxSlots);
  const uint32_t base = (raw + 16u * kMaxSlots + 12u * T.hmax + 1023u) & ~1023u;
  const unsigned char* slots = smem_raw + (base - raw);
  const int NS = T.slots;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const int by = blockIdx.x % T.nty, bz = blockIdx.x / T.nty;
  const int y0 = by * T.ty, y1 = min(y0 + T.ty, ny);
  const int z0 = bz * T.zc, z1 = min(z0 + T.zc, nz);
  // Home rows/planes; on closed axes the ghost cells -1 and n belong to the
  // boundary tiles.
  const int hy0 = (!g.periodic[1] && y0 == 0) ? -1 : y0;
  const int hy1 = (!g.periodic[1] && y1 == ny) ? ny + 1 : y1;
  const int hz0 = (!g.periodic[2] && z0 == 0) ? -1 : z0;
  const int hz1 = (!g.periodic[2] && z1 == nz) ? nz + 1 : z1;
  const int fr = hy1 - hy0 + 3;       // field rows hy0-2 .. hy1
  const int nplanes = hz1 - hz0 + 3;  // field planes hz0-2 .. hz1
  const int H = hz1 - hz0;            // home planes (steps)
  // One box load per plane unless the rows wrap around a periodic y edge.
  const bool box = T.box_ok && (!g.periodic[1] || (hy0 - 2 >= 0 && hy1 < ny));
  const uint32_t plane_bytes = (uint32_t)(box ? T.frmax : fr) * (uint32_t)nx * (uint32_t)sizeof(TF);

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      tma::mbar_init(full0 + 8u * i, 1);
      tma::mbar_init(empty0 + 8u * i, kIConsumers);
    }
    tma::fence_mbar_init();
  }
  // Sorted point range of every home plane (its rows [hy0, hy1) are
  // contiguous) and the running count of 8-point groups before it.
  for (int jj = tid; jj < H; jj += kIThreads) {
    const int s = hz0 + jj;
    const int sw = g.periodic[2] ? wrap_cell(s, nz) : s;
    rs[jj] = __ldg(rowstart + row_id(g, hy0, sw));
    rs[T.hmax + jj] = __ldg(rowstart + row_id(g, hy1 - 1, sw) + 1);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int jj = 0; jj < H; ++jj) {
      rs[2 * T.hmax + jj] = acc;
      acc += (rs[T.hmax + jj] - rs[jj] + 7u) >> 3;
    }
  }
  __syncthreads();

  // Points homed outside the grid (the extra bucket row, normally empty):
  // their interpolated value is 0 -- every support offset is invalid.
  {
    const uint32_t o0 = __ldg(rowstart + g.nrows), o1 = __ldg(rowstart + g.nrows + 1);
    for (uint32_t r = o0 + blockIdx.x * kIThreads + tid; r < o1; r += gridDim.x * kIThreads)
      out[(uint32_t)__double_as_longlong(rec[8 * (size_t)r + 6])] = TF(0);
  }

  if (warp == kIConsumers) {
    // ------------------------------------------------------------ producer
    for (int i = 0; i < nplanes; ++i) {
      const int slot = i % NS;
      if (i >= NS) tma::mbar_wait(empty0 + 8u * slot, ((i / NS) - 1) & 1);
      int t = hz0 - 2 + i;
      if (g.periodic[2]) t = wrap_cell(t, nz);
      const uint32_t bar = full0 + 8u * slot;
      const int jr = i - 3;  // step whose records ride with this plane
      uint32_t nrec = 0, ra = 0, over = 0;
      if (jr >= 0 && jr < H) {
        ra = rs[jr];
        const uint32_t all = rs[T.hmax + jr] - ra;
        nrec = min(all, (uint32_t)T.rec_cap);
        over = all - nrec;  // read from global by the consumers: pull them into L2 now
      }
      const uint32_t dst = base + (uint32_t)slot * T.slot_stride;
      tma::fence_proxy_async();
      if (lane == 0) {
        tma::mbar_expect_tx(bar, plane_bytes + nrec * 64u);
        if (nrec) tma::bulk_g2s(dst + T.slot_bytes, rec + 8 * (size_t)ra, nrec * 64u, bar);
        if (over) tma::prefetch_bytes(rec + 8 * (size_t)(ra + nrec), over * 64u);
        if (box) tma::load_4d(dst, &tmap_box, 0, 0, hy0 - 2, t, bar);
      }
      __syncwarp();
      if (!box) {
        for (int f = lane; f < fr; f += 32) {
          int y = hy0 - 2 + f;
          if (g.periodic[1]) y = wrap_cell(y, ny);
          tma::load_4d(dst + (uint32_t)f * T.pitch, &tmap_row, 0, 0, y, t, bar);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  // Quad layout: point p = lane / 4 of an 8-point group, kx = lane % 4.
  const int kx = lane & 3;
  const bool px = g.periodic[0] != 0;
  const double q = 0.25 * g.inv_h;
  // Slot of plane j (j % NS) and fill parity of plane j + 3, advanced
  // incrementally (no integer division in the loop).
  int slot_j = 0, slot_3 = 3 % NS;
  uint32_t par_3 = (3 / NS) & 1;
  for (int i = 0; i < 3; ++i) tma::mbar_wait(full0 + 8u * (i % NS), (i / NS) & 1);
  for (int j = 0; j < H; ++j) {
    // Planes j .. j+3 are this step's window; j+3 is the only new one.
    tma::mbar_wait(full0 + 8u * slot_3, par_3);
    const uint32_t a = rs[j], b = rs[T.hmax + j];
    const uint32_t gfirst = rs[2 * T.hmax + j];
    const unsigned char* sl[4];
#pragma unroll
    for (int kz = 0; kz < 4; ++kz) {
      const int sk = slot_j + kz;
      sl[kz] = slots + (size_t)(sk >= NS ? sk - NS : sk) * T.slot_stride;
    }
    const double2* srec = reinterpret_cast<const double2*>(sl[3] + T.slot_bytes);  // 4 x double2 per point
    // This warp's groups: k with (gfirst + k) % kIConsumers == warp.
    const uint32_t k0 =
        (uint32_t)(warp - (int)(gfirst % kIConsumers) + kIConsumers) % kIConsumers;

    for (uint32_t g0 = a + 8u * k0; g0 < b; g0 += 8u * kIConsumers) {
      const uint32_t r = g0 + (uint32_t)(lane >> 2);
      const bool valid = r < b;
      // Record: {sx, cx', sy, cy', sz, cz', (index, home cx), home cy}.
      double2 tx = make_double2(0.0, 1.0), ty = tx, tz = tx, id = make_double2(0.0, 0.0);
      if (valid) {
        const double2* r2 = r - a < (uint32_t)T.rec_cap
                                ? srec + 4 * (r - a)
                                : reinterpret_cast<const double2*>(rec) + 4 * (size_t)r;
        tx = r2[0];
        ty = r2[1];
        tz = r2[2];
        id = r2[3];
      }
      const long long pk = __double_as_longlong(id.x);
      const uint32_t idx = (uint32_t)pk;
      const int cx = (int)(pk >> 32);
      const int cy = (int)__double_as_longlong(id.y);
      // phi(sigma - t)/h for sigma = -2..1: (1-c), (1+s), (1+c), (1-s) over 4h.
      const double wy[4] = {fma(-q, ty.y, q), fma(q, ty.x, q), fma(q, ty.y, q), fma(-q, ty.x, q)};
      const double wz[4] = {fma(-q, tz.y, q), fma(q, tz.x, q), fma(q, tz.y, q), fma(-q, tz.x, q)};
      const double vx = (kx & 1) ? tx.x : tx.y;
      double wxk = fma((kx == 0 || kx == 3) ? -q : q, vx, q);
      int x = cx + kx - 2;
      if (px) {
        x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
      } else if (x < 0 || x >= nx) {
        wxk = 0.0;  // off the closed grid: the reference skips the term
        x = 0;
      }
      const uint32_t xo = (uint32_t)x * (uint32_t)sizeof(TF) + (uint32_t)(valid ? cy - hy0 : 0) * T.pitch;
      double acc = 0.0;
      if (valid) {
        // Pairwise sums (dependency depth 6 instead of 20 fused multiply-adds).
        double az[4];
#pragma unroll
        for (int kz = 0; kz < 4; ++kz) {
          const unsigned char* p = sl[kz] + xo;
          double v[4];
#pragma unroll
          for (int ky = 0; ky < 4; ++ky)
            v[ky] = (double)*reinterpret_cast<const TF*>(p + (uint32_t)ky * T.pitch);
          az[kz] = fma(wy[1], v[1], wy[0] * v[0]) + fma(wy[3], v[3], wy[2] * v[2]);
        }
        acc = (fma(wz[1], az[1], wz[0] * az[0]) + fma(wz[3], az[3], wz[2] * az[2])) * wxk;
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (valid && kx == 0) out[idx] = (TF)(acc * g.hd);
    }
    // Plane j is not read by any later step.
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8u * slot_j)
                   : "memory");
    slot_j = slot_j + 1 == NS ? 0 : slot_j + 1;
    if (++slot_3 == NS) {
      slot_3 = 0;
      par_3 ^= 1u;
    }
  }
}

}  // namespace sw
}  // namespace ibc
