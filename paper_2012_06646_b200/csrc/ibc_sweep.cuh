// ibc_sweep.cuh -- 3-D interpolation gather fed by TMA (sm_100a).
//
// Replaces the per-point loop of ib::interpolate (interpolate.hpp:22-58,
// Alg. 3).  Points arrive sorted by their home row (cy, cz), each as a 32-byte
// record {x, y, z, input index} written by the last radix pass.
//
// A CTA owns TY home rows [y0, y0 + TY) of a z-chunk [z0, z1) and sweeps its
// home planes in order.  The field planes a home plane s needs (s-2 .. s+1,
// rows y0-2 .. y0+TY) live in a ring of kISlots shared-memory slots, each
// filled by one TMA tensor load per field row (128-byte swizzle; periodic
// rows/planes are wrapped by the producer, non-periodic ones fall outside the
// tensor and arrive zero-filled -- exactly the reference's skipped
// `invalid_offset` terms).  While the CTA gathers plane s, the TMA engine
// streams plane s+3 into the slot plane s-2 vacates; the CTA's only barrier
// per plane is the one that frees that slot.  Every field value is read from
// HBM once per CTA column (plus the 3-row y halo), every point once.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ibc_device.cuh"
#include "ibc_tma.cuh"

namespace ibc {
namespace sw {

constexpr int kIThreads = 256;
constexpr int kISlots = 5;  // 4 planes in use + 1 in flight

struct InterpTiling {
  int ty, zc, nty, nzc;
  int frmax;            // field rows per slot (ty + 3, + 1 ghost row on closed y)
  uint32_t pitch;       // bytes per field row in shared memory (multiple of 1024)
  uint32_t slot_bytes;  // frmax * pitch
};

__device__ __forceinline__ uint32_t row_id(const DevGrid& g, int cyw, int czw) {
  return (uint32_t)(cyw + 1) + (uint32_t)(czw + 1) * (uint32_t)(g.n[1] + 2);
}

// Cell (unwrapped) and the four delta weights phi(sigma - t) / h of one axis.
__device__ __forceinline__ int axis_weights(const DevGrid& g, int a, double x, double w[4]) {
  double xw;
  const int c = cell_of(g, a, x, &xw);
  cosine_weights(displacement(g, a, xw, c), g.inv_h, w);
  return c;
}

__global__ void __launch_bounds__(kIThreads) interp_tma_kernel(
    DevGrid g, InterpTiling T, const __grid_constant__ CUtensorMap tmap,
    const uint32_t* __restrict__ rowstart, const double* __restrict__ rec,
    double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t raw = tma::smem_u32(smem_raw);
  const uint32_t bar0 = raw;  // kISlots mbarriers
  const uint32_t base = (raw + 8u * kISlots + 1023u) & ~1023u;
  const unsigned char* slots = smem_raw + (base - raw);

  const int tid = threadIdx.x;
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
  const int fr = hy1 - hy0 + 3;           // field rows hy0-2 .. hy1
  const int nplanes = hz1 - hz0 + 3;      // field planes hz0-2 .. hz1
  const uint32_t plane_bytes = (uint32_t)fr * (uint32_t)nx * 8u;

  if (tid == 0) {
    for (int i = 0; i < kISlots; ++i) tma::mbar_init(bar0 + 8u * i, 1);
    tma::fence_mbar_init();
  }
  __syncthreads();

  // Producer: field plane index i (plane hz0 - 2 + i) into slot i % kISlots.
  auto issue = [&](int i) {
    if (i >= nplanes) return;
    const int slot = i % kISlots;
    int t = hz0 - 2 + i;
    if (g.periodic[2]) t = wrap_cell(t, nz);
    const uint32_t bar = bar0 + 8u * slot;
    tma::mbar_expect_tx(bar, plane_bytes);
    const uint32_t dst = base + (uint32_t)slot * T.slot_bytes;
    for (int f = 0; f < fr; ++f) {
      int y = hy0 - 2 + f;
      if (g.periodic[1]) y = wrap_cell(y, ny);
      tma::load_4d(dst + (uint32_t)f * T.pitch, &tmap, 0, 0, y, t, bar);
    }
  };
  if (tid == 0)
    for (int i = 0; i < kISlots; ++i) issue(i);

  const bool px = g.periodic[0] != 0;
  for (int j = 0; j < hz1 - hz0; ++j) {
    if (j > 0) {
      __syncthreads();  // step j-1 is done with plane j-1: refill its slot
      if (tid == 0) {
        tma::fence_proxy_async();
        issue(j + kISlots - 1);
      }
    }
    // Planes j .. j+3 are this step's window; j+3 is the only new one.
    if (j == 0)
      for (int i = 0; i < 3; ++i) tma::mbar_wait(bar0 + 8u * (i % kISlots), (i / kISlots) & 1);
    tma::mbar_wait(bar0 + 8u * ((j + 3) % kISlots), ((j + 3) / kISlots) & 1);

    const int s = hz0 + j;
    const int sw = g.periodic[2] ? wrap_cell(s, nz) : s;
    const uint32_t rb = __ldg(rowstart + row_id(g, hy0, sw));
    const uint32_t re = __ldg(rowstart + row_id(g, hy1 - 1, sw) + 1);
    const unsigned char* sl[4];
#pragma unroll
    for (int kz = 0; kz < 4; ++kz) sl[kz] = slots + (size_t)((j + kz) % kISlots) * T.slot_bytes;

    for (uint32_t r = rb + tid; r < re; r += kIThreads) {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(rec) + 2 * (size_t)r);
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(rec) + 2 * (size_t)r + 1);
      const uint32_t idx = (uint32_t)__double_as_longlong(q1.y);
      double wx[4], wy[4], wz[4];
      int cx = axis_weights(g, 0, q0.x, wx);
      int cy = axis_weights(g, 1, q0.y, wy);
      axis_weights(g, 2, q1.x, wz);
      if (px) cx = wrap_cell(cx, nx);
      if (g.periodic[1]) cy = wrap_cell(cy, ny);
      uint32_t xo[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int x = cx + k - 2;
        if (px) {
          x = x < 0 ? x + nx : (x >= nx ? x - nx : x);
        } else if (x < 0 || x >= nx) {
          wx[k] = 0.0;  // off the closed grid: the reference skips the term
          x = 0;
        }
        xo[k] = tma::swz128(x);
      }
      const uint32_t f0 = (uint32_t)(cy - hy0) * T.pitch;
      double acc = 0.0;
#pragma unroll
      for (int kz = 0; kz < 4; ++kz) {
        double az = 0.0;
#pragma unroll
        for (int ky = 0; ky < 4; ++ky) {
          const unsigned char* row = sl[kz] + f0 + (uint32_t)ky * T.pitch;
          double ar = 0.0;
#pragma unroll
          for (int kx = 0; kx < 4; ++kx)
            ar = fma(wx[kx], *reinterpret_cast<const double*>(row + xo[kx]), ar);
          az = fma(wy[ky], ar, az);
        }
        acc = fma(wz[kz], az, acc);
      }
      out[idx] = acc * g.hd;
    }
  }
}

}  // namespace sw
}  // namespace ibc
