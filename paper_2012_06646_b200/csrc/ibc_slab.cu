// ibc_slab.cu -- peer-memory exchanges of the z-slab decomposition (SURVEY
// 8(e)): the ghost-plane sum after spreading and the halo fill before
// interpolating, done by pulling the ring neighbours' planes straight out of
// their slab buffers over NVLink / NVSwitch peer memory (CUDA IPC across
// processes; plain pointers within one), with device-side signal flags for
// the cross-rank ordering.  No NCCL call, no host round trip: an exchange is
// three kernels on the context stream and can be captured in a CUDA graph
// together with the local operators.
//
// Local slab layout (include/ibcuda.h ibc_slab): planes [z0 - 2, z1 + 1) of
// the global grid, local plane k = global plane z0 - 2 + k, owned planes
// k = 2 .. nloc + 1.  A point homed in [z0, z1) reaches planes z0-2 .. z1.
//   ghost sum: own[2]      += below.local[nloc_below + 2]   (below's plane z0)
//              own[nloc]   += above.local[0]                (above's z1 - 2)
//              own[nloc+1] += above.local[1]                (above's z1 - 1)
//   halo fill: local[0, 1]     = below.local[nloc_below, nloc_below + 1]
//              local[nloc + 2] = above.local[2]
// Signal block (8 x uint64, one per rank, written by the neighbours):
//   [0] ready epoch from below  [1] ready epoch from above
//   [2] done epoch from below   [3] done epoch from above
//   [4] this rank's exchange counter, [5] its current epoch (automatic epochs)
//   [7] timeout flag
#include <cuda_runtime.h>

#include <cstdint>

#include "ibc_internal.h"

namespace ibc {
namespace {

constexpr int kSigReadyDown = 0, kSigReadyUp = 1, kSigDoneDown = 2, kSigDoneUp = 3;
constexpr int kSigCount = 4, kSigEpoch = 5, kSigError = 7;
constexpr long long kSpinCycles = 4LL << 30;  // ~2 s at 1.9 GHz: a lost neighbour is an error, not a hang

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Tell the neighbours "epoch e" in slot `slot_for_below` of the rank below's
// block and `slot_for_above` of the rank above's, then wait until both
// neighbours told this rank the same (slots own_a / own_b).  One thread.
// e == 0: automatic epochs -- the "ready" handshake takes the next value of
// this rank's device-side exchange counter, the "done" handshake reuses it
// (every rank runs the same exchange sequence, so the counters agree; a
// replayed CUDA graph advances them like eager calls).
__global__ void handshake_kernel(ibc_slab_link L, uint64_t e, int slot_at_below, int slot_at_above,
                                 int own_from_below, int own_from_above, int first) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  if (e == 0) {
    if (first) {
      e = L.d_sig[kSigCount] + 1;
      L.d_sig[kSigCount] = e;
      L.d_sig[kSigEpoch] = e;
    } else {
      e = L.d_sig[kSigEpoch];
    }
  }
  __threadfence_system();  // this rank's earlier writes (slab planes) before the flag
  if (L.has_down) st_release_sys(L.d_sig_down + slot_at_below, e);
  if (L.has_up) st_release_sys(L.d_sig_up + slot_at_above, e);
  const long long t0 = clock64();
  while ((L.has_down && ld_acquire_sys(L.d_sig + own_from_below) < e) ||
         (L.has_up && ld_acquire_sys(L.d_sig + own_from_above) < e)) {
    if (clock64() - t0 > kSpinCycles) {
      st_release_sys(L.d_sig + kSigError, 1);
      return;
    }
    __nanosleep(64);
  }
}

// own planes += the neighbours' ghost planes (peer loads, 16 bytes each).
__global__ void __launch_bounds__(256) ghost_add_kernel(ibc_slab_link L) {
  pdl_wait();
  const size_t P = L.plane;
  double* own = L.d_local;
  const size_t vec = P / 2;  // double2 per plane (P even; odd tail below)
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * vec; i += stride) {
    const int which = (int)(i / vec);
    const size_t j = i - (size_t)which * vec;
    const double* src;
    double* dst;
    if (which == 0) {
      if (!L.has_down) continue;
      src = L.d_down + (size_t)(L.nloc_down + 2) * P;
      dst = own + 2 * P;
    } else {
      if (!L.has_up) continue;
      src = L.d_up + (size_t)(which - 1) * P;
      dst = own + (size_t)(L.nloc + which - 1) * P;
    }
    const double2 g = reinterpret_cast<const double2*>(src)[j];
    double2 o = reinterpret_cast<double2*>(dst)[j];
    o.x += g.x;
    o.y += g.y;
    reinterpret_cast<double2*>(dst)[j] = o;
  }
  if (P & 1 && blockIdx.x == 0 && threadIdx.x < 3) {  // odd plane size: last element
    const int which = threadIdx.x;
    if (which == 0 && L.has_down)
      own[2 * P + P - 1] += L.d_down[(size_t)(L.nloc_down + 2) * P + P - 1];
    if (which > 0 && L.has_up)
      own[(size_t)(L.nloc + which - 1) * P + P - 1] += L.d_up[(size_t)(which - 1) * P + P - 1];
  }
}

// ghost planes = the neighbours' owned edge planes (peer loads); zero on a
// closed end of the global axis.
__global__ void __launch_bounds__(256) halo_copy_kernel(ibc_slab_link L) {
  pdl_wait();
  const size_t P = L.plane;
  double* loc = L.d_local;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * P; i += stride) {
    const int which = (int)(i / P);
    const size_t j = i - (size_t)which * P;
    if (which < 2) {
      loc[(size_t)which * P + j] =
          L.has_down ? L.d_down[(size_t)(L.nloc_down + which) * P + j] : 0.0;
    } else {
      loc[(size_t)(L.nloc + 2) * P + j] = L.has_up ? L.d_up[2 * P + j] : 0.0;
    }
  }
}

}  // namespace

void slab_exchange(Context& ctx, const ibc_slab_link& L, uint64_t epoch, bool ghost_sum) {
  cudaStream_t st = ctx.stream;
  const unsigned blocks = (unsigned)ctx.sms * 4;
  // 1. "my planes are ready for epoch e" <-> the neighbours'.
  handshake_kernel<<<1, 32, 0, st>>>(L, epoch, kSigReadyUp, kSigReadyDown, kSigReadyDown,
                                     kSigReadyUp, 1);
  // 2. pull.
  if (ghost_sum) ghost_add_kernel<<<blocks, 256, 0, st>>>(L);
  else halo_copy_kernel<<<blocks, 256, 0, st>>>(L);
  // 3. "done reading your planes": afterwards both sides may overwrite.
  handshake_kernel<<<1, 32, 0, st>>>(L, epoch, kSigDoneUp, kSigDoneDown, kSigDoneDown, kSigDoneUp,
                                     0);
  ctx.launches += 3;
  IBC_CUDA(cudaGetLastError());
}

}  // namespace ibc
