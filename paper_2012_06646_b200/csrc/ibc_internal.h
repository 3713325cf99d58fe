// ibc_internal.h -- host-side objects behind the C ABI (not installed).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ibc_device.cuh"
#include "ibcuda.h"

namespace ibc {

struct CudaError {
  cudaError_t code;
  std::string where;
};

// A device-side precondition the caller violated (-> IBC_ERR_INVALID_ARGUMENT).
struct ArgError {
  std::string msg;
};

inline void check_cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw CudaError{e, where};
}
#define IBC_CUDA(x) ::ibc::check_cuda((x), #x)

// Device buffer owned by a workspace or context.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;  // elements
  void ensure(size_t n) {
    if (n <= cap && p) return;
    release();
    const size_t want = n ? n : 1;
    IBC_CUDA(cudaMalloc(&p, want * sizeof(T)));
    cap = want;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

enum ProfClass { kProfKeys = 0, kProfSort, kProfRows, kProfPrep, kProfSpread, kProfInterp, kProfCount };

// Scratch of one key-sort + tiled operator over up to `cap` points.
struct PointScratch {
  size_t cap = 0;
  DevBuf<uint32_t> keys[2], vals[2];
  DevBuf<uint32_t> hist, base, counters;  // per-tile digit histograms, digit totals
  DevBuf<uint32_t> rowstart;
  DevBuf<uint32_t> rowaux;  // bucket sort: row counts | scan status | ticket | long rows
  DevBuf<unsigned long long> bpair;  // bucket sort: (key << 32 | index) in row buckets
  DevBuf<unsigned long long> bpair_tmp;  // merge passes of rows longer than kLongSortMax
  size_t bpair_tmp_half = 0;
  const uint32_t* maxrow = nullptr;  // bucket sort: largest row count (device)
  uint32_t bank_rows = 0;            // spread: bank-mode row threshold (bucket::bank_mode)
  bool obs_pending = false;          // spread: ws.keys / ws.perm not materialised yet
  DevGrid obs_grid{};                // spread: the grid of the last spread (for them)
  DevBuf<int> rec_cx;
  DevBuf<double> rec;         // 12 x cap weight records (spread)
  DevBuf<uint32_t> run_keys;  // lazily filled
  DevBuf<uint32_t> block_counts;
  DevBuf<uint32_t> prim_u32;          // primitives: run keys + run starts
  DevBuf<unsigned char> prim_bytes;   // primitives: payload gather
  const uint32_t* sorted_keys = nullptr;
  const uint32_t* sorted_perm = nullptr;
  size_t last_n = 0;
  bool run_keys_valid = false;
  bool keys_are_rows = false;  // last sort was by row id only (interpolation)
  void reserve_points(size_t n, bool spread);
  void reserve_rows(size_t nrows);
  void release_all();
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool profiling = false;
  int spread_path = IBC_SPREAD_PATH_AUTO;  // ibc_context_set_spread_path
  int sms = 0;                             // multiprocessors of `device` (queried at creation)
  uint64_t launches = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> event_pool;
  double prof_ms[kProfCount] = {0, 0, 0, 0, 0, 0};
  uint64_t spread_calls = 0, interp_calls = 0;
  PointScratch spread_scratch;  // spreads without a user workspace
  PointScratch interp_scratch;  // interpolation
  PointScratch prim_scratch;    // sort / reduce primitives
  DevBuf<double> h_stage[4];    // device staging for host-buffer calls
  DevBuf<double> wide[2];       // FP32 storage mode: points / values widened to FP64
  cudaEvent_t acquire_event();
  void prof_begin(int cls, cudaEvent_t* ev);
  void prof_end(int cls, cudaEvent_t ev);

  // Host-buffer calls run on a lane: a sub-context with its own stream,
  // staging and scratch, ordered after the work already on `stream`.  Host
  // calls from different threads (the reference's threading contract:
  // concurrent calls on disjoint outputs are safe, spread.hpp:26) then
  // overlap on the device and on both PCIe directions.
  Context* parent = nullptr;
  cudaStream_t copy_stream = nullptr;  // lanes: a second stream for overlapped copies
  // Pinned stage for pageable host buffers (host_copy in ibc_api.cu).
  static constexpr int kStages = 3;
  void* stage[kStages] = {nullptr, nullptr, nullptr};
  cudaEvent_t stage_free[kStages] = {nullptr, nullptr, nullptr};
  size_t stage_bytes = 0;
  void ensure_stage(size_t bytes);
  std::unique_ptr<std::mutex> lanes_mu = std::make_unique<std::mutex>();
  std::vector<std::unique_ptr<Context>> lanes;
  std::vector<Context*> free_lanes;
  Context* acquire_lane();
  void release_lane(Context* lane);
  uint64_t total_launches() const;
  void release_resources();  // scratch, staging, events, lanes (not the user's stream)
};

// RAII lane of a context for one host-buffer call.
class Lane {
 public:
  explicit Lane(Context& c) : parent_(c), lane_(c.acquire_lane()) {}
  ~Lane() { parent_.release_lane(lane_); }
  Lane(const Lane&) = delete;
  Lane& operator=(const Lane&) = delete;
  Context& operator*() const { return *lane_; }

 private:
  Context& parent_;
  Context* lane_;
};

struct Workspace {
  Context* ctx = nullptr;
  int device = 0;  // destroy must not touch ctx (it may already be gone)
  size_t point_count = 0;
  size_t grid_points = 0;
  int sweep_width = 0;
  PointScratch s;
};

// Pipelines (ibc_kernels.cu).  All enqueue on ctx.stream; no host sync.
DevGrid make_devgrid(const ibc_grid& g, int kernel);
DevGrid make_devgrid(const ibc_grid& g, const ibc_slab& slab, int kernel);  // z-slab of a larger grid
// Support of a kernel id (ibc_kernel); 0 for an unknown id.
inline int kernel_support(int k) {
  switch (k) {
    case kKernelCosine4: case kKernelPeskin4: return 4;
    case kKernelRoma3: return 3;
    case kKernelLinear2: return 2;
    default: return 0;
  }
}
// Wrapped home cell along the last axis of every point (slab binning key).
void home_planes(Context& ctx, const DevGrid& g, const double* d_points, size_t n, int* d_planes);
// TO / TF: the grid value type in memory (double; float in the FP32 storage
// mode -- points and values are widened to double before the pipeline, all
// arithmetic is FP64, one rounding at the store).
template <typename TO>
void spread_pipeline(Context& ctx, const DevGrid& g, const double* d_points,
                     const double* d_values, size_t n, PointScratch& s, TO* d_out);
// Interpolation split into a field-independent binning and the gather.
struct InterpPlan {
  bool tma = false;
  sw::InterpTiling T{};
};
InterpPlan interp_bin(Context& ctx, const DevGrid& g, const double* d_points, size_t n,
                      PointScratch& s, bool allow_tma);
template <typename TF>
void interp_gather(Context& ctx, const DevGrid& g, const InterpPlan& P, const TF* d_field,
                   const double* d_points, size_t n, PointScratch& s, TF* d_out);
template <typename TF>
void interp_pipeline(Context& ctx, const DevGrid& g, const TF* d_field,
                     const double* d_points, size_t n, PointScratch& s, TF* d_out);
// FP32 storage mode: m floats widened (exactly) to doubles in buf, on ctx.stream.
const double* widen(Context& ctx, const float* d_in, size_t m, DevBuf<double>& buf);
// ws.run_keys on the device; returns q (synchronizes).
size_t compute_run_keys(Context& ctx, PointScratch& s);
// The stable (key, index) order of the last spread (ws.keys / ws.perm), on request.
void ensure_observables(Context& ctx, PointScratch& s);
size_t read_run_count(Context& ctx, PointScratch& s);

// Peer-memory slab exchange (ibc_slab.cu): ghost_sum or halo fill.
void slab_exchange(Context& ctx, const ibc_slab_link& L, uint64_t epoch, bool ghost_sum);

// Primitives (sort.hpp / reduce.hpp) on device buffers, in the context stream.
// Stable sort of n 32-bit keys in place, with a payload of `bytes` bytes per
// key (may be null).
void sort_keys_device(Context& ctx, uint32_t* d_keys, void* d_payload, size_t bytes, size_t n,
                      PointScratch& s);
// Runs of sorted keys: q (synchronizes); run keys to d_run_keys (may be
// null); with values, the left fold of each run's rows of `width` doubles to
// d_out.  *unsorted: some key decreases.
size_t runs_device(Context& ctx, const uint32_t* d_keys, size_t n, PointScratch& s,
                   uint32_t* d_run_keys, const double* d_values, size_t width, double* d_out,
                   bool* unsorted);

}  // namespace ibc
