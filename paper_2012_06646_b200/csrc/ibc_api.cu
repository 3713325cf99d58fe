// ibc_api.cu -- extern "C" boundary (include/ibcuda.h).
//
// Argument validation mirrors the reference exactly (same conditions, same
// messages) so the C++ shim can rethrow the reference's exception types:
//   StaggeredGrid ctor        grid.hpp:37-60
//   check_spread_args         spread.hpp:60-66
//   check_workspace           spread.hpp:68-77
//   SpreadWorkspace ctor      spread.hpp:43-45
//   spread_buffered_otf       spread.hpp:314
//   spread_vector (null ws)   spread.hpp:335,339
//   interpolate               interpolate.hpp:27-28
#include <cuda_runtime.h>

#include <type_traits>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>
#include <cmath>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "ibc_internal.h"

struct ibc_context {
  ibc::Context c;
};
struct ibc_workspace {
  ibc::Workspace w;
};
struct ibc_binned {
  ibc::PointScratch s;
  ibc::DevGrid g{};
  ibc::InterpPlan P;
  ibc::DevBuf<double> wide;  // FP32 storage mode: the points widened to FP64
  const double* d_points = nullptr;
  size_t n = 0;
  size_t grid_points = 0;
  int device = 0;
  bool ready = false;
};

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_delta_evaluations{0};

struct ApiError {
  ibc_status status;
  std::string msg;
};

[[noreturn]] void invalid(const char* msg) { throw ApiError{IBC_ERR_INVALID_ARGUMENT, msg}; }

template <class F>
ibc_status guarded(F&& f) {
  try {
    f();
    return IBC_OK;
  } catch (const ApiError& e) {
    g_last_error = e.msg;
    return e.status;
  } catch (const ibc::ArgError& e) {
    g_last_error = e.msg;
    return IBC_ERR_INVALID_ARGUMENT;
  } catch (const ibc::CudaError& e) {
    g_last_error = e.where + ": " + cudaGetErrorString(e.code);
    return e.code == cudaErrorMemoryAllocation ? IBC_ERR_ALLOC : IBC_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    g_last_error = "allocation failed";
    return IBC_ERR_ALLOC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return IBC_ERR_CUDA;
  }
}

void check_grid(const ibc_grid* g) {
  if (!g) invalid("grid is null");
  if (g->dim < 1 || g->dim > 3) invalid("grids are 1-, 2-, or 3-dimensional");
  if (!(g->spacing > 0.0) || !std::isfinite(g->spacing)) invalid("grid spacing must be positive");
  uint64_t extended = 1;
  for (int a = 0; a < g->dim; ++a) {
    if (g->extent[a] < 1) invalid("grid extent must be >= 1");
    if (!(g->staggering[a] >= 0.0 && g->staggering[a] < 1.0))
      invalid("staggering must lie in [0, 1)");
    extended *= (uint64_t)g->extent[a] + 2;
    if (extended >= (uint64_t{1} << 32))
      throw ApiError{IBC_ERR_LENGTH, "extended grid exceeds 32-bit key range"};
  }
}

size_t grid_points(const ibc_grid* g) {
  size_t p = 1;
  for (int a = 0; a < g->dim; ++a) p *= (size_t)g->extent[a];
  return p;
}

static_assert(IBC_KERNEL_COSINE4 == ibc::kKernelCosine4 && IBC_KERNEL_PESKIN4 == ibc::kKernelPeskin4 &&
                  IBC_KERNEL_ROMA3 == ibc::kKernelRoma3 && IBC_KERNEL_LINEAR2 == ibc::kKernelLinear2,
              "kernel ids");

// check_spread_args (spread.hpp:64-65): support in [1, max_support]; the
// device takes the kernels of ibc_kernel.
void check_kernel(ibc_kernel k) {
  if (ibc::kernel_support((int)k) == 0) invalid("unsupported kernel support size");
}

void check_points(size_t n) {
  if (n > ibc::kMaxPoints) invalid("point count exceeds the device limit of 2^30 - 1");
}

uint64_t shift_count(int dim, ibc_kernel k) {  // kernel.hpp:40-45
  uint64_t s = 1;
  for (int a = 0; a < dim; ++a) s *= (uint64_t)ibc::kernel_support((int)k);
  return s;
}

void use_device(ibc::Context& c) { IBC_CUDA(cudaSetDevice(c.device)); }

constexpr size_t kPiece = size_t{8} << 20;

// Page-locked (or device / managed) memory: the copy engines reach it directly.
bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type != cudaMemoryTypeUnregistered;
}

// Host memcpy split over a small pool of host threads (one pageable <->
// pinned stage piece).  Plain std::thread: the library does not pull an
// OpenMP runtime into its callers' processes.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t kSlice = size_t{1} << 20;
    const size_t slices = (bytes + kSlice - 1) / kSlice;
    if (slices <= 1 || workers_.empty()) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::unique_lock<std::mutex> lock(call_mu_);  // one pageable copy at a time uses the pool
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      next_ = 0;
      slices_ = slices;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();  // the caller helps
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return done_ == slices_; });
  }

 private:
  CopyPool() {
    unsigned n = std::thread::hardware_concurrency();
    n = n > 8 ? 8 : n;
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  void work() {
    constexpr size_t kSlice = size_t{1} << 20;
    for (;;) {
      size_t i;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (next_ >= slices_) return;
        i = next_++;
      }
      const size_t o = i * kSlice, b = bytes_ - o < kSlice ? bytes_ - o : kSlice;
      std::memcpy(dst_ + o, src_ + o, b);
      {
        std::lock_guard<std::mutex> g(mu_);
        if (++done_ == slices_) done_cv_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, next_ = 0, slices_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  CopyPool::get().copy(dst, src, bytes);
}

// Host <-> device copy of a host-buffer call, in 8 MiB pieces.  A copy
// engine works through its queue in order, so one large transfer would hold
// back every other stream's copy in the same direction; in pieces, the copies
// of concurrent host calls (other lanes) interleave with it.  Pageable host
// memory (a std::vector behind the C++ drop-in) goes through the lane's
// pinned stage: the host copies piece k while the engine moves piece k - 1.
void host_copy(ibc::Context& c, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
               cudaStream_t st) {
  if (!bytes) return;
  const bool h2d = kind == cudaMemcpyHostToDevice;
  const void* host = h2d ? src : dst;
  if (is_pinned(host)) {
    for (size_t o = 0; o < bytes; o += kPiece) {
      const size_t b = bytes - o < kPiece ? bytes - o : kPiece;
      IBC_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, b,
                               kind, st));
    }
    return;
  }
  c.ensure_stage(kPiece);
  const size_t pieces = (bytes + kPiece - 1) / kPiece;
  for (size_t k = 0; k <= pieces; ++k) {
    // H2D: fill stage k % S on the host, then queue its DMA.
    // D2H: queue the DMA of piece k, then drain piece k - 1 on the host.
    if (k < pieces) {
      const size_t o = k * kPiece, b = bytes - o < kPiece ? bytes - o : kPiece;
      const int sl = (int)(k % ibc::Context::kStages);
      IBC_CUDA(cudaEventSynchronize(c.stage_free[sl]));  // its previous DMA is done
      if (h2d) {
        parallel_memcpy(c.stage[sl], static_cast<const char*>(src) + o, b);
        IBC_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + o, c.stage[sl], b, kind, st));
      } else {
        IBC_CUDA(cudaMemcpyAsync(c.stage[sl], static_cast<const char*>(src) + o, b, kind, st));
      }
      IBC_CUDA(cudaEventRecord(c.stage_free[sl], st));
    }
    if (!h2d && k > 0) {
      const size_t o = (k - 1) * kPiece, b = bytes - o < kPiece ? bytes - o : kPiece;
      const int sl = (int)((k - 1) % ibc::Context::kStages);
      IBC_CUDA(cudaEventSynchronize(c.stage_free[sl]));
      parallel_memcpy(static_cast<char*>(dst) + o, c.stage[sl], b);
    }
  }
}

ibc::PointScratch& spread_scratch_for(ibc::Context& c, ibc_workspace* ws, size_t n,
                                      const ibc::DevGrid& g) {
  ibc::PointScratch& s = ws ? ws->w.s : c.spread_scratch;
  if (!ws) s.reserve_points(n, true);
  else if (s.cap < n) s.reserve_points(n, true);
  s.reserve_rows(g.nrows);
  return s;
}

}  // namespace

// ---------------------------------------------------------------- Context
namespace ibc {
cudaEvent_t Context::acquire_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  IBC_CUDA(cudaEventCreate(&e));
  return e;
}
void Context::prof_begin(int, cudaEvent_t* ev) {
  *ev = nullptr;
  if (!profiling) return;
  *ev = acquire_event();
  IBC_CUDA(cudaEventRecord(*ev, stream));
}
void Context::prof_end(int cls, cudaEvent_t ev) {
  if (!profiling || !ev) return;
  cudaEvent_t e = acquire_event();
  IBC_CUDA(cudaEventRecord(e, stream));
  pending.push_back({cls, {ev, e}});
}

Context* Context::acquire_lane() {
  // A thread gets back the lane it used last when it is free: its staging and
  // scratch are already sized for that thread's calls (a lane that has to grow
  // a buffer calls cudaMalloc, which synchronizes the whole device).
  thread_local const Context* last_owner = nullptr;
  thread_local Context* last_lane = nullptr;
  Context* lane = nullptr;
  {
    std::lock_guard<std::mutex> lock(*lanes_mu);
    auto it = free_lanes.end();
    if (last_owner == this) it = std::find(free_lanes.begin(), free_lanes.end(), last_lane);
    if (it != free_lanes.end()) {
      lane = *it;
      free_lanes.erase(it);
    } else if (!free_lanes.empty()) {
      lane = free_lanes.back();
      free_lanes.pop_back();
    } else {
      auto l = std::make_unique<Context>();
      l->device = device;
      l->sms = sms;
      l->parent = this;
      IBC_CUDA(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking));
      IBC_CUDA(cudaStreamCreateWithFlags(&l->copy_stream, cudaStreamNonBlocking));
      lane = l.get();
      lanes.push_back(std::move(l));
    }
    lane->spread_path = spread_path;
    lane->profiling = profiling;
  }
  last_owner = this;
  last_lane = lane;
  // Ordered after everything already enqueued on the context's stream.
  cudaEvent_t e = lane->acquire_event();
  IBC_CUDA(cudaEventRecord(e, stream));
  IBC_CUDA(cudaStreamWaitEvent(lane->stream, e, 0));
  lane->event_pool.push_back(e);
  return lane;
}

void Context::release_lane(Context* lane) {
  std::lock_guard<std::mutex> lock(*lanes_mu);
  free_lanes.push_back(lane);
}

void Context::ensure_stage(size_t bytes) {
  if (stage_bytes >= bytes) return;
  for (int i = 0; i < kStages; ++i) {
    if (stage[i]) cudaFreeHost(stage[i]);
    stage[i] = nullptr;
    IBC_CUDA(cudaHostAlloc(&stage[i], bytes, cudaHostAllocDefault));
    if (!stage_free[i]) IBC_CUDA(cudaEventCreateWithFlags(&stage_free[i], cudaEventDisableTiming));
  }
  stage_bytes = bytes;
}

uint64_t Context::total_launches() const {
  uint64_t n = launches;
  std::lock_guard<std::mutex> lock(*lanes_mu);
  for (const auto& l : lanes) n += l->launches;
  return n;
}

void Context::release_resources() {
  for (auto& l : lanes) {
    cudaStreamSynchronize(l->stream);
    l->release_resources();
    cudaStreamDestroy(l->stream);
    cudaStreamDestroy(l->copy_stream);
  }
  lanes.clear();
  free_lanes.clear();
  spread_scratch.release_all();
  interp_scratch.release_all();
  prim_scratch.release_all();
  for (auto& b : h_stage) b.release();
  for (auto& b : wide) b.release();
  for (auto& p : pending) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  pending.clear();
  for (auto e : event_pool) cudaEventDestroy(e);
  event_pool.clear();
  for (int i = 0; i < kStages; ++i) {
    if (stage[i]) cudaFreeHost(stage[i]);
    if (stage_free[i]) cudaEventDestroy(stage_free[i]);
    stage[i] = nullptr;
    stage_free[i] = nullptr;
  }
  stage_bytes = 0;
}
}  // namespace ibc

extern "C" {

int ibc_version(void) { return IBC_API_VERSION; }
const char* ibc_last_error(void) { return g_last_error.c_str(); }

ibc_status ibc_context_create(int device, ibc_context** out) {
  return guarded([&] {
    if (!out) invalid("out is null");
    int count = 0;
    IBC_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) invalid("no such CUDA device");
    IBC_CUDA(cudaSetDevice(device));
    auto* ctx = new ibc_context();
    ctx->c.device = device;
    IBC_CUDA(cudaDeviceGetAttribute(&ctx->c.sms, cudaDevAttrMultiProcessorCount, device));
    if (ctx->c.sms < 1) ctx->c.sms = 1;
    *out = ctx;
  });
}

ibc_status ibc_context_destroy(ibc_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->c.device);
    cudaStreamSynchronize(ctx->c.stream);
    ctx->c.release_resources();
    delete ctx;
  });
}

ibc_status ibc_context_set_stream(ibc_context* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    ctx->c.stream = static_cast<cudaStream_t>(stream);
  });
}

ibc_status ibc_context_set_spread_path(ibc_context* ctx, ibc_spread_path path) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    if (path < IBC_SPREAD_PATH_AUTO || path > IBC_SPREAD_PATH_RADIX) invalid("unknown spread path");
    ctx->c.spread_path = path;
  });
}

ibc_status ibc_context_synchronize(ibc_context* ctx) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    use_device(ctx->c);
    IBC_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

ibc_status ibc_context_set_profiling(ibc_context* ctx, int on) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    ctx->c.profiling = on != 0;
  });
}

static void fold_profile(ibc::Context& c) {
  IBC_CUDA(cudaStreamSynchronize(c.stream));
  for (auto& p : c.pending) {
    float ms = 0.f;
    IBC_CUDA(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
    c.prof_ms[p.first] += ms;
    c.event_pool.push_back(p.second.first);
    c.event_pool.push_back(p.second.second);
  }
  c.pending.clear();
}

ibc_status ibc_context_get_profile(ibc_context* ctx, ibc_profile* out) {
  return guarded([&] {
    if (!ctx || !out) invalid("null argument");
    auto& c = ctx->c;
    use_device(c);
    std::lock_guard<std::mutex> lock(*c.lanes_mu);
    double ms[ibc::kProfCount] = {0, 0, 0, 0, 0, 0};
    uint64_t sc = 0, ic = 0;
    auto add = [&](ibc::Context& x) {
      fold_profile(x);
      for (int k = 0; k < ibc::kProfCount; ++k) ms[k] += x.prof_ms[k];
      sc += x.spread_calls;
      ic += x.interp_calls;
    };
    add(c);
    for (auto& l : c.lanes) add(*l);
    out->keys_ms = ms[ibc::kProfKeys];
    out->sort_ms = ms[ibc::kProfSort];
    out->rows_ms = ms[ibc::kProfRows];
    out->prep_ms = ms[ibc::kProfPrep];
    out->spread_ms = ms[ibc::kProfSpread];
    out->interp_ms = ms[ibc::kProfInterp];
    out->spread_calls = sc;
    out->interp_calls = ic;
  });
}

ibc_status ibc_context_reset_profile(ibc_context* ctx) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    auto& c = ctx->c;
    std::lock_guard<std::mutex> lock(*c.lanes_mu);
    auto reset = [](ibc::Context& x) {
      IBC_CUDA(cudaStreamSynchronize(x.stream));
      for (auto& p : x.pending) {
        x.event_pool.push_back(p.second.first);
        x.event_pool.push_back(p.second.second);
      }
      x.pending.clear();
      for (double& v : x.prof_ms) v = 0.0;
      x.spread_calls = x.interp_calls = 0;
    };
    reset(c);
    for (auto& l : c.lanes) reset(*l);
  });
}

uint64_t ibc_context_launches(const ibc_context* ctx) { return ctx ? ctx->c.total_launches() : 0; }

ibc_status ibc_grid_check(const ibc_grid* grid) { return guarded([&] { check_grid(grid); }); }

// ---------------------------------------------------------------- Workspace
ibc_status ibc_workspace_create(ibc_context* ctx, size_t n, const ibc_grid* grid, int sweep_width,
                                ibc_workspace** out) {
  return guarded([&] {
    if (!ctx || !out) invalid("null argument");
    check_grid(grid);
    if (sweep_width < 0) invalid("sweep width must be >= 1 (or 0 for none)");
    check_points(n);
    use_device(ctx->c);
    auto* ws = new ibc_workspace();
    try {
      ws->w.ctx = &ctx->c;
      ws->w.device = ctx->c.device;
      ws->w.point_count = n;
      ws->w.grid_points = grid_points(grid);
      ws->w.sweep_width = sweep_width;
      ws->w.s.reserve_points(n, true);
      ws->w.s.reserve_rows(ibc::make_devgrid(*grid, IBC_KERNEL_COSINE4).nrows);
    } catch (...) {
      ws->w.s.release_all();
      delete ws;
      throw;
    }
    *out = ws;
  });
}

ibc_status ibc_workspace_destroy(ibc_workspace* ws) {
  return guarded([&] {
    if (!ws) return;
    // No stream sync through ws->w.ctx: the context may be destroyed first
    // (e.g. garbage collection at interpreter exit); cudaFree synchronizes.
    cudaSetDevice(ws->w.device);
    ws->w.s.release_all();
    delete ws;
  });
}

ibc_status ibc_workspace_info(const ibc_workspace* ws, size_t* point_count, size_t* gp,
                              int* sweep_width) {
  return guarded([&] {
    if (!ws) invalid("workspace is null");
    if (point_count) *point_count = ws->w.point_count;
    if (gp) *gp = ws->w.grid_points;
    if (sweep_width) *sweep_width = ws->w.sweep_width;
  });
}

ibc_status ibc_workspace_run_count(ibc_workspace* ws, size_t* q) {
  return guarded([&] {
    if (!ws || !q) invalid("null argument");
    use_device(*ws->w.ctx);
    *q = ws->w.s.last_n ? ibc::read_run_count(*ws->w.ctx, ws->w.s) : 0;
  });
}

static void copy_sorted(ibc_workspace* ws, uint32_t* host, size_t n, bool perm) {
  if (!ws || (!host && n)) invalid("null argument");
  auto& s = ws->w.s;
  if (n != s.last_n) invalid("buffer size differs from the last spread's point count");
  if (!n) return;
  use_device(*ws->w.ctx);
  ibc::ensure_observables(*ws->w.ctx, s);
  IBC_CUDA(cudaMemcpyAsync(host, perm ? s.sorted_perm : s.sorted_keys, n * 4,
                           cudaMemcpyDeviceToHost, ws->w.ctx->stream));
  IBC_CUDA(cudaStreamSynchronize(ws->w.ctx->stream));
}

ibc_status ibc_workspace_get_keys(ibc_workspace* ws, uint32_t* host_keys, size_t n) {
  return guarded([&] { copy_sorted(ws, host_keys, n, false); });
}

ibc_status ibc_workspace_get_perm(ibc_workspace* ws, uint32_t* host_perm, size_t n) {
  return guarded([&] { copy_sorted(ws, host_perm, n, true); });
}

ibc_status ibc_workspace_get_run_keys(ibc_workspace* ws, uint32_t* host, size_t cap, size_t* q) {
  return guarded([&] {
    if (!ws || !q) invalid("null argument");
    auto& s = ws->w.s;
    use_device(*ws->w.ctx);
    if (!s.last_n) {
      *q = 0;
      return;
    }
    const size_t runs = ibc::compute_run_keys(*ws->w.ctx, s);
    *q = runs;
    if (!host) return;
    if (cap < runs) invalid("run key buffer too small");
    IBC_CUDA(cudaMemcpyAsync(host, s.run_keys.p, runs * 4, cudaMemcpyDeviceToHost,
                             ws->w.ctx->stream));
    IBC_CUDA(cudaStreamSynchronize(ws->w.ctx->stream));
  });
}

// ---------------------------------------------------------------- Operators
static void spread_checks(const ibc_grid* grid, ibc_kernel kernel, ibc_spread_algorithm algo,
                          size_t n_points, size_t n_values, int sweep_width, ibc_workspace* ws) {
  check_grid(grid);
  if (n_values != n_points) invalid("one value per point required");
  check_kernel(kernel);
  check_points(n_points);
  switch (algo) {
    case IBC_SPREAD_SERIAL:
      break;
    case IBC_SPREAD_FUSED:
    case IBC_SPREAD_BUFFERED: {
      if (!ws)
        invalid(algo == IBC_SPREAD_FUSED ? "fused spreading needs a workspace"
                                         : "buffered spreading needs a workspace");
      if (ws->w.point_count != n_points) invalid("workspace sized for a different point count");
      if (ws->w.grid_points != grid_points(grid)) invalid("workspace sized for a different grid");
      if (algo == IBC_SPREAD_BUFFERED && ws->w.sweep_width < 1)
        invalid("workspace has no sweep buffers");
      break;
    }
    case IBC_SPREAD_OTF:
      if (sweep_width < 1) invalid("sweep width must be >= 1");
      break;
    default:
      invalid("unknown spreading algorithm");
  }
}

// Host-buffer and device-resident operators, FP64 or the FP32 storage mode
// (T = float: inputs widened exactly to FP64 on the device, FP64 arithmetic,
// one rounding per stored result).
}  // extern "C"
namespace {
const double* as_f64(ibc::Context& c, const double* d, size_t, int) { (void)c; return d; }
const double* as_f64(ibc::Context& c, const float* d, size_t m, int slot) {
  return ibc::widen(c, d, m, c.wide[slot]);
}

template <class T>
void spread_host(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                 ibc_spread_algorithm algorithm, const T* points, const T* values, size_t n_points,
                 size_t n_values, int sweep_width, ibc_workspace* ws, T* out) {
  if (!ctx) invalid("context is null");
  spread_checks(grid, kernel, algorithm, n_points, n_values, sweep_width, ws);
  if ((!points || !values) && n_points) invalid("null input buffer");
  if (!out) invalid("null output buffer");
  use_device(ctx->c);
  ibc::Lane lane(ctx->c);
  auto& c = *lane;
  const ibc::DevGrid g = ibc::make_devgrid(*grid, (int)kernel);
  // Serial/otf own no caller workspace: they run on the context's scratch.
  ibc_workspace* use_ws =
      (algorithm == IBC_SPREAD_FUSED || algorithm == IBC_SPREAD_BUFFERED) ? ws : nullptr;
  ibc::PointScratch& s = spread_scratch_for(c, use_ws, n_points, g);
  const size_t np = grid_points(grid);
  c.h_stage[0].ensure(n_points * grid->dim);
  c.h_stage[1].ensure(n_points);
  c.h_stage[2].ensure(np);
  T* d_pts = reinterpret_cast<T*>(c.h_stage[0].p);
  T* d_val = reinterpret_cast<T*>(c.h_stage[1].p);
  T* d_out = reinterpret_cast<T*>(c.h_stage[2].p);
  if (n_points) {
    host_copy(c, d_pts, points, n_points * grid->dim * sizeof(T), cudaMemcpyHostToDevice, c.stream);
    host_copy(c, d_val, values, n_points * sizeof(T), cudaMemcpyHostToDevice, c.stream);
  }
  ibc::spread_pipeline(c, g, as_f64(c, d_pts, n_points * grid->dim, 0), as_f64(c, d_val, n_points, 1),
                       n_points, s, d_out);
  host_copy(c, out, d_out, np * sizeof(T), cudaMemcpyDeviceToHost, c.stream);
  IBC_CUDA(cudaStreamSynchronize(c.stream));
  g_delta_evaluations.fetch_add(n_points * shift_count(grid->dim, kernel), std::memory_order_relaxed);
}

template <class T>
void interp_host(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel, const T* field,
                 const T* points, size_t n_points, T* out) {
  if (!ctx) invalid("context is null");
  check_grid(grid);
  check_kernel(kernel);
  check_points(n_points);
  if (!field) invalid("null field");
  if (n_points && (!points || !out)) invalid("null point buffer");
  use_device(ctx->c);
  ibc::Lane lane(ctx->c);
  auto& c = *lane;
  const ibc::DevGrid g = ibc::make_devgrid(*grid, (int)kernel);
  const size_t np = grid_points(grid);
  c.interp_scratch.reserve_points(n_points, false);
  c.interp_scratch.reserve_rows(g.nrows);
  c.h_stage[2].ensure(np);
  c.h_stage[0].ensure(n_points * grid->dim);
  c.h_stage[3].ensure(n_points);
  T* d_pts = reinterpret_cast<T*>(c.h_stage[0].p);
  T* d_field = reinterpret_cast<T*>(c.h_stage[2].p);
  T* d_out = reinterpret_cast<T*>(c.h_stage[3].p);
  // Points first: their binning (keys, row sort, records) runs while the
  // field is still arriving on the lane's copy stream.
  if (n_points)
    host_copy(c, d_pts, points, n_points * grid->dim * sizeof(T), cudaMemcpyHostToDevice, c.stream);
  cudaEvent_t field_in = c.acquire_event();
  host_copy(c, d_field, field, np * sizeof(T), cudaMemcpyHostToDevice, c.copy_stream);
  IBC_CUDA(cudaEventRecord(field_in, c.copy_stream));
  const double* pts = as_f64(c, d_pts, n_points * grid->dim, 0);
  const ibc::InterpPlan P = ibc::interp_bin(c, g, pts, n_points, c.interp_scratch, true);
  IBC_CUDA(cudaStreamWaitEvent(c.stream, field_in, 0));
  c.event_pool.push_back(field_in);
  ibc::interp_gather(c, g, P, (const T*)d_field, pts, n_points, c.interp_scratch, d_out);
  if (n_points) host_copy(c, out, d_out, n_points * sizeof(T), cudaMemcpyDeviceToHost, c.stream);
  IBC_CUDA(cudaStreamSynchronize(c.stream));
  g_delta_evaluations.fetch_add(n_points * shift_count(grid->dim, kernel), std::memory_order_relaxed);
}

template <class T>
void spread_dev(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel, const T* d_points,
                const T* d_values, size_t n, ibc_workspace* ws, T* d_out) {
  if (!ctx) invalid("context is null");
  check_grid(grid);
  check_kernel(kernel);
  check_points(n);
  if (ws) {
    if (ws->w.point_count != n) invalid("workspace sized for a different point count");
    if (ws->w.grid_points != grid_points(grid)) invalid("workspace sized for a different grid");
  }
  if (!d_out) invalid("null output buffer");
  auto& c = ctx->c;
  use_device(c);
  const ibc::DevGrid g = ibc::make_devgrid(*grid, (int)kernel);
  ibc::PointScratch& s = spread_scratch_for(c, ws, n, g);
  ibc::spread_pipeline(c, g, as_f64(c, d_points, n * grid->dim, 0), as_f64(c, d_values, n, 1), n, s,
                       d_out);
  g_delta_evaluations.fetch_add(n * shift_count(grid->dim, kernel), std::memory_order_relaxed);
}

template <class T>
void interp_dev(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel, const T* d_field,
                const T* d_points, size_t n, T* d_out) {
  if (!ctx) invalid("context is null");
  check_grid(grid);
  check_kernel(kernel);
  check_points(n);
  auto& c = ctx->c;
  use_device(c);
  const ibc::DevGrid g = ibc::make_devgrid(*grid, (int)kernel);
  c.interp_scratch.reserve_points(n, false);
  c.interp_scratch.reserve_rows(g.nrows);
  ibc::interp_pipeline(c, g, d_field, as_f64(c, d_points, n * grid->dim, 0), n, c.interp_scratch,
                       d_out);
  g_delta_evaluations.fetch_add(n * shift_count(grid->dim, kernel), std::memory_order_relaxed);
}
}  // namespace
extern "C" {

ibc_status ibc_spread(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                      ibc_spread_algorithm algorithm, const double* points, const double* values,
                      size_t n_points, size_t n_values, int sweep_width, ibc_workspace* ws,
                      int workers, double* out) {
  (void)workers;
  return guarded([&] {
    spread_host(ctx, grid, kernel, algorithm, points, values, n_points, n_values, sweep_width, ws, out);
  });
}

ibc_status ibc_spread_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                          ibc_spread_algorithm algorithm, const float* points, const float* values,
                          size_t n_points, size_t n_values, int sweep_width, ibc_workspace* ws,
                          int workers, float* out) {
  (void)workers;
  return guarded([&] {
    spread_host(ctx, grid, kernel, algorithm, points, values, n_points, n_values, sweep_width, ws, out);
  });
}

ibc_status ibc_interpolate(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                           const double* field, const double* points, size_t n_points,
                           int workers, double* out) {
  (void)workers;
  return guarded([&] { interp_host(ctx, grid, kernel, field, points, n_points, out); });
}

ibc_status ibc_interpolate_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                               const float* field, const float* points, size_t n_points,
                               int workers, float* out) {
  (void)workers;
  return guarded([&] { interp_host(ctx, grid, kernel, field, points, n_points, out); });
}

ibc_status ibc_spread_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                             const double* d_points, const double* d_values, size_t n,
                             ibc_workspace* ws, double* d_out) {
  return guarded([&] { spread_dev(ctx, grid, kernel, d_points, d_values, n, ws, d_out); });
}

ibc_status ibc_spread_device_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                 const float* d_points, const float* d_values, size_t n,
                                 ibc_workspace* ws, float* d_out) {
  return guarded([&] { spread_dev(ctx, grid, kernel, d_points, d_values, n, ws, d_out); });
}

ibc_status ibc_interpolate_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                  const double* d_field, const double* d_points, size_t n,
                                  double* d_out) {
  return guarded([&] { interp_dev(ctx, grid, kernel, d_field, d_points, n, d_out); });
}

ibc_status ibc_interpolate_device_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                      const float* d_field, const float* d_points, size_t n,
                                      float* d_out) {
  return guarded([&] { interp_dev(ctx, grid, kernel, d_field, d_points, n, d_out); });
}

static void check_slab(const ibc_grid* grid, const ibc_slab* slab, ibc_kernel kernel) {
  if (!slab) invalid("slab is null");
  if (ibc::kernel_support((int)kernel) != ibc::kSupport)
    invalid("the slab decomposition takes 4-point kernels (2 ghost planes below, 1 above)");
  if (grid->dim < 2) invalid("slab decomposition needs a 2- or 3-dimensional grid");
  const int a = grid->dim - 1;
  if (grid->periodic[a]) invalid("the slab axis of a local grid is not periodic");
  if (slab->nz_global < 1 || grid->extent[a] < 3) invalid("bad slab extents");
}

ibc_status ibc_spread_slab_device(ibc_context* ctx, const ibc_grid* grid, const ibc_slab* slab,
                                  ibc_kernel kernel, const double* d_points,
                                  const double* d_values, size_t n, ibc_workspace* ws,
                                  double* d_out) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    check_grid(grid);
    check_slab(grid, slab, kernel);
    check_kernel(kernel);
    check_points(n);
    if (ws) {
      if (ws->w.point_count != n) invalid("workspace sized for a different point count");
      if (ws->w.grid_points != grid_points(grid)) invalid("workspace sized for a different grid");
    }
    if (!d_out) invalid("null output buffer");
    auto& c = ctx->c;
    use_device(c);
    const ibc::DevGrid g = ibc::make_devgrid(*grid, *slab, (int)kernel);
    ibc::PointScratch& s = spread_scratch_for(c, ws, n, g);
    ibc::spread_pipeline(c, g, d_points, d_values, n, s, d_out);
    g_delta_evaluations.fetch_add(n * shift_count(grid->dim, kernel), std::memory_order_relaxed);
  });
}

ibc_status ibc_interpolate_slab_device(ibc_context* ctx, const ibc_grid* grid,
                                       const ibc_slab* slab, ibc_kernel kernel,
                                       const double* d_field, const double* d_points, size_t n,
                                       double* d_out) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    check_grid(grid);
    check_slab(grid, slab, kernel);
    check_kernel(kernel);
    check_points(n);
    auto& c = ctx->c;
    use_device(c);
    const ibc::DevGrid g = ibc::make_devgrid(*grid, *slab, (int)kernel);
    c.interp_scratch.reserve_points(n, false);
    c.interp_scratch.reserve_rows(g.nrows);
    ibc::interp_pipeline(c, g, d_field, d_points, n, c.interp_scratch, d_out);
    g_delta_evaluations.fetch_add(n * shift_count(grid->dim, kernel), std::memory_order_relaxed);
  });
}

ibc_status ibc_home_planes_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                  const double* d_points, size_t n, int32_t* d_planes) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    check_grid(grid);
    check_kernel(kernel);
    check_points(n);
    if (n && (!d_points || !d_planes)) invalid("null buffer");
    auto& c = ctx->c;
    use_device(c);
    ibc::home_planes(c, ibc::make_devgrid(*grid, (int)kernel), d_points, n, d_planes);
  });
}

int ibc_kernel_support(ibc_kernel kernel) { return ibc::kernel_support((int)kernel); }

// ---------------------------------------------------------------- Binned points
ibc_status ibc_binned_create(ibc_context* ctx, ibc_binned** out) {
  return guarded([&] {
    if (!ctx || !out) invalid("null argument");
    auto* b = new ibc_binned();
    b->device = ctx->c.device;
    *out = b;
  });
}

ibc_status ibc_binned_destroy(ibc_binned* b) {
  return guarded([&] {
    if (!b) return;
    cudaSetDevice(b->device);
    b->s.release_all();
    b->wide.release();
    delete b;
  });
}

}  // extern "C"
namespace {
template <class T>
void bin_points_dev(ibc_context* ctx, ibc_binned* b, const ibc_grid* grid, ibc_kernel kernel,
                    const T* d_points, size_t n) {
  if (!ctx || !b) invalid("null argument");
  check_grid(grid);
  check_kernel(kernel);
  check_points(n);
  if (n && !d_points) invalid("null point buffer");
  auto& c = ctx->c;
  use_device(c);
  b->ready = false;
  b->g = ibc::make_devgrid(*grid, (int)kernel);
  b->s.reserve_points(n, false);
  b->s.reserve_rows(b->g.nrows);
  const double* pts = nullptr;
  if constexpr (std::is_same_v<T, float>) pts = ibc::widen(c, d_points, n * grid->dim, b->wide);
  else pts = d_points;
  b->P = ibc::interp_bin(c, b->g, pts, n, b->s, true);
  b->d_points = pts;
  b->n = n;
  b->grid_points = grid_points(grid);
  b->ready = true;
}

template <class T>
void interp_binned_dev(ibc_context* ctx, const ibc_binned* b, const T* d_field, T* d_out) {
  if (!ctx || !b) invalid("null argument");
  if (!b->ready) invalid("points have not been binned");
  if (b->n && (!d_field || !d_out)) invalid("null buffer");
  auto& c = ctx->c;
  use_device(c);
  ibc::interp_gather(c, b->g, b->P, d_field, b->d_points, b->n, const_cast<ibc::PointScratch&>(b->s),
                     d_out);
  g_delta_evaluations.fetch_add(b->n * (uint64_t)std::pow(b->g.support, b->g.dim),
                                std::memory_order_relaxed);
}
}  // namespace
extern "C" {

ibc_status ibc_bin_points_device(ibc_context* ctx, ibc_binned* b, const ibc_grid* grid,
                                 ibc_kernel kernel, const double* d_points, size_t n) {
  return guarded([&] { bin_points_dev(ctx, b, grid, kernel, d_points, n); });
}

ibc_status ibc_bin_points_device_f32(ibc_context* ctx, ibc_binned* b, const ibc_grid* grid,
                                     ibc_kernel kernel, const float* d_points, size_t n) {
  return guarded([&] { bin_points_dev(ctx, b, grid, kernel, d_points, n); });
}

ibc_status ibc_interpolate_binned_device(ibc_context* ctx, const ibc_binned* b,
                                         const double* d_field, double* d_out) {
  return guarded([&] { interp_binned_dev(ctx, b, d_field, d_out); });
}

ibc_status ibc_interpolate_binned_device_f32(ibc_context* ctx, const ibc_binned* b,
                                             const float* d_field, float* d_out) {
  return guarded([&] { interp_binned_dev(ctx, b, d_field, d_out); });
}

// ---------------------------------------------------------------- Primitives
ibc_status ibc_key_value_sort_device(ibc_context* ctx, uint32_t* d_keys, void* d_payload,
                                     size_t payload_bytes, size_t n) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    if (n && !d_keys) invalid("null key buffer");
    if (n && payload_bytes && !d_payload) invalid("null payload buffer");
    check_points(n);
    use_device(ctx->c);
    ibc::sort_keys_device(ctx->c, d_keys, payload_bytes ? d_payload : nullptr, payload_bytes, n,
                          ctx->c.prim_scratch);
  });
}

ibc_status ibc_key_value_sort(ibc_context* ctx, uint32_t* keys, void* payload, size_t payload_bytes,
                              size_t n, int workers) {
  (void)workers;
  return guarded([&] {
    if (!ctx) invalid("context is null");
    if (n && !keys) invalid("null key buffer");
    if (n && payload_bytes && !payload) invalid("null payload buffer");
    check_points(n);
    if (n < 2) return;
    use_device(ctx->c);
    ibc::Lane lane(ctx->c);
    auto& c = *lane;
    c.h_stage[0].ensure((n * 4 + 7) / 8);
    c.h_stage[1].ensure((n * payload_bytes + 7) / 8 + 1);
    auto* dk = reinterpret_cast<uint32_t*>(c.h_stage[0].p);
    void* dp = payload_bytes ? static_cast<void*>(c.h_stage[1].p) : nullptr;
    IBC_CUDA(cudaMemcpyAsync(dk, keys, n * 4, cudaMemcpyHostToDevice, c.stream));
    if (dp) IBC_CUDA(cudaMemcpyAsync(dp, payload, n * payload_bytes, cudaMemcpyHostToDevice, c.stream));
    ibc::sort_keys_device(c, dk, dp, payload_bytes, n, c.prim_scratch);
    IBC_CUDA(cudaMemcpyAsync(keys, dk, n * 4, cudaMemcpyDeviceToHost, c.stream));
    if (dp) IBC_CUDA(cudaMemcpyAsync(payload, dp, n * payload_bytes, cudaMemcpyDeviceToHost, c.stream));
    IBC_CUDA(cudaStreamSynchronize(c.stream));
  });
}

static void reduce_host(ibc_context* ctx, const uint32_t* keys, const double* values, size_t n,
                        size_t width, uint32_t* out_keys, size_t out_keys_cap, double* out_values,
                        size_t out_values_cap, size_t* q) {
  if (!ctx || !q) invalid("null argument");
  if (n && !keys) invalid("null key buffer");
  if (values && width < 1) invalid("row width must be >= 1");
  check_points(n);
  *q = 0;
  if (n == 0) return;
  use_device(ctx->c);
  ibc::Lane lane(ctx->c);
  auto& c = *lane;
  c.h_stage[0].ensure((n * 4 + 7) / 8);
  auto* dk = reinterpret_cast<uint32_t*>(c.h_stage[0].p);
  IBC_CUDA(cudaMemcpyAsync(dk, keys, n * 4, cudaMemcpyHostToDevice, c.stream));
  double* dv = nullptr;
  double* dout = nullptr;
  if (values) {
    c.h_stage[1].ensure(n * width);
    c.h_stage[2].ensure(n * width);
    dv = c.h_stage[1].p;
    dout = c.h_stage[2].p;
    IBC_CUDA(cudaMemcpyAsync(dv, values, n * width * 8, cudaMemcpyHostToDevice, c.stream));
  }
  c.h_stage[3].ensure((n * 4 + 7) / 8);
  auto* drk = reinterpret_cast<uint32_t*>(c.h_stage[3].p);
  bool unsorted = false;
  const size_t runs = ibc::runs_device(c, dk, n, c.prim_scratch, drk, dv, width, dout, &unsorted);
  if (unsorted) invalid("keys must be sorted (nondecreasing)");
  if (out_keys && out_keys_cap < runs) invalid("run key buffer too small");
  if (out_values && out_values_cap < runs * width) invalid("run value buffer too small");
  if (out_keys) IBC_CUDA(cudaMemcpyAsync(out_keys, drk, runs * 4, cudaMemcpyDeviceToHost, c.stream));
  if (out_values && dout)
    IBC_CUDA(cudaMemcpyAsync(out_values, dout, runs * width * 8, cudaMemcpyDeviceToHost, c.stream));
  IBC_CUDA(cudaStreamSynchronize(c.stream));
  *q = runs;
}

ibc_status ibc_segmented_reduce_rows(ibc_context* ctx, const uint32_t* sorted_keys,
                                     const double* values, size_t n, size_t width,
                                     uint32_t* out_keys, size_t out_keys_cap, double* out_values,
                                     size_t out_values_cap, int workers, size_t* q) {
  (void)workers;
  return guarded([&] {
    if (n && !values) invalid("null value buffer");
    reduce_host(ctx, sorted_keys, values, n, width, out_keys, out_keys_cap, out_values,
                out_values_cap, q);
  });
}

ibc_status ibc_count_unique(ibc_context* ctx, const uint32_t* sorted_keys, size_t n, int workers,
                            size_t* q) {
  (void)workers;
  return guarded([&] { reduce_host(ctx, sorted_keys, nullptr, n, 0, nullptr, 0, nullptr, 0, q); });
}

ibc_status ibc_collect_unique_keys(ibc_context* ctx, const uint32_t* sorted_keys, size_t n,
                                   uint32_t* out_keys, size_t out_cap, size_t* q) {
  return guarded([&] {
    reduce_host(ctx, sorted_keys, nullptr, n, 0, out_keys, out_cap, nullptr, 0, q);
  });
}

// ---------------------------------------------------------------- Slab peers
ibc_status ibc_device_alloc(ibc_context* ctx, size_t bytes, void** d_ptr) {
  return guarded([&] {
    if (!ctx || !d_ptr) invalid("null argument");
    use_device(ctx->c);
    IBC_CUDA(cudaMalloc(d_ptr, bytes ? bytes : 1));
  });
}

ibc_status ibc_device_free(ibc_context* ctx, void* d_ptr) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    use_device(ctx->c);
    if (d_ptr) IBC_CUDA(cudaFree(d_ptr));
  });
}

ibc_status ibc_ipc_get_handle(ibc_context* ctx, void* d_ptr, ibc_ipc_handle* out) {
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(ibc_ipc_handle), "IPC handle size");
  return guarded([&] {
    if (!ctx || !d_ptr || !out) invalid("null argument");
    use_device(ctx->c);
    cudaIpcMemHandle_t h;
    IBC_CUDA(cudaIpcGetMemHandle(&h, d_ptr));
    std::memcpy(out->bytes, &h, sizeof(h));
  });
}

ibc_status ibc_ipc_open_handle(ibc_context* ctx, const ibc_ipc_handle* h, void** d_peer) {
  return guarded([&] {
    if (!ctx || !h || !d_peer) invalid("null argument");
    use_device(ctx->c);
    cudaIpcMemHandle_t m;
    std::memcpy(&m, h->bytes, sizeof(m));
    IBC_CUDA(cudaIpcOpenMemHandle(d_peer, m, cudaIpcMemLazyEnablePeerAccess));
  });
}

ibc_status ibc_ipc_close_handle(ibc_context* ctx, void* d_peer) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    use_device(ctx->c);
    if (d_peer) IBC_CUDA(cudaIpcCloseMemHandle(d_peer));
  });
}

ibc_status ibc_slab_signals_create(ibc_context* ctx, uint64_t** d_sig) {
  return guarded([&] {
    if (!ctx || !d_sig) invalid("null argument");
    use_device(ctx->c);
    IBC_CUDA(cudaMalloc(reinterpret_cast<void**>(d_sig), 8 * sizeof(uint64_t)));
    IBC_CUDA(cudaMemset(*d_sig, 0, 8 * sizeof(uint64_t)));
  });
}

static void check_link(const ibc_slab_link* L) {
  if (!L) invalid("link is null");
  if (L->nloc < 2 || (L->has_down && L->nloc_down < 2)) invalid("a slab owns at least 2 planes");
  if (!L->d_local || !L->d_sig) invalid("null local slab or signal block");
  if (L->has_down && (!L->d_down || !L->d_sig_down)) invalid("missing the rank below's buffers");
  if (L->has_up && (!L->d_up || !L->d_sig_up)) invalid("missing the rank above's buffers");
}

ibc_status ibc_slab_ghost_sum_device(ibc_context* ctx, const ibc_slab_link* link, uint64_t epoch) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    check_link(link);
    use_device(ctx->c);
    ibc::slab_exchange(ctx->c, *link, epoch, true);
  });
}

ibc_status ibc_slab_halo_fill_device(ibc_context* ctx, const ibc_slab_link* link, uint64_t epoch) {
  return guarded([&] {
    if (!ctx) invalid("context is null");
    check_link(link);
    use_device(ctx->c);
    ibc::slab_exchange(ctx->c, *link, epoch, false);
  });
}

ibc_status ibc_slab_link_error(ibc_context* ctx, const ibc_slab_link* link, int* timed_out) {
  return guarded([&] {
    if (!ctx || !timed_out) invalid("null argument");
    check_link(link);
    use_device(ctx->c);
    uint64_t v = 0;
    IBC_CUDA(cudaMemcpyAsync(&v, link->d_sig + 7, 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    IBC_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *timed_out = v != 0;
  });
}

uint64_t ibc_fnv1a(const void* data, size_t bytes, uint64_t hash) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; ++i) {
    hash ^= p[i];
    hash *= 1099511628211ull;
  }
  return hash;
}

void ibc_add_delta_evaluations(uint64_t n) {
  g_delta_evaluations.fetch_add(n, std::memory_order_relaxed);
}

uint64_t ibc_delta_evaluations(void) { return g_delta_evaluations.load(std::memory_order_relaxed); }
void ibc_reset_delta_evaluations(void) { g_delta_evaluations.store(0, std::memory_order_relaxed); }

}  // extern "C"
