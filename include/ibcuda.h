/*
 * ibcuda.h -- C ABI of the B200-native immersed-boundary coupling library
 * (libibcuda.so, built from paper_2012_06646_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/ib/, a header-only C++20 template library).
 * Each entry point names the reference interface it replaces.  The C++
 * shim include/ib_b200/ib.hpp re-exposes these as the reference's own
 * ib:: templates (same names, argument meaning and exceptions); the ctypes
 * binding paper_2012_06646_b200/_capi.py is what tests and bench.py use.
 *
 * Conventions
 *  - Points are AoS, n x dim doubles (ib::PointSet<D> = vector<array<double,D>>,
 *    grid.hpp:187-188).  Fields are colexicographic, axis 0 fastest
 *    (ib::GridField<D>, grid.hpp:85-92).
 *  - Status codes mirror the reference's exceptions:
 *      IBC_ERR_INVALID_ARGUMENT <-> std::invalid_argument
 *      IBC_ERR_LENGTH           <-> std::length_error
 *      IBC_ERR_ALLOC            <-> std::bad_alloc (workspace construction)
 *    ibc_last_error() returns the message of the calling thread's last failure.
 *  - Host-buffer entry points (ibc_spread, ibc_interpolate) are synchronous,
 *    like the reference calls.  *_device entry points take device pointers,
 *    enqueue on the context's stream and return immediately; they never
 *    allocate or synchronize once the workspace/context scratch is sized, so
 *    they may be captured in a CUDA graph.
 *  - `workers` is accepted for signature compatibility with the reference and
 *    ignored: the device decides its own parallelism.
 *  - Results are deterministic: repeated calls on the same inputs are bitwise
 *    identical (no floating-point atomics anywhere on the path).
 */
#ifndef IBCUDA_H
#define IBCUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IBC_API_VERSION 1

typedef enum {
  IBC_OK = 0,
  IBC_ERR_INVALID_ARGUMENT = 1,
  IBC_ERR_LENGTH = 2,
  IBC_ERR_CUDA = 3,
  IBC_ERR_ALLOC = 4
} ibc_status;

/* Delta kernels (the reference's Kernel concept, kernel.hpp:16-21, is a
 * compile-time template parameter; the device takes these, by id).
 *   COSINE4  the reference's CosineKernel: phi(r) = (1 + cos(pi r / 2)) / 4 on
 *            |r| < 2, support 4 (kernel.hpp:23-36);
 *   PESKIN4  Peskin's standard 4-point kernel (Peskin 2002, Eq. 6.27):
 *            (3 - 2|r| + sqrt(1 + 4|r| - 4r^2)) / 8 on |r| <= 1,
 *            (5 - 2|r| - sqrt(-7 + 12|r| - 4r^2)) / 8 on 1 < |r| < 2;
 *   ROMA3    the 3-point kernel of Roma, Peskin & Berger (1999), odd support
 *            (cell_index half = 0.5, grid.hpp:121-130):
 *            (1 + sqrt(1 - 3r^2)) / 3 on |r| <= 1/2,
 *            (5 - 3|r| - sqrt(1 - 3(1 - |r|)^2)) / 6 on 1/2 < |r| < 3/2;
 *   LINEAR2  the 2-point hat, 1 - |r| on |r| < 1.
 * Support-4 kernels run the fast paths (bank / pull sweeps, TMA gather);
 * the others the generic radix-sorted tiles.  Unknown ids are rejected with
 * IBC_ERR_INVALID_ARGUMENT ("unsupported kernel support size",
 * spread.hpp:64-65). */
typedef enum {
  IBC_KERNEL_COSINE4 = 0,
  IBC_KERNEL_PESKIN4 = 1,
  IBC_KERNEL_ROMA3 = 2,
  IBC_KERNEL_LINEAR2 = 3
} ibc_kernel;

/* Kernel::support() of an id (kernel.hpp:34); 0 for an unknown id. */
int ibc_kernel_support(ibc_kernel kernel);

/* ib::SpreadAlgorithm (spread.hpp:21).  Every algorithm computes the same
 * operator; on the device all of them run the write-once tiled spread. */
typedef enum {
  IBC_SPREAD_SERIAL = 0,
  IBC_SPREAD_FUSED = 1,
  IBC_SPREAD_BUFFERED = 2,
  IBC_SPREAD_OTF = 3
} ibc_spread_algorithm;

/* ib::StaggeredGrid<D> (grid.hpp:33-83).  Entries past `dim` are ignored. */
typedef struct {
  int dim;              /* 1..3 */
  int extent[3];        /* grid points per axis, >= 1 */
  double spacing;       /* h > 0 */
  double staggering[3]; /* alpha in [0, 1) */
  int periodic[3];      /* 0 / 1 */
  double origin[3];
} ibc_grid;

typedef struct ibc_context ibc_context;
typedef struct ibc_workspace ibc_workspace;

/* Per-kernel-class device times (ms) accumulated while profiling is on. */
typedef struct {
  double keys_ms;    /* fused cell-key + radix-histogram kernel      */
  double sort_ms;    /* digit scan + onesweep passes                 */
  double rows_ms;    /* row-start table + run count                  */
  double prep_ms;    /* sorted per-point weight records (spread)     */
  double spread_ms;  /* write-once tiled spread                      */
  double interp_ms;  /* interpolation gather                          */
  uint64_t spread_calls;
  uint64_t interp_calls;
} ibc_profile;

int ibc_version(void);
const char* ibc_last_error(void);

/* Context = device + stream + scratch.  Replaces the reference's implicit
 * OpenMP team (parallel.hpp:25-36). */
ibc_status ibc_context_create(int device, ibc_context** out);
ibc_status ibc_context_destroy(ibc_context* ctx);
/* cudaStream_t to enqueue on (NULL = the legacy default stream). */
ibc_status ibc_context_set_stream(ibc_context* ctx, void* stream);
ibc_status ibc_context_synchronize(ibc_context* ctx);
ibc_status ibc_context_set_profiling(ibc_context* ctx, int on);
ibc_status ibc_context_get_profile(ibc_context* ctx, ibc_profile* out); /* synchronizes */
ibc_status ibc_context_reset_profile(ibc_context* ctx);
/* Number of device kernels this context has launched so far. */
uint64_t ibc_context_launches(const ibc_context* ctx);

/* Spread path selection.  AUTO (the default) picks per call on the device
 * from the densest row / fullest bucket of the bucket sort; the others force
 * one path (all compute the same operator; tests run each against the
 * oracle): BANK -- bucket sort + bank-mode sweep, PULL -- bucket sort + row
 * ranking + pull-mode sweep, RADIX -- stable onesweep radix sort + pull-mode
 * sweep. */
typedef enum {
  IBC_SPREAD_PATH_AUTO = 0,
  IBC_SPREAD_PATH_BANK = 1,
  IBC_SPREAD_PATH_PULL = 2,
  IBC_SPREAD_PATH_RADIX = 3
} ibc_spread_path;
ibc_status ibc_context_set_spread_path(ibc_context* ctx, ibc_spread_path path);

/* StaggeredGrid<D> constructor validation (grid.hpp:37-60). */
ibc_status ibc_grid_check(const ibc_grid* grid);

/* ib::SpreadWorkspace<D>(n, grid, b) (spread.hpp:27-56): device buffers sized
 * once for (point count, grid, sweep width).  b < 0 -> invalid_argument. */
ibc_status ibc_workspace_create(ibc_context* ctx, size_t n, const ibc_grid* grid,
                                int sweep_width, ibc_workspace** out);
ibc_status ibc_workspace_destroy(ibc_workspace* ws);
ibc_status ibc_workspace_info(const ibc_workspace* ws, size_t* point_count,
                              size_t* grid_points, int* sweep_width);
/* Observable results of the most recent spread through `ws` (synchronize):
 * ws.run_count, ws.keys (sorted), ws.perm, ws.run_keys[0..q) (spread.hpp:33-41).
 * The spread itself only buckets the points; the stable (key, index) order
 * is computed on the first of these calls after it (bit-exact with the
 * reference's key_value_sort, sort.hpp:17-71). */
ibc_status ibc_workspace_run_count(ibc_workspace* ws, size_t* q);
ibc_status ibc_workspace_get_keys(ibc_workspace* ws, uint32_t* host_keys, size_t n);
ibc_status ibc_workspace_get_perm(ibc_workspace* ws, uint32_t* host_perm, size_t n);
ibc_status ibc_workspace_get_run_keys(ibc_workspace* ws, uint32_t* host_run_keys, size_t cap,
                                      size_t* q);

/* Spreading, host buffers.  Replaces ib::spread_serial (spread.hpp:129-131),
 * ib::spread_fused (:165-168), ib::spread_buffered (:223-226) and
 * ib::spread_buffered_otf (:309-313) -- selected by `algorithm` with the
 * reference's argument checks (:60-77, :314).  `ws` is required for FUSED and
 * BUFFERED (BUFFERED additionally needs sweep_width >= 1 in ws), ignored
 * otherwise.  out: prod(extent) doubles, fully overwritten. */
ibc_status ibc_spread(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                      ibc_spread_algorithm algorithm, const double* points,
                      const double* values, size_t n_points, size_t n_values,
                      int sweep_width, ibc_workspace* ws, int workers, double* out);

/* Interpolation, host buffers.  Replaces ib::interpolate (interpolate.hpp:22-24). */
ibc_status ibc_interpolate(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                           const double* field, const double* points, size_t n_points,
                           int workers, double* out);

/* Device-resident variants (async on the context stream).  `ws` may be NULL
 * (context scratch is used).  d_out of the spread is fully overwritten. */
ibc_status ibc_spread_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                             const double* d_points, const double* d_values, size_t n,
                             ibc_workspace* ws, double* d_out);
ibc_status ibc_interpolate_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                  const double* d_field, const double* d_points, size_t n,
                                  double* d_out);

/* FP32 storage mode (the SURVEY 8(b) precision F32; the reference itself is
 * FP64-only): points, values, fields and results are float in memory.  The
 * inputs are widened exactly to double on the device, cells / weights / sums
 * are the FP64 operator above, and each result is rounded once when stored
 * -- so a result differs from the FP64 operator on the same (float-valued)
 * inputs by that one rounding.  Same arguments, checks and errors as the
 * FP64 entry points (binned points: ibc_bin_points_device_f32 below);
 * multi-GPU slabs stay FP64. */
ibc_status ibc_spread_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                          ibc_spread_algorithm algorithm, const float* points,
                          const float* values, size_t n_points, size_t n_values,
                          int sweep_width, ibc_workspace* ws, int workers, float* out);
ibc_status ibc_interpolate_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                               const float* field, const float* points, size_t n_points,
                               int workers, float* out);
ibc_status ibc_spread_device_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                 const float* d_points, const float* d_values, size_t n,
                                 ibc_workspace* ws, float* d_out);
ibc_status ibc_interpolate_device_f32(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                      const float* d_field, const float* d_points, size_t n,
                                      float* d_out);

/* Binned points: the field-independent half of an interpolation (cell keys,
 * row bucket sort, per-point weight records), kept so several fields can be
 * interpolated at the same points -- the reference's step interpolates the
 * same velocity at X^n twice (bench/run.hpp:94-115) and a vector field is 3
 * fields.  ibc_interpolate_binned_device(ctx, b, f, out) equals
 * ibc_interpolate_device(ctx, grid, kernel, f, points, n, out) bit for bit.
 * The binning refers to d_points (the generic path re-reads them): they must
 * stay allocated and unchanged until it is rebinned or destroyed.  Both calls
 * are asynchronous on the context stream; a binning is not shared between
 * concurrent calls. */
typedef struct ibc_binned ibc_binned;
ibc_status ibc_binned_create(ibc_context* ctx, ibc_binned** out);
ibc_status ibc_binned_destroy(ibc_binned* b);
ibc_status ibc_bin_points_device(ibc_context* ctx, ibc_binned* b, const ibc_grid* grid,
                                 ibc_kernel kernel, const double* d_points, size_t n);
ibc_status ibc_interpolate_binned_device(ibc_context* ctx, const ibc_binned* b,
                                         const double* d_field, double* d_out);
/* The FP32 storage mode of the two (float points / fields / results, FP64
 * arithmetic; the binning keeps its own widened copy of the points). */
ibc_status ibc_bin_points_device_f32(ibc_context* ctx, ibc_binned* b, const ibc_grid* grid,
                                     ibc_kernel kernel, const float* d_points, size_t n);
ibc_status ibc_interpolate_binned_device_f32(ibc_context* ctx, const ibc_binned* b,
                                             const float* d_field, float* d_out);

/* Multi-GPU z-slab decomposition (no reference analog: the
 * paper defers multi-device runs).  A rank owns home planes
 * [z0, z1) of the last axis of a global grid and works on a LOCAL grid of
 * planes [z0 - 2, z1 + 1): same extents/spacing/staggering/origin as the
 * global grid except extent[dim-1] = z1 - z0 + 3 and periodic[dim-1] = 0.
 * Cells along that axis are computed in global coordinates (bit-identical to
 * the single-grid keys) and shifted by z_first = z0 - 2, so a point homed in
 * [z0, z1) spreads into local planes [0, z1 - z0 + 3) with no loss, and reads
 * them when interpolating.  The ghost-plane sum after spreading and the halo
 * fill before interpolating are the caller's exchange (paper_2012_06646_b200/
 * slab.py, NCCL send/recv between ring neighbours). */
typedef struct {
  int z_first;          /* global plane of local plane 0 (z0 - 2) */
  int nz_global;        /* global extent of the last axis */
  int periodic_global;  /* global periodicity of the last axis */
} ibc_slab;

ibc_status ibc_spread_slab_device(ibc_context* ctx, const ibc_grid* local_grid,
                                  const ibc_slab* slab, ibc_kernel kernel, const double* d_points,
                                  const double* d_values, size_t n, ibc_workspace* ws,
                                  double* d_out);
ibc_status ibc_interpolate_slab_device(ibc_context* ctx, const ibc_grid* local_grid,
                                       const ibc_slab* slab, ibc_kernel kernel,
                                       const double* d_field, const double* d_points, size_t n,
                                       double* d_out);
/* ---- Peer-memory exchanges of the slab decomposition (NVLink / NVSwitch).
 * Each rank shares its local slab buffer and an 8-word signal block with its
 * ring neighbours -- CUDA IPC handles across processes (ibc_ipc_*), plain
 * device pointers within one process -- and each exchange pulls the
 * neighbours' planes straight out of their buffers with one kernel, ordered
 * across ranks by device-side release/acquire flags (a handshake kernel
 * before and after it).  No NCCL, no host synchronisation: capturable in a
 * CUDA graph with the local operators.  Every rank calls the same sequence of
 * exchanges, either with the same strictly increasing epochs (>= 1) or with
 * epoch 0 = automatic (a device-side counter per rank: what a replayed CUDA
 * graph needs; do not mix the two on one signal block).  A neighbour that never
 * arrives sets the signal block's timeout flag after ~2 s instead of hanging
 * the device (ibc_slab_link_error). */
typedef struct {
  int nloc;              /* owned planes of this rank, z1 - z0 (>= 2) */
  int nloc_down;         /* owned planes of the rank below */
  size_t plane;          /* values per plane: prod of the other extents */
  int has_down, has_up;  /* 0 at a closed end of the global axis */
  double* d_local;       /* this rank's local slab: nloc + 3 planes */
  const double* d_down;  /* the rank below's local slab (peer pointer) */
  const double* d_up;    /* the rank above's local slab (peer pointer) */
  uint64_t* d_sig;       /* this rank's signal block (ibc_slab_signals_create) */
  uint64_t* d_sig_down;  /* the rank below's signal block (peer pointer) */
  uint64_t* d_sig_up;    /* the rank above's signal block (peer pointer) */
} ibc_slab_link;

typedef struct {
  unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} ibc_ipc_handle;

/* cudaMalloc'd device memory (a whole allocation: shareable by IPC). */
ibc_status ibc_device_alloc(ibc_context* ctx, size_t bytes, void** d_ptr);
ibc_status ibc_device_free(ibc_context* ctx, void* d_ptr);
ibc_status ibc_ipc_get_handle(ibc_context* ctx, void* d_ptr, ibc_ipc_handle* out);
ibc_status ibc_ipc_open_handle(ibc_context* ctx, const ibc_ipc_handle* h, void** d_peer);
ibc_status ibc_ipc_close_handle(ibc_context* ctx, void* d_peer);
/* An 8 x uint64 signal block, zeroed (a whole allocation). */
ibc_status ibc_slab_signals_create(ibc_context* ctx, uint64_t** d_sig);
/* Ghost-plane sum after the local spread into link->d_local (ibc_spread_slab_device):
 * own[2] += below's plane z0, own[nloc], own[nloc+1] += above's planes z1-2, z1-1. */
ibc_status ibc_slab_ghost_sum_device(ibc_context* ctx, const ibc_slab_link* link, uint64_t epoch);
/* Halo fill before the local gather: link->d_local's planes 0, 1 and nloc+2 from
 * the neighbours' owned planes (zero at a closed end). */
ibc_status ibc_slab_halo_fill_device(ibc_context* ctx, const ibc_slab_link* link, uint64_t epoch);
/* 1 if a handshake on this rank timed out (synchronizes the context stream). */
ibc_status ibc_slab_link_error(ibc_context* ctx, const ibc_slab_link* link, int* timed_out);

/* Wrapped home cell along the last axis (cell_index + wrap, grid.hpp:121-151)
 * of every point of a global grid: the slab each point belongs to. */
ibc_status ibc_home_planes_device(ibc_context* ctx, const ibc_grid* grid, ibc_kernel kernel,
                                  const double* d_points, size_t n, int32_t* d_planes);

/* ---- Primitives of the reference's sort / reduce API (sort.hpp, reduce.hpp).
 * The operators never call these (their sort and reduction are fused into the
 * bucket sort and the write-once sweeps); they are exported so the
 * reference's own callers of the primitives (bench/verify.hpp:234-322,
 * tests/primitives_test.cpp) run on the device too.  Host-buffer forms are
 * synchronous; `workers` is accepted and ignored. */

/* ib::key_value_sort<Payload> (sort.hpp:16-71): stable LSD radix sort of n
 * 32-bit keys, in place, carrying a payload of payload_bytes bytes per key
 * (4 for uint32_t; 0 = none).  Bit-identical to std::stable_sort by key. */
ibc_status ibc_key_value_sort(ibc_context* ctx, uint32_t* keys, void* payload,
                              size_t payload_bytes, size_t n, int workers);
ibc_status ibc_key_value_sort_device(ibc_context* ctx, uint32_t* d_keys, void* d_payload,
                                     size_t payload_bytes, size_t n); /* async */
/* ib::segmented_reduce_rows (reduce.hpp:70-137; ib::segmented_reduce at
 * width 1, :139-145): sums consecutive rows of `width` doubles while their
 * (nondecreasing) keys match; writes q run keys and q summed rows.  Each run
 * is a left fold in index order (the reference at workers == 1, bit for
 * bit).  Decreasing keys -> IBC_ERR_INVALID_ARGUMENT (the reference asserts). */
ibc_status ibc_segmented_reduce_rows(ibc_context* ctx, const uint32_t* sorted_keys,
                                     const double* values, size_t n, size_t width,
                                     uint32_t* out_keys, size_t out_keys_cap, double* out_values,
                                     size_t out_values_cap, int workers, size_t* q);
/* ib::count_unique (reduce.hpp:57-69) and detail::collect_unique_keys
 * (:36-52): number of runs / the run keys of sorted keys. */
ibc_status ibc_count_unique(ibc_context* ctx, const uint32_t* sorted_keys, size_t n, int workers,
                            size_t* q);
ibc_status ibc_collect_unique_keys(ibc_context* ctx, const uint32_t* sorted_keys, size_t n,
                                   uint32_t* out_keys, size_t out_cap, size_t* q);

/* ib::stats (stats.hpp:9-25): every operation adds n_points * support^dim. */
uint64_t ibc_delta_evaluations(void);
void ibc_reset_delta_evaluations(void);
/* ib::bench::fnv1a (bench/run.hpp:44-52): 64-bit FNV-1a of `bytes` bytes
 * continuing from `hash` (14695981039346656037 to start) -- the step loop's
 * physics fingerprint (run.hpp:120-126), host memory. */
uint64_t ibc_fnv1a(const void* data, size_t bytes, uint64_t hash);
/* ib::stats::add_delta_evaluations (stats.hpp:23-25). */
void ibc_add_delta_evaluations(uint64_t n);

#ifdef __cplusplus
}
#endif
#endif /* IBCUDA_H */
