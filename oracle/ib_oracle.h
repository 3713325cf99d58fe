/*
 * ib_oracle.h -- CPU restatement of the reference IB coupling algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2012_06646_b200/_lib/libibcuda.so) never links or calls it.
 *
 * Every function restates one reference function (file:line into
 * /root/reference/proj/include/ib/) for the 4-point cosine kernel; the
 * arithmetic is written in the same operation order so that integer outputs
 * (keys, permutations, run counts) are bit-exact and floating-point outputs
 * round identically on an x86-64 baseline build without FMA contraction.
 *
 * Parity pinning: oracle outputs are checked against (a) the reference's
 * own known-answer tests (tests/grid_test.cpp, kernel_test.cpp,
 * primitives_test.cpp, coupling_test.cpp) re-asserted in
 * tests/test_oracle_kat.py and (b) golden vectors produced by the reference
 * headers themselves, compiled by oracle/Makefile into oracle/_ref/ and
 * frozen under tests/golden/ by tests/golden/make_golden.py.
 */
#ifndef IB_ORACLE_H
#define IB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as ibc_grid in include/ibcuda.h (StaggeredGrid<D>, grid.hpp:33-83). */
typedef struct {
  int dim;
  int extent[3];
  double spacing;
  double staggering[3];
  int periodic[3];
  double origin[3];
} or_grid;

/* 0 ok, 1 invalid_argument, 2 length_error (grid.hpp:37-60). */
int or_grid_check(const or_grid* g);

void or_wrap_position(const or_grid* g, const double* x, double* w);       /* grid.hpp:197-207 */
void or_cell_index(const or_grid* g, const double* x, int support, int* i); /* grid.hpp:121-130 */
void or_point_of(const or_grid* g, const int* i, double* x);               /* grid.hpp:106-111 */
uint32_t or_grid_index(const or_grid* g, const int* i);                    /* grid.hpp:136-151 */
uint32_t or_cell_key(const or_grid* g, const int* i);                      /* grid.hpp:158-170 */
void or_cell_key_inverse(const or_grid* g, uint32_t k, int* i);            /* grid.hpp:174-184 */
double or_cosine_phi(double r);                                            /* kernel.hpp:24-27 */
void or_shift(int dim, int64_t j, int support, int* sigma);                /* kernel.hpp:49-58 */
double or_delta_weight(int dim, const double* dx, const int* sigma, double h); /* kernel.hpp:64-69 */

/* Stable LSD radix sort, 4 x 8-bit passes (sort.hpp:17-71 at workers=1). */
void or_key_value_sort(uint32_t* keys, uint32_t* payload, size_t n);
/* Run heads of a sorted key array (reduce.hpp:36-52); returns q. */
size_t or_collect_unique_keys(const uint32_t* sorted, size_t n, uint32_t* out_keys);
/* Left-fold segmented reduce (reduce.hpp:80-145 at workers=1); returns q. */
size_t or_segmented_reduce(const uint32_t* sorted, const double* values, size_t n,
                           uint32_t* out_keys, double* out_sums);

/* Keys of every point + sort + unique (spread.hpp:88-103). Returns q. */
size_t or_prepare_keys(const or_grid* g, const double* points, size_t n, uint32_t* keys,
                       uint32_t* perm, uint32_t* run_keys);

/* Algorithm 2 (spread.hpp:129-159).  out has prod(extent) entries. */
int or_spread_serial(const or_grid* g, const double* points, const double* values, size_t n,
                     double* out);
/* Algorithm 4 at workers=1 (spread.hpp:165-216).  keys/perm/run_keys are n
 * entries each (may be NULL); *q receives ws.run_count. */
int or_spread_fused(const or_grid* g, const double* points, const double* values, size_t n,
                    double* out, uint32_t* keys, uint32_t* perm, uint32_t* run_keys, size_t* q);
/* Algorithm 3 (interpolate.hpp:22-58). */
int or_interpolate(const or_grid* g, const double* field, const double* points, size_t n,
                   double* out);

/* Kernel-generic forms (kernel ids of include/ibcuda.h: 0 cosine, 1 Peskin
 * 4-point, 2 Roma 3-point, 3 hat): the reference's templates over other
 * Kernel types (kernel.hpp:16-21; odd support: grid.hpp:121-130). */
int or_kernel_support(int kernel);
double or_kernel_phi(int kernel, double r);
size_t or_prepare_keys_k(const or_grid* g, int kernel, const double* points, size_t n,
                         uint32_t* keys, uint32_t* perm, uint32_t* run_keys);
int or_spread_serial_k(const or_grid* g, int kernel, const double* points, const double* values,
                       size_t n, double* out);
int or_spread_fused_k(const or_grid* g, int kernel, const double* points, const double* values,
                      size_t n, double* out, uint32_t* keys, uint32_t* perm, uint32_t* run_keys,
                      size_t* q);
int or_interpolate_k(const or_grid* g, int kernel, const double* field, const double* points,
                     size_t n, double* out);

/* Home cells of n points (periodic axes wrapped into [0, n) when wrap != 0). */
void or_home_cells(const or_grid* g, const double* points, size_t n, int support, int wrap,
                   int32_t* out /* n * dim */);

/* Deterministic synthetic inputs used by tests and the CPU baseline:
 * scatter_points (bench/setup.hpp:46-53): mt19937_64(seed), (rng()>>11)*2^-53*edge. */
void or_scatter_points(uint64_t n, double edge, uint64_t seed, double* out /* n*3 */);

#ifdef __cplusplus
}
#endif
#endif
