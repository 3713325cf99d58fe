/*
 * ib_oracle.c -- CPU restatement of the reference IB coupling path.
 * TEST INFRASTRUCTURE ONLY (see ib_oracle.h).  Citations are file:line into
 * /root/reference/proj/include/ib/.
 *
 * Build: oracle/Makefile (gcc -O2 -std=c11 -ffp-contract=off): no FMA
 * contraction, matching the reference's CMake Release build on x86-64.
 */
#include "ib_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_PI 3.14159265358979323846 /* std::numbers::pi */
#define OR_SUPPORT 4              /* CosineKernel::support (kernel.hpp:34) */
#define OR_MAX_SUPPORT 8          /* detail::max_support (support_window.hpp:11) */
static const int64_t or_invalid_offset = INT64_MIN / 4; /* support_window.hpp:15-16 */

int or_grid_check(const or_grid* g) {
  /* StaggeredGrid ctor (grid.hpp:37-60). */
  if (g->dim < 1 || g->dim > 3) return 1;
  if (!(g->spacing > 0.0) || !isfinite(g->spacing)) return 1;
  uint64_t extended = 1;
  for (int a = 0; a < g->dim; ++a) {
    if (g->extent[a] < 1) return 1;
    if (!(g->staggering[a] >= 0.0 && g->staggering[a] < 1.0)) return 1;
    extended *= (uint64_t)g->extent[a] + 2;
    if (extended >= ((uint64_t)1 << 32)) return 2;
  }
  return 0;
}

static int wrap_cell(int i, int extent) { /* grid.hpp:97-101 */
  int r = i % extent;
  if (r < 0) r += extent;
  return r;
}

void or_wrap_position(const or_grid* g, const double* x, double* w) {
  for (int a = 0; a < g->dim; ++a) {
    w[a] = x[a];
    if (!g->periodic[a]) continue;
    const double len = g->extent[a] * g->spacing; /* axis_length, grid.hpp:72 */
    double r = fmod(x[a] - g->origin[a], len);
    if (r < 0.0) r += len;
    w[a] = g->origin[a] + r;
  }
}

void or_cell_index(const or_grid* g, const double* x, int support, int* i) {
  const double half = (support % 2 == 0) ? 0.0 : 0.5;
  for (int a = 0; a < g->dim; ++a) {
    const double t = (x[a] - g->origin[a]) / g->spacing - g->staggering[a];
    i[a] = (int)ceil(t - half);
  }
}

void or_point_of(const or_grid* g, const int* i, double* x) {
  for (int a = 0; a < g->dim; ++a) {
    const double s = (double)i[a] + g->staggering[a];
    const double p = g->spacing * s;
    x[a] = p + g->origin[a];
  }
}

uint32_t or_grid_index(const or_grid* g, const int* i) {
  size_t flat = 0, stride = 1;
  for (int a = 0; a < g->dim; ++a) {
    int c = i[a];
    const int e = g->extent[a];
    if (g->periodic[a]) c = wrap_cell(c, e);
    else if (c < 0 || c >= e) return UINT32_MAX;
    flat += (size_t)c * stride;
    stride *= (size_t)e;
  }
  return (uint32_t)flat;
}

uint32_t or_cell_key(const or_grid* g, const int* i) {
  uint64_t k = 0, stride = 1;
  for (int a = 0; a < g->dim; ++a) {
    const int e = g->extent[a];
    int c = i[a];
    if (g->periodic[a]) c = wrap_cell(c, e);
    k += (uint64_t)(c + 1) * stride;
    stride *= (uint64_t)e + 2;
  }
  return (uint32_t)k;
}

void or_cell_key_inverse(const or_grid* g, uint32_t k, int* i) {
  uint64_t rem = k;
  for (int a = 0; a < g->dim; ++a) {
    const uint64_t stride = (uint64_t)g->extent[a] + 2;
    i[a] = (int)(rem % stride) - 1;
    rem /= stride;
  }
}

double or_cosine_phi(double r) {
  if (!(fabs(r) < 2.0)) return 0.0;
  return 0.25 * (1.0 + cos(0.5 * OR_PI * r));
}

/* The other kernels the device takes (include/ibcuda.h ibc_kernel); the
 * reference's Kernel concept (kernel.hpp:16-21) admits any such phi.  The
 * same formulas are compiled into the reference build as Kernel structs
 * (oracle/ref_driver.cpp) to pin this restatement. */
int or_kernel_support(int kernel) {
  switch (kernel) {
    case 0: case 1: return 4;
    case 2: return 3;
    case 3: return 2;
    default: return 0;
  }
}

double or_kernel_phi(int kernel, double r) {
  const double a = fabs(r);
  switch (kernel) {
    case 1: /* Peskin 4-point (Peskin 2002, Eq. 6.27) */
      if (!(a < 2.0)) return 0.0;
      if (a <= 1.0) return (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * a * a)) * 0.125;
      return (5.0 - 2.0 * a - sqrt(fmax(0.0, -7.0 + 12.0 * a - 4.0 * a * a))) * 0.125;
    case 2: /* Roma, Peskin & Berger (1999) 3-point */
      if (!(a < 1.5)) return 0.0;
      if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * a * a)) / 3.0;
      return (5.0 - 3.0 * a - sqrt(1.0 - 3.0 * (1.0 - a) * (1.0 - a))) / 6.0;
    case 3: /* 2-point hat */
      return a < 1.0 ? 1.0 - a : 0.0;
    default:
      return or_cosine_phi(r);
  }
}

void or_shift(int dim, int64_t j, int support, int* sigma) {
  int64_t z = j - 1;
  for (int a = 0; a < dim; ++a) {
    sigma[a] = (int)(z % support) - support / 2;
    z /= support;
  }
}

double or_delta_weight(int dim, const double* dx, const int* sigma, double h) {
  double w = 1.0;
  for (int a = 0; a < dim; ++a) w *= or_cosine_phi(sigma[a] - dx[a] / h) / h;
  return w;
}

/* detail::CellOffsets::build (support_window.hpp:22-42). */
static void cell_offsets(const or_grid* g, const int* home, int support,
                         int64_t offset[3][OR_MAX_SUPPORT]) {
  int64_t stride = 1;
  for (int a = 0; a < g->dim; ++a) {
    const int extent = g->extent[a];
    for (int k = 0; k < support; ++k) {
      const int c = home[a] + k - support / 2;
      if (g->periodic[a]) offset[a][k] = stride * wrap_cell(c, extent);
      else if (c < 0 || c >= extent) offset[a][k] = or_invalid_offset;
      else offset[a][k] = stride * c;
    }
    stride *= extent;
  }
}

/* displacement_ratio / SupportWindow::build (support_window.hpp:48-70). */
static void support_window(const or_grid* g, const double* x, int support, double* t,
                           int64_t offset[3][OR_MAX_SUPPORT]) {
  double xw[3], hp[3];
  int home[3];
  or_wrap_position(g, x, xw);
  or_cell_index(g, xw, support, home);
  or_point_of(g, home, hp);
  for (int a = 0; a < g->dim; ++a) t[a] = (xw[a] - hp[a]) / g->spacing;
  if (offset) cell_offsets(g, home, support, offset);
}

static void advance_digits(int* digits, int dim, int support) { /* support_window.hpp:75-80 */
  for (int a = 0; a < dim; ++a) {
    if (++digits[a] < support) break;
    digits[a] = 0;
  }
}

static size_t grid_points(const or_grid* g) {
  size_t p = 1;
  for (int a = 0; a < g->dim; ++a) p *= (size_t)g->extent[a];
  return p;
}

static int64_t shift_count(int dim, int support) {
  int64_t n = 1;
  for (int a = 0; a < dim; ++a) n *= support;
  return n;
}

void or_key_value_sort(uint32_t* keys, uint32_t* payload, size_t n) {
  /* sort.hpp:17-71 with workers == 1: LSD radix, 8-bit digits, 4 passes. */
  if (n < 2) return;
  uint32_t* key_buf = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* pay_buf = (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t *src_k = keys, *dst_k = key_buf, *src_p = payload, *dst_p = pay_buf;
  size_t hist[256];
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = pass * 8;
    memset(hist, 0, sizeof(hist));
    for (size_t i = 0; i < n; ++i) ++hist[(src_k[i] >> shift) & 255u];
    size_t sum = 0;
    for (int d = 0; d < 256; ++d) {
      const size_t c = hist[d];
      hist[d] = sum;
      sum += c;
    }
    for (size_t i = 0; i < n; ++i) {
      const size_t pos = hist[(src_k[i] >> shift) & 255u]++;
      dst_k[pos] = src_k[i];
      dst_p[pos] = src_p[i];
    }
    uint32_t* t = src_k; src_k = dst_k; dst_k = t;
    t = src_p; src_p = dst_p; dst_p = t;
  }
  /* Four passes: the result is back in the caller's arrays. */
  free(key_buf);
  free(pay_buf);
}

size_t or_collect_unique_keys(const uint32_t* sorted, size_t n, uint32_t* out_keys) {
  size_t q = 0;
  for (size_t i = 0; i < n; ++i)
    if (i == 0 || sorted[i] != sorted[i - 1]) {
      if (out_keys) out_keys[q] = sorted[i];
      ++q;
    }
  return q;
}

size_t or_segmented_reduce(const uint32_t* sorted, const double* values, size_t n,
                           uint32_t* out_keys, double* out_sums) {
  size_t out = 0;
  for (size_t i = 0; i < n; ++i) {
    if (i == 0 || sorted[i] != sorted[i - 1]) {
      out_keys[out] = sorted[i];
      out_sums[out] = values[i];
      ++out;
    } else {
      out_sums[out - 1] += values[i];
    }
  }
  return out;
}

size_t or_prepare_keys_k(const or_grid* g, int kernel, const double* points, size_t n,
                         uint32_t* keys, uint32_t* perm, uint32_t* run_keys) {
  /* prepare_spread head (spread.hpp:93-103). */
  const int D = g->dim;
  const int support = or_kernel_support(kernel);
  for (size_t i = 0; i < n; ++i) {
    double xw[3];
    int c[3];
    or_wrap_position(g, points + i * D, xw);
    or_cell_index(g, xw, support, c);
    keys[i] = or_cell_key(g, c);
    perm[i] = (uint32_t)i;
  }
  or_key_value_sort(keys, perm, n);
  return or_collect_unique_keys(keys, n, run_keys);
}

size_t or_prepare_keys(const or_grid* g, const double* points, size_t n, uint32_t* keys,
                       uint32_t* perm, uint32_t* run_keys) {
  return or_prepare_keys_k(g, 0, points, n, keys, perm, run_keys);
}

int or_spread_serial_k(const or_grid* g, int kernel, const double* points, const double* values,
                       size_t n, double* out) {
  /* spread.hpp:129-159 */
  const int D = g->dim, s = or_kernel_support(kernel), half = s / 2;
  const int64_t nshift = shift_count(D, s);
  const double h = g->spacing;
  memset(out, 0, grid_points(g) * sizeof(double));
  for (size_t i = 0; i < n; ++i) {
    double t[3];
    int64_t off_tab[3][OR_MAX_SUPPORT];
    support_window(g, points + i * D, s, t, off_tab);
    const double value = values[i];
    int dig[3] = {0, 0, 0};
    for (int64_t j = 0; j < nshift; ++j) {
      double w = or_kernel_phi(kernel, (dig[0] - half) - t[0]) / h;
      int64_t off = off_tab[0][dig[0]];
      for (int a = 1; a < D; ++a) {
        w *= or_kernel_phi(kernel, (dig[a] - half) - t[a]) / h;
        off += off_tab[a][dig[a]];
      }
      if (off >= 0) out[off] += w * value;
      advance_digits(dig, D, s);
    }
  }
  return 0;
}

int or_spread_serial(const or_grid* g, const double* points, const double* values, size_t n,
                     double* out) {
  return or_spread_serial_k(g, 0, points, values, n, out);
}

int or_spread_fused_k(const or_grid* g, int kernel, const double* points, const double* values,
                      size_t n, double* out, uint32_t* keys_out, uint32_t* perm_out,
                      uint32_t* run_keys_out, size_t* q_out) {
  /* spread.hpp:165-216 with workers == 1 (segmented reduce = left fold). */
  const int D = g->dim, s = or_kernel_support(kernel);
  const int64_t nshift = shift_count(D, s);
  const double h = g->spacing;
  size_t alloc = n ? n : 1;
  uint32_t* keys = (uint32_t*)malloc(alloc * sizeof(uint32_t));
  uint32_t* perm = (uint32_t*)malloc(alloc * sizeof(uint32_t));
  uint32_t* run_keys = (uint32_t*)malloc(alloc * sizeof(uint32_t));
  double* disp = (double*)malloc(alloc * D * sizeof(double));
  double* staging = (double*)malloc(alloc * sizeof(double));
  double* run_values = (double*)malloc(alloc * sizeof(double));
  uint32_t* tmp_keys = (uint32_t*)malloc(alloc * sizeof(uint32_t));

  const size_t q = or_prepare_keys_k(g, kernel, points, n, keys, perm, run_keys);
  for (size_t i = 0; i < n; ++i) support_window(g, points + (size_t)perm[i] * D, s, disp + i * D, NULL);
  int64_t* run_offsets = (int64_t*)malloc((q ? q : 1) * D * s * sizeof(int64_t));
  for (size_t r = 0; r < q; ++r) {
    int home[3];
    int64_t tab[3][OR_MAX_SUPPORT];
    or_cell_key_inverse(g, run_keys[r], home);
    cell_offsets(g, home, s, tab);
    for (int a = 0; a < D; ++a)
      for (int k = 0; k < s; ++k) run_offsets[(size_t)(a * s + k) * q + r] = tab[a][k];
  }

  memset(out, 0, grid_points(g) * sizeof(double));
  for (int64_t j = 1; j <= nshift; ++j) {
    int sigma[3];
    or_shift(D, j, s, sigma);
    const int64_t* col[3];
    for (int a = 0; a < D; ++a) col[a] = run_offsets + (size_t)(a * s + sigma[a] + s / 2) * q;
    for (size_t i = 0; i < n; ++i) {
      const double* t = disp + i * D;
      double w = or_kernel_phi(kernel, sigma[0] - t[0]) / h;
      for (int a = 1; a < D; ++a) w *= or_kernel_phi(kernel, sigma[a] - t[a]) / h;
      staging[i] = w * values[perm[i]];
    }
    const size_t runs = or_segmented_reduce(keys, staging, n, tmp_keys, run_values);
    (void)runs;
    for (size_t r = 0; r < q; ++r) {
      int64_t off = col[0][r];
      for (int a = 1; a < D; ++a) off += col[a][r];
      if (off >= 0) out[off] += run_values[r];
    }
  }
  if (keys_out) memcpy(keys_out, keys, n * sizeof(uint32_t));
  if (perm_out) memcpy(perm_out, perm, n * sizeof(uint32_t));
  if (run_keys_out) memcpy(run_keys_out, run_keys, q * sizeof(uint32_t));
  if (q_out) *q_out = q;
  free(keys); free(perm); free(run_keys); free(disp); free(staging); free(run_values);
  free(tmp_keys); free(run_offsets);
  return 0;
}

int or_spread_fused(const or_grid* g, const double* points, const double* values, size_t n,
                    double* out, uint32_t* keys_out, uint32_t* perm_out, uint32_t* run_keys_out,
                    size_t* q_out) {
  return or_spread_fused_k(g, 0, points, values, n, out, keys_out, perm_out, run_keys_out, q_out);
}

int or_interpolate_k(const or_grid* g, int kernel, const double* field, const double* points,
                     size_t n, double* out) {
  /* interpolate.hpp:22-58 */
  const int D = g->dim, s = or_kernel_support(kernel), half = s / 2;
  const int64_t nshift = shift_count(D, s);
  const double hd = pow(g->spacing, (double)D);
  const double h = g->spacing;
  for (size_t i = 0; i < n; ++i) {
    double t[3];
    int64_t off_tab[3][OR_MAX_SUPPORT];
    support_window(g, points + i * D, s, t, off_tab);
    double acc = 0.0;
    int dig[3] = {0, 0, 0};
    for (int64_t j = 0; j < nshift; ++j) {
      double w = or_kernel_phi(kernel, (dig[0] - half) - t[0]) / h;
      int64_t off = off_tab[0][dig[0]];
      for (int a = 1; a < D; ++a) {
        w *= or_kernel_phi(kernel, (dig[a] - half) - t[a]) / h;
        off += off_tab[a][dig[a]];
      }
      if (off >= 0) acc += w * field[off];
      advance_digits(dig, D, s);
    }
    out[i] = acc * hd;
  }
  return 0;
}

int or_interpolate(const or_grid* g, const double* field, const double* points, size_t n,
                   double* out) {
  return or_interpolate_k(g, 0, field, points, n, out);
}

/* Home cells of many points (wrap_position + cell_index, grid.hpp:121-130,
 * 197-207), periodic axes wrapped into [0, n) when wrap != 0: the binning
 * the sampled-parity tests use to pick the points that reach a grid region. */
void or_home_cells(const or_grid* g, const double* points, size_t n, int support, int wrap,
                   int32_t* out) {
  const int D = g->dim;
  for (size_t i = 0; i < n; ++i) {
    double xw[3];
    int c[3];
    or_wrap_position(g, points + i * D, xw);
    or_cell_index(g, xw, support, c);
    for (int a = 0; a < D; ++a) {
      int v = c[a];
      if (wrap && g->periodic[a]) v = wrap_cell(v, g->extent[a]);
      out[i * D + a] = v;
    }
  }
}

/* ---- std::mt19937_64 (parameters of the C++ standard, [rand.predef]) ---- */
typedef struct {
  uint64_t mt[312];
  int idx;
} or_mt64;

static void mt64_seed(or_mt64* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

static uint64_t mt64_next(or_mt64* r) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (r->mt[i] & um) | (r->mt[i + 1] & lm);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (r->mt[i] & um) | (r->mt[i + 1] & lm);
      r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (r->mt[311] & um) | (r->mt[0] & lm);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

void or_scatter_points(uint64_t n, double edge, uint64_t seed, double* out) {
  or_mt64 r;
  mt64_seed(&r, seed);
  for (uint64_t i = 0; i < n * 3; ++i) out[i] = (double)(mt64_next(&r) >> 11) * 0x1.0p-53 * edge;
}
