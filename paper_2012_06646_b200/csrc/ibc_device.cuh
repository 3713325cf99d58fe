// ibc_device.cuh -- grid geometry, cell keys and delta weights on the device.
//
// Integer results (cells, keys) must be bit-identical to the reference
// (/root/reference/proj/include/ib/grid.hpp).  The floating-point steps that
// decide them are therefore written with explicit round-to-nearest intrinsics
// so nvcc cannot contract them into FMAs: the reference's x86-64 Release build
// has no FMA (plain -O3, no -march).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ibc {

constexpr int kSupport = 4;     // support of the fast paths (4-point kernels)
constexpr int kMaxSupport = 4;  // largest support the generic paths take
// Delta kernels (ibc_kernel in include/ibcuda.h).
constexpr int kKernelCosine4 = 0;  // CosineKernel (kernel.hpp:23-36)
constexpr int kKernelPeskin4 = 1;  // Peskin's standard 4-point kernel
constexpr int kKernelRoma3 = 2;    // Roma-Peskin-Berger 3-point kernel (odd support)
constexpr int kKernelLinear2 = 3;  // 2-point hat kernel
// The onesweep look-back packs per-digit counts into 30 bits.
constexpr uint32_t kMaxPoints = (1u << 30) - 1;

// Precomputed, kernel-argument-sized view of ib::StaggeredGrid<D>.
// Axes past `dim` are padded: extent 1, not periodic, zero strides.
struct DevGrid {
  int dim;
  int n[3];
  int periodic[3];
  double h;
  double alpha[3];
  double origin[3];
  double len[3];        // extent * spacing exactly as axis_length (grid.hpp:72)
  uint64_t kstride[3];  // cell_key strides prod_{b<a} (n_b + 2) (grid.hpp:158-170)
  uint32_t rowdiv;      // n[0] + 2: key / rowdiv = extended row id
  uint32_t nrows;       // number of extended rows (prod_{a>=1,a<dim} (n_a + 2))
  int64_t npts;         // prod(extent)
  double hd;            // pow(h, dim), computed on the host with std::pow
  double inv_h;
  // z-slab of a larger grid (multi-GPU, ibc_slab): the last axis is local
  // planes [zfirst, zfirst + n[dim-1]) of a global axis of zg_n planes.  Its
  // cells are computed in global coordinates -- bit-identical to the single
  // grid's -- then shifted by zfirst; locally the axis is not periodic.
  int zslab;            // 0 / 1
  int zfirst;           // global plane of local plane 0
  int zg_n;             // global extent of the last axis
  int zg_periodic;      // global periodicity of the last axis
  double zg_len;        // global axis length
  // Delta kernel (kernel.hpp:16-21): id, support s, first shift -floor(s/2)
  // (kernel.hpp:49-58) and cell_index's half = 0 / 0.5 for even / odd s
  // (grid.hpp:121-130).
  int kernel;
  int support;
  int slo;
  double half;
};

__device__ __forceinline__ int wrap_cell(int i, int e) {  // grid.hpp:97-101
  if (i >= 0 && i < e) return i;  // common case, no integer division
  if (i < 0 && i >= -e) return i + e;
  if (i >= e && i < 2 * e) return i - e;
  int r = i % e;
  if (r < 0) r += e;
  return r;
}

// wrap_position (grid.hpp:197-207) + cell_index for even support
// (grid.hpp:121-130) on one axis.  Returns the cell; *xw gets the wrapped x.
// The cell must equal ceil((xw - o) / h - alpha) exactly as the reference
// rounds it.  Fast path: q = (xw - o) * (1/h) is within ~2.3e-16 |q| of the
// correctly rounded quotient, so unless t = q - alpha lies within 1e-13 (|q|+1)
// of an integer, ceil(t) is the reference's cell; otherwise (a ~1e-13 fraction
// of points) the IEEE division is evaluated.
__device__ __forceinline__ int cell_of_slab(const DevGrid& g, double x, double* xw);

__device__ __forceinline__ int cell_of(const DevGrid& g, int a, double x, double* xw) {
  if (g.zslab && a == g.dim - 1) return cell_of_slab(g, x, xw);
  double w = x;
  if (g.periodic[a]) {
    const double d = __dsub_rn(x, g.origin[a]);
    // fmod(d, len) == d exactly when |d| < len: skip the iterative fmod.
    double r = fabs(d) < g.len[a] ? d : fmod(d, g.len[a]);
    if (r < 0.0) r = __dadd_rn(r, g.len[a]);
    w = __dadd_rn(g.origin[a], r);
  }
  *xw = w;
  const double d = __dsub_rn(w, g.origin[a]);
  const double q = __dmul_rn(d, g.inv_h);
  const double t = __dsub_rn(__dsub_rn(q, g.alpha[a]), g.half);
  const double c = ceil(t);
  const double margin = 1e-13 * (fabs(q) + 1.0);
  if (c - t > margin && t - (c - 1.0) > margin) return (int)c;
  return (int)ceil(__dsub_rn(__dsub_rn(__ddiv_rn(d, g.h), g.alpha[a]), g.half));
}

// Last axis of a slab grid: global wrap and cell (same arithmetic as
// cell_of), wrapped into [0, zg_n) on a periodic global axis, then shifted to
// the local plane.  *xw moves with the wrap (by whole periods) so the
// displacement (xw - h (c + alpha) - o) / h is unchanged.
__device__ __forceinline__ int cell_of_slab(const DevGrid& g, double x, double* xw) {
  const int a = g.dim - 1;
  double w = x;
  if (g.zg_periodic) {
    const double d = __dsub_rn(x, g.origin[a]);
    double r = fabs(d) < g.zg_len ? d : fmod(d, g.zg_len);
    if (r < 0.0) r = __dadd_rn(r, g.zg_len);
    w = __dadd_rn(g.origin[a], r);
  }
  const double d = __dsub_rn(w, g.origin[a]);
  const double q = __dmul_rn(d, g.inv_h);
  const double t = __dsub_rn(__dsub_rn(q, g.alpha[a]), g.half);
  double c = ceil(t);
  const double margin = 1e-13 * (fabs(q) + 1.0);
  if (!(c - t > margin && t - (c - 1.0) > margin))
    c = ceil(__dsub_rn(__dsub_rn(__ddiv_rn(d, g.h), g.alpha[a]), g.half));
  const int cu = (int)c;
  const int cw = g.zg_periodic ? wrap_cell(cu, g.zg_n) : cu;
  *xw = w - (double)(cu - cw) * g.h;
  return cw - g.zfirst;
}

// One axis of a DevGrid picked with a runtime index (selects, so the grid
// stays in the parameter bank instead of being copied to local memory).
struct Axis {
  double o, len, alpha, half;
  int n, periodic;
  int shift;  // slab axis: local = global - shift
};

__device__ __forceinline__ Axis axis_of(const DevGrid& g, int a) {
  Axis r;
  r.o = a == 0 ? g.origin[0] : (a == 1 ? g.origin[1] : g.origin[2]);
  r.len = a == 0 ? g.len[0] : (a == 1 ? g.len[1] : g.len[2]);
  r.alpha = a == 0 ? g.alpha[0] : (a == 1 ? g.alpha[1] : g.alpha[2]);
  r.n = a == 0 ? g.n[0] : (a == 1 ? g.n[1] : g.n[2]);
  r.periodic = a == 0 ? g.periodic[0] : (a == 1 ? g.periodic[1] : g.periodic[2]);
  r.half = g.half;
  r.shift = 0;
  if (g.zslab && a == g.dim - 1) {  // global wrap, then the local shift
    r.len = g.zg_len;
    r.n = g.zg_n;
    r.periodic = g.zg_periodic;
    r.shift = g.zfirst;
  }
  return r;
}

// cell_of + displacement for an Axis: returns the home cell (wrapped on a
// periodic axis) and u = -t in [0, 1) (t = displacement ratio).
__device__ __forceinline__ int cell_and_u(const Axis& A, double h, double inv_h, double x, double* u) {
  double w = x;
  if (A.periodic) {
    const double d = __dsub_rn(x, A.o);
    double r = fabs(d) < A.len ? d : fmod(d, A.len);
    if (r < 0.0) r = __dadd_rn(r, A.len);
    w = __dadd_rn(A.o, r);
  }
  const double d = __dsub_rn(w, A.o);
  const double q = __dmul_rn(d, inv_h);
  const double t = __dsub_rn(__dsub_rn(q, A.alpha), A.half);
  double c = ceil(t);
  const double margin = 1e-13 * (fabs(q) + 1.0);
  if (!(c - t > margin && t - (c - 1.0) > margin))
    c = ceil(__dsub_rn(__dsub_rn(__ddiv_rn(d, h), A.alpha), A.half));
  const int ci = (int)c;
  const double hp = __dadd_rn(__dmul_rn(h, __dadd_rn(c, A.alpha)), A.o);
  *u = -((w - hp) * inv_h);
  return (A.periodic ? wrap_cell(ci, A.n) : ci) - A.shift;
}

// displacement_ratio (support_window.hpp:48-55): (xw - h*(i+alpha) - o) / h.
// Only feeds the weights (not bit-exact anyway): multiply by 1/h.
__device__ __forceinline__ double displacement(const DevGrid& g, int a, double xw, int c) {
  if (g.zslab && a == g.dim - 1) c += g.zfirst;  // local plane -> global cell
  const double hp = __dadd_rn(__dmul_rn(g.h, __dadd_rn((double)c, g.alpha[a])), g.origin[a]);
  return (xw - hp) * g.inv_h;
}

// cell_key (grid.hpp:158-170) of already-computed (unwrapped) cells.
__device__ __forceinline__ uint32_t cell_key(const DevGrid& g, const int* c) {
  uint64_t k = 0;
  for (int a = 0; a < 3; ++a) {
    if (a >= g.dim) break;
    int ca = c[a];
    if (g.periodic[a]) ca = wrap_cell(ca, g.n[a]);
    k += (uint64_t)(int64_t)(ca + 1) * g.kstride[a];
  }
  return (uint32_t)k;
}

// sin(pi u / 2) and cos(pi u / 2) for u in [0, 1] (plus rounding slack):
// reflect to theta = pi y, y in [0, 1/4], then degree-15/16 Taylor
// polynomials (truncation < 5e-17 on [0, pi/4]).  ~22 FP64 ops instead of the
// ~130 instructions of the general sincospi.
__device__ __forceinline__ void sincos_half_pi(double u, double* sn, double* cs) {
  const double x = 0.5 * u;
  const bool flip = x > 0.25;
  const double y = flip ? 0.5 - x : x;
  const double th = y * 3.141592653589793116;
  const double z = th * th;
  double ps = -7.6471637318198164759e-13;          // -1/15!
  ps = fma(ps, z, 1.6059043836821614599e-10);      //  1/13!
  ps = fma(ps, z, -2.5052108385441718775e-8);      // -1/11!
  ps = fma(ps, z, 2.7557319223985890653e-6);       //  1/9!
  ps = fma(ps, z, -1.9841269841269841270e-4);      // -1/7!
  ps = fma(ps, z, 8.3333333333333333333e-3);       //  1/5!
  ps = fma(ps, z, -1.6666666666666666667e-1);      // -1/3!
  const double s_th = fma(th * z, ps, th);
  double pc = 4.7794773323873852974e-14;           //  1/16!
  pc = fma(pc, z, -1.1470745597729724714e-11);     // -1/14!
  pc = fma(pc, z, 2.0876756987868098979e-9);       //  1/12!
  pc = fma(pc, z, -2.7557319223985890653e-7);      // -1/10!
  pc = fma(pc, z, 2.4801587301587301587e-5);       //  1/8!
  pc = fma(pc, z, -1.3888888888888888889e-3);      // -1/6!
  pc = fma(pc, z, 4.1666666666666666667e-2);       //  1/4!
  pc = fma(pc, z, -0.5);
  const double c_th = fma(z, pc, 1.0);
  *sn = flip ? c_th : s_th;
  *cs = flip ? s_th : c_th;
}

// Per-axis weights phi(sigma - t) / h for sigma = -2..1 (index sigma + 2) of
// the 4-point cosine kernel (kernel.hpp:24-36, 64-69).  With u = -t and
// theta = pi u / 2 the four values are (1-cos), (1+sin), (1+cos), (1-sin)
// over 4: one sine/cosine pair per axis instead of four cos.  The |r| >= 2
// cut-offs fall out exactly (the terms vanish at the ends of the support).
__device__ __forceinline__ void cosine_weights(double t, double inv_h, double w[4]) {
  double s, c;
  sincos_half_pi(-t, &s, &c);
  w[0] = (0.25 * (1.0 - c)) * inv_h;
  w[1] = (0.25 * (1.0 + s)) * inv_h;
  w[2] = (0.25 * (1.0 + c)) * inv_h;
  w[3] = (0.25 * (1.0 - s)) * inv_h;
}

// Padded axis (a >= dim): only sigma = 0 (index -slo) contributes, factor 1.
__device__ __forceinline__ void unit_weights(double w[4], int slo = -2) {
#pragma unroll
  for (int k = 0; k < 4; ++k) w[k] = k == -slo ? 1.0 : 0.0;
}

// phi(r) of every supported kernel, written as the oracle writes it
// (oracle/ib_oracle.c or_kernel_phi):
//  COSINE4  (1 + cos(pi r / 2)) / 4 on |r| < 2 (kernel.hpp:24-27);
//  PESKIN4  (3 - 2|r| + sqrt(1 + 4|r| - 4r^2)) / 8 on |r| <= 1,
//           (5 - 2|r| - sqrt(-7 + 12|r| - 4r^2)) / 8 on 1 < |r| < 2;
//  ROMA3    (1 + sqrt(1 - 3r^2)) / 3 on |r| <= 1/2,
//           (5 - 3|r| - sqrt(1 - 3(1 - |r|)^2)) / 6 on 1/2 < |r| < 3/2;
//  LINEAR2  1 - |r| on |r| < 1.
__device__ __forceinline__ double kernel_phi(int k, double r) {
  const double a = fabs(r);
  if (k == kKernelPeskin4) {
    if (!(a < 2.0)) return 0.0;
    if (a <= 1.0) return (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * a * a)) * 0.125;
    return (5.0 - 2.0 * a - sqrt(fmax(0.0, -7.0 + 12.0 * a - 4.0 * a * a))) * 0.125;
  }
  if (k == kKernelRoma3) {
    if (!(a < 1.5)) return 0.0;
    if (a <= 0.5) return (1.0 + sqrt(1.0 - 3.0 * a * a)) / 3.0;
    const double b = 1.0 - a;
    return (5.0 - 3.0 * a - sqrt(1.0 - 3.0 * b * b)) / 6.0;
  }
  if (k == kKernelLinear2) return a < 1.0 ? 1.0 - a : 0.0;
  if (!(a < 2.0)) return 0.0;
  return 0.25 * (1.0 + cospi(0.5 * r));
}

// Weights phi(sigma - t) / h for sigma = slo .. slo + s - 1 (index sigma -
// slo; entries past the support are 0) of any kernel: the generic paths.
__device__ __forceinline__ void kernel_weights(const DevGrid& g, double t, double w[4]) {
  if (g.kernel == kKernelCosine4) {
    cosine_weights(t, g.inv_h, w);
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    w[k] = k < g.support ? kernel_phi(g.kernel, (double)(g.slo + k) - t) * g.inv_h : 0.0;
}

// The 4-point kernels' weight pair.  Both satisfy the even/odd partition of
// unity (phi(-2+u) + phi(u) = phi(-1+u) + phi(1+u) = 1/2), so with u = -t in
// [0, 1) their four weights are (1 - c)/4, (1 + s)/4, (1 + c)/4, (1 - s)/4 for
// one pair (s, c) per axis -- the fast paths' records carry that pair:
//   COSINE4  s = sin(pi u / 2), c = cos(pi u / 2);
//   PESKIN4  with R = sqrt(1 + 4u - 4u^2): c = (1 - 2u + R) / 2,
//            s = (2u - 1 + R) / 2.
__device__ __forceinline__ void kernel_pair(int k, double u, double* sn, double* cs) {
  if (k == kKernelPeskin4) {
    const double R = sqrt(fma(4.0 * u, 1.0 - u, 1.0));
    *cs = 0.5 * (1.0 - 2.0 * u + R);
    *sn = 0.5 * (2.0 * u - 1.0 + R);
    return;
  }
  sincos_half_pi(u, sn, cs);
}

namespace sw {
// Tiling of the TMA interpolation gather (ibc_sweep.cuh, chosen on the host).
struct InterpTiling {
  int ty, zc, nty, nzc;
  int frmax;             // field rows per slot (ty + 3, + ghost rows on closed y)
  int slots;             // ring depth (>= 5)
  uint32_t pitch;        // bytes per field row in shared memory (multiple of 1024)
  uint32_t slot_bytes;   // frmax * pitch
  int rec_cap;           // point records staged per step (64 B each)
  int hmax;              // max home planes per CTA (row-range table entries)
  uint32_t slot_stride;  // slot_bytes + rec_cap * 64, rounded up to 1024
  int box_ok;            // one TMA per plane allowed (nx % 128 == 0)
};
}  // namespace sw

// Programmatic dependent launch: the pipeline's kernels are launched with
// programmatic stream serialization (their launch and block scheduling
// overlap the predecessor's tail) and wait here, before touching memory,
// until the predecessor grid has completed and flushed.  A no-op for a
// normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): one 32-byte sector
// per instruction instead of two half-sector 128-bit ones.
__device__ __forceinline__ void st_v4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ double4 ld_v4_nc(const double* p) {
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
      : "l"(p));
  return v;
}

}  // namespace ibc
