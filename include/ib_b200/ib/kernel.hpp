// ib_b200/ib/kernel.hpp -- overlay of the reference's ib/kernel.hpp.
//
// The Kernel concept and CosineKernel are the reference's (kernel.hpp:16-36);
// the device takes kernels by id (include/ibcuda.h ibc_kernel), so the other
// kernels it implements are declared here too.  b200::kernel_id<K>() maps a
// kernel TYPE to its device id at compile time: an operator called with any
// other Kernel type does not compile (the device evaluates phi itself and
// cannot run a caller's own phi; a silent substitution would return another
// kernel's results).
#pragma once

#include <cassert>
#include <cmath>
#include <concepts>
#include <cstdint>
#include <numbers>
#include <type_traits>

#include "grid.hpp"

namespace ib {

template <class K>
concept Kernel = requires(const K& k, double r) {
  { k.phi(r) } -> std::convertible_to<double>;
  { k.support() } -> std::convertible_to<int>;
  { k.radius() } -> std::convertible_to<double>;
};

// kernel.hpp:23-27.
inline double cosine_phi(double r) {
  if (!(std::abs(r) < 2.0)) return 0.0;
  return 0.25 * (1.0 + std::cos(0.5 * std::numbers::pi * r));
}

// kernel.hpp:29-36: the reference's kernel (IBC_KERNEL_COSINE4).
class CosineKernel {
 public:
  double phi(double r) const { return cosine_phi(r); }
  int support() const { return 4; }
  double radius() const { return 2.0; }
};

// Peskin's standard 4-point kernel (Peskin 2002, Eq. 6.27; IBC_KERNEL_PESKIN4).
class Peskin4Kernel {
 public:
  double phi(double r) const {
    const double a = std::abs(r);
    if (!(a < 2.0)) return 0.0;
    if (a <= 1.0) return (3.0 - 2.0 * a + std::sqrt(1.0 + 4.0 * a - 4.0 * a * a)) * 0.125;
    return (5.0 - 2.0 * a - std::sqrt(std::fmax(0.0, -7.0 + 12.0 * a - 4.0 * a * a))) * 0.125;
  }
  int support() const { return 4; }
  double radius() const { return 2.0; }
};

// 3-point kernel of Roma, Peskin & Berger (1999), odd support (IBC_KERNEL_ROMA3).
class Roma3Kernel {
 public:
  double phi(double r) const {
    const double a = std::abs(r);
    if (!(a < 1.5)) return 0.0;
    if (a <= 0.5) return (1.0 + std::sqrt(1.0 - 3.0 * a * a)) / 3.0;
    return (5.0 - 3.0 * a - std::sqrt(1.0 - 3.0 * (1.0 - a) * (1.0 - a))) / 6.0;
  }
  int support() const { return 3; }
  double radius() const { return 1.5; }
};

// 2-point hat (IBC_KERNEL_LINEAR2).
class Linear2Kernel {
 public:
  double phi(double r) const {
    const double a = std::abs(r);
    return a < 1.0 ? 1.0 - a : 0.0;
  }
  int support() const { return 2; }
  double radius() const { return 1.0; }
};

// Number of shifts s^D (kernel.hpp:38-45).
template <std::size_t D>
constexpr std::int64_t shift_count(int support) {
  std::int64_t n = 1;
  for (std::size_t a = 0; a < D; ++a) n *= support;
  return n;
}

// The j-th shift (1-based), colex, components in [-floor(s/2), floor((s-1)/2)]
// (kernel.hpp:47-58).
template <std::size_t D>
CellIndex<D> shift(std::int64_t j, int support) {
  assert(j >= 1 && j <= shift_count<D>(support));
  std::int64_t rest = j - 1;
  CellIndex<D> sigma;
  for (std::size_t a = 0; a < D; ++a) {
    sigma[a] = static_cast<int>(rest % support) - support / 2;
    rest /= support;
  }
  return sigma;
}

// prod_a phi(sigma_a - dx_a / h) / h (kernel.hpp:60-69).
template <std::size_t D, Kernel K>
double delta_weight(const Vec<D>& dx, const CellIndex<D>& sigma, double h, const K& kernel) {
  double w = 1.0;
  for (std::size_t a = 0; a < D; ++a) w *= kernel.phi(sigma[a] - dx[a] / h) / h;
  return w;
}

namespace b200 {
template <class>
inline constexpr bool unsupported_kernel = false;

// Device id of a kernel type (compile time).
template <class K>
constexpr ibc_kernel kernel_id() {
  using T = std::remove_cvref_t<K>;
  if constexpr (std::same_as<T, CosineKernel>) return IBC_KERNEL_COSINE4;
  else if constexpr (std::same_as<T, Peskin4Kernel>) return IBC_KERNEL_PESKIN4;
  else if constexpr (std::same_as<T, Roma3Kernel>) return IBC_KERNEL_ROMA3;
  else if constexpr (std::same_as<T, Linear2Kernel>) return IBC_KERNEL_LINEAR2;
  else {
    static_assert(unsupported_kernel<T>,
                  "libibcuda evaluates the delta kernel on the device: use ib::CosineKernel, "
                  "ib::Peskin4Kernel, ib::Roma3Kernel or ib::Linear2Kernel");
    return IBC_KERNEL_COSINE4;
  }
}

// spread.hpp:64-65 / interpolate.hpp:27-28: support in [1, max_support].
template <Kernel K>
ibc_kernel kernel_id(const K& kernel) {
  if (kernel.support() < 1 || kernel.support() > 8)
    throw std::invalid_argument("unsupported kernel support size");
  return kernel_id<K>();
}
}  // namespace b200

}  // namespace ib
