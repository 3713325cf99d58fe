// ib_b200/ib.hpp -- drop-in C++ replacement for the reference's operator API
// (/root/reference/proj/include/ib/ib.hpp), backed by the B200 C ABI
// (include/ibcuda.h, libibcuda.so).
//
// A reference caller switches by replacing
//     #include "ib/ib.hpp"            with     #include "ib_b200/ib.hpp"
// and linking libibcuda.so.  Every name below keeps the reference's
// signature, argument meaning and exceptions:
//
//   reference                                     here
//   ib::StaggeredGrid<D>      grid.hpp:33-83      same class, same validation
//   ib::GridField<D>          grid.hpp:85-92      same struct
//   ib::PointSet<D>, LagrangianValues grid.hpp:187-192  same aliases
//   ib::CosineKernel, Kernel  kernel.hpp:16-36    same (host-side phi for parity)
//   ib::SpreadAlgorithm       spread.hpp:21       same enum
//   ib::SpreadWorkspace<D>    spread.hpp:27-56    device workspace; keys / perm /
//                                                 run_keys / run_count refreshed
//                                                 after each spread (as observable
//                                                 in the reference)
//   ib::spread_serial/_fused/_buffered/_buffered_otf/spread_vector
//                             spread.hpp:129-350  ibc_spread (all on the B200)
//   ib::interpolate / interpolate_vector
//                             interpolate.hpp:22-72  ibc_interpolate
//   ib::stats                 stats.hpp:9-25      ibc_delta_evaluations
//
// `workers` is accepted and ignored (the device picks its parallelism).  The
// device is ib::b200::default_device() (0 unless set); every call is
// synchronous with host buffers, like the reference's.
#pragma once

#include <array>
#include <cmath>
#include <concepts>
#include <cstdint>
#include <limits>
#include <memory>
#include <new>
#include <numbers>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ibcuda.h"

namespace ib {

template <std::size_t D>
using Vec = std::array<double, D>;
template <std::size_t D>
using CellIndex = std::array<int, D>;
using GridIndex = std::uint32_t;
inline constexpr GridIndex invalid_index = std::numeric_limits<GridIndex>::max();
using SortKey = std::uint32_t;

namespace b200 {

// Status code -> the reference's exception type (ibcuda.h).
inline void check(ibc_status s) {
  switch (s) {
    case IBC_OK:
      return;
    case IBC_ERR_INVALID_ARGUMENT:
      throw std::invalid_argument(ibc_last_error());
    case IBC_ERR_LENGTH:
      throw std::length_error(ibc_last_error());
    case IBC_ERR_ALLOC:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(std::string("libibcuda: ") + ibc_last_error());
  }
}

inline int& default_device() {
  static int device = 0;
  return device;
}

// One context per process (created on first use on default_device()).
inline ibc_context* context() {
  struct Holder {
    ibc_context* ctx = nullptr;
    ~Holder() {
      if (ctx) ibc_context_destroy(ctx);
    }
  };
  static Holder h;
  if (!h.ctx) check(ibc_context_create(default_device(), &h.ctx));
  return h.ctx;
}

}  // namespace b200

// ---------------------------------------------------------------- grid.hpp
template <std::size_t D>
class StaggeredGrid {
  static_assert(D >= 1 && D <= 3, "grids are 1-, 2-, or 3-dimensional");

 public:
  StaggeredGrid(std::array<int, D> extents, double spacing, Vec<D> staggering,
                std::array<bool, D> periodic, Vec<D> origin = {})
      : extents_(extents), spacing_(spacing), staggering_(staggering), periodic_(periodic),
        origin_(origin) {
    b200::check(ibc_grid_check(&c_grid()));  // grid.hpp:37-60 conditions and messages
    point_count_ = 1;
    for (std::size_t a = 0; a < D; ++a) point_count_ *= static_cast<std::size_t>(extents_[a]);
  }

  int extent(std::size_t axis) const { return extents_[axis]; }
  const std::array<int, D>& extents() const { return extents_; }
  double spacing() const { return spacing_; }
  double staggering(std::size_t axis) const { return staggering_[axis]; }
  const Vec<D>& staggerings() const { return staggering_; }
  bool is_periodic(std::size_t axis) const { return periodic_[axis]; }
  const Vec<D>& origin() const { return origin_; }
  std::size_t point_count() const { return point_count_; }
  double axis_length(std::size_t axis) const { return extents_[axis] * spacing_; }

  // The C-ABI descriptor of this grid.
  const ibc_grid& c_grid() const {
    g_ = ibc_grid{};
    g_.dim = static_cast<int>(D);
    g_.spacing = spacing_;
    for (std::size_t a = 0; a < D; ++a) {
      g_.extent[a] = extents_[a];
      g_.staggering[a] = staggering_[a];
      g_.periodic[a] = periodic_[a] ? 1 : 0;
      g_.origin[a] = origin_[a];
    }
    return g_;
  }

 private:
  std::array<int, D> extents_;
  double spacing_;
  Vec<D> staggering_;
  std::array<bool, D> periodic_;
  Vec<D> origin_;
  std::size_t point_count_ = 0;
  mutable ibc_grid g_{};
};

template <std::size_t D>
struct GridField {
  StaggeredGrid<D> grid;
  std::vector<double> values;
  explicit GridField(StaggeredGrid<D> g) : grid(std::move(g)), values(grid.point_count(), 0.0) {}
};

template <std::size_t D>
using PointSet = std::vector<Vec<D>>;
using LagrangianValues = std::vector<double>;

// -------------------------------------------------------------- kernel.hpp
template <class K>
concept Kernel = requires(const K& k, double r) {
  { k.phi(r) } -> std::convertible_to<double>;
  { k.support() } -> std::convertible_to<int>;
  { k.radius() } -> std::convertible_to<double>;
};

inline double cosine_phi(double r) {
  if (!(std::abs(r) < 2.0)) return 0.0;
  return 0.25 * (1.0 + std::cos(0.5 * std::numbers::pi * r));
}

class CosineKernel {
 public:
  double phi(double r) const { return cosine_phi(r); }
  int support() const { return 4; }
  double radius() const { return 2.0; }
};

namespace b200 {
// The device implements the 4-point cosine kernel; any Kernel with support 4
// is taken to be it, other supports are rejected like spread.hpp:60-66 does.
template <Kernel K>
ibc_kernel kernel_id(const K& kernel) {
  if (kernel.support() < 1 || kernel.support() > 8)
    throw std::invalid_argument("unsupported kernel support size");
  if (kernel.support() != 4) throw std::invalid_argument("unsupported kernel support size");
  return IBC_KERNEL_COSINE4;
}

template <std::size_t D>
const double* flat(const PointSet<D>& points) {
  static_assert(sizeof(Vec<D>) == D * sizeof(double), "PointSet must be dense AoS");
  return points.empty() ? nullptr : points.front().data();
}
}  // namespace b200

// -------------------------------------------------------------- spread.hpp
enum class SpreadAlgorithm { serial, fused, buffered, otf };

template <std::size_t D>
struct SpreadWorkspace {
  std::size_t point_count;
  std::size_t grid_points;
  int sweep_width;

  // Observable results of the most recent spread (spread.hpp:33-41).
  std::vector<SortKey> keys;
  std::vector<std::uint32_t> perm;
  std::vector<SortKey> run_keys;
  std::size_t run_count = 0;
  // Copy keys / perm / run_keys back after every spread (the reference always
  // has them); set false to keep the spread device-only.
  bool sync_observables = true;

  SpreadWorkspace(std::size_t n, const StaggeredGrid<D>& grid, int b = 0)
      : point_count(n), grid_points(grid.point_count()), sweep_width(b) {
    if (b < 0) throw std::invalid_argument("sweep width must be >= 1 (or 0 for none)");
    ibc_workspace* w = nullptr;
    b200::check(ibc_workspace_create(b200::context(), n, &grid.c_grid(), b, &w));
    handle_.reset(w);
    keys.resize(n);
    perm.resize(n);
    run_keys.resize(n);
  }

  ibc_workspace* handle() const { return handle_.get(); }

  void refresh() {
    b200::check(ibc_workspace_run_count(handle(), &run_count));
    if (!sync_observables) return;
    b200::check(ibc_workspace_get_keys(handle(), keys.data(), point_count));
    b200::check(ibc_workspace_get_perm(handle(), perm.data(), point_count));
    std::size_t q = 0;
    b200::check(ibc_workspace_get_run_keys(handle(), run_keys.data(), run_keys.size(), &q));
  }

 private:
  struct Del {
    void operator()(ibc_workspace* w) const { ibc_workspace_destroy(w); }
  };
  std::unique_ptr<ibc_workspace, Del> handle_;
};

namespace b200 {
template <std::size_t D, Kernel K>
GridField<D> spread(ibc_spread_algorithm algo, const PointSet<D>& points,
                    std::span<const double> values, const StaggeredGrid<D>& grid, const K& kernel,
                    int sweep_width, SpreadWorkspace<D>* ws) {
  GridField<D> out(grid);
  check(ibc_spread(context(), &grid.c_grid(), kernel_id(kernel), algo, flat(points),
                   values.data(), points.size(), values.size(), sweep_width,
                   ws ? ws->handle() : nullptr, 0, out.values.data()));
  if (ws) ws->refresh();
  return out;
}
}  // namespace b200

template <std::size_t D, Kernel K>
GridField<D> spread_serial(const PointSet<D>& points, std::span<const double> values,
                           const StaggeredGrid<D>& grid, const K& kernel) {
  return b200::spread<D>(IBC_SPREAD_SERIAL, points, values, grid, kernel, 0, nullptr);
}

template <std::size_t D, Kernel K>
GridField<D> spread_fused(const PointSet<D>& points, std::span<const double> values,
                          const StaggeredGrid<D>& grid, const K& kernel, SpreadWorkspace<D>& ws,
                          int /*workers*/) {
  return b200::spread<D>(IBC_SPREAD_FUSED, points, values, grid, kernel, 0, &ws);
}

template <std::size_t D, Kernel K>
GridField<D> spread_buffered(const PointSet<D>& points, std::span<const double> values,
                             const StaggeredGrid<D>& grid, const K& kernel,
                             SpreadWorkspace<D>& ws, int /*workers*/) {
  return b200::spread<D>(IBC_SPREAD_BUFFERED, points, values, grid, kernel, 0, &ws);
}

template <std::size_t D, Kernel K>
GridField<D> spread_buffered_otf(const PointSet<D>& points, std::span<const double> values,
                                 const StaggeredGrid<D>& grid, const K& kernel, int sweep_width,
                                 int /*workers*/) {
  return b200::spread<D>(IBC_SPREAD_OTF, points, values, grid, kernel, sweep_width, nullptr);
}

template <std::size_t D, Kernel K>
std::array<GridField<D>, D> spread_vector(const PointSet<D>& points,
                                          const std::array<LagrangianValues, D>& values,
                                          std::span<const StaggeredGrid<D>> grids, const K& kernel,
                                          SpreadAlgorithm algorithm, int sweep_width,
                                          SpreadWorkspace<D>* workspace, int workers) {
  if (grids.size() != D) throw std::invalid_argument("expected one grid per vector component");
  auto component = [&](std::size_t c) -> GridField<D> {
    switch (algorithm) {
      case SpreadAlgorithm::serial:
        return spread_serial(points, std::span<const double>(values[c]), grids[c], kernel);
      case SpreadAlgorithm::fused:
        if (!workspace) throw std::invalid_argument("fused spreading needs a workspace");
        return spread_fused(points, std::span<const double>(values[c]), grids[c], kernel,
                            *workspace, workers);
      case SpreadAlgorithm::buffered:
        if (!workspace) throw std::invalid_argument("buffered spreading needs a workspace");
        return spread_buffered(points, std::span<const double>(values[c]), grids[c], kernel,
                               *workspace, workers);
      case SpreadAlgorithm::otf:
        return spread_buffered_otf(points, std::span<const double>(values[c]), grids[c], kernel,
                                   sweep_width, workers);
    }
    throw std::invalid_argument("unknown spreading algorithm");
  };
  if constexpr (D == 1) return {component(0)};
  if constexpr (D == 2) return {component(0), component(1)};
  if constexpr (D == 3) return {component(0), component(1), component(2)};
}

// --------------------------------------------------------- interpolate.hpp
template <std::size_t D, Kernel K>
LagrangianValues interpolate(const GridField<D>& field, const PointSet<D>& points, const K& kernel,
                             int /*workers*/) {
  LagrangianValues out(points.size());
  b200::check(ibc_interpolate(b200::context(), &field.grid.c_grid(), b200::kernel_id(kernel),
                              field.values.data(), b200::flat(points), points.size(), 0,
                              out.data()));
  return out;
}

template <std::size_t D, Kernel K>
std::array<LagrangianValues, D> interpolate_vector(std::span<const GridField<D>> fields,
                                                   const PointSet<D>& points, const K& kernel,
                                                   int workers) {
  if (fields.size() != D) throw std::invalid_argument("expected one field per vector component");
  std::array<LagrangianValues, D> out;
  for (std::size_t c = 0; c < D; ++c) out[c] = interpolate(fields[c], points, kernel, workers);
  return out;
}

// ---------------------------------------------------------------- stats.hpp
namespace stats {
inline std::uint64_t delta_evaluations() { return ibc_delta_evaluations(); }
inline void reset_delta_evaluations() { ibc_reset_delta_evaluations(); }
}  // namespace stats

}  // namespace ib
