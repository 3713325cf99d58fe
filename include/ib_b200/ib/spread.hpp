// ib_b200/ib/spread.hpp -- overlay of the reference's ib/spread.hpp: every
// spreading algorithm runs on the B200 through ibc_spread (one write-once
// device operator; SpreadAlgorithm keeps the reference's argument checks).
#pragma once

#include <array>
#include <cassert>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "b200.hpp"
#include "detail/support_window.hpp"
#include "grid.hpp"
#include "kernel.hpp"
#include "parallel.hpp"
#include "reduce.hpp"
#include "sort.hpp"
#include "stats.hpp"

namespace ib {

enum class SpreadAlgorithm { serial, fused, buffered, otf };  // spread.hpp:21

// spread.hpp:23-56.  The reference's scratch vectors (staging, run_values,
// displacements, run_offsets, buffers) live on the device inside the
// workspace handle; the observable results -- keys (sorted), perm, run_keys,
// run_count -- read like the reference's members and are copied back from
// the device on first read after a spread (b200::observable_vector).
template <std::size_t D>
struct SpreadWorkspace {
  std::size_t point_count;
  std::size_t grid_points;
  int sweep_width;

  b200::observable_vector<SortKey> keys;
  b200::observable_vector<std::uint32_t> perm;
  b200::observable_vector<SortKey> run_keys;
  b200::observable_count run_count;

  SpreadWorkspace(std::size_t n, const StaggeredGrid<D>& grid, int b = 0)
      : point_count(n), grid_points(grid.point_count()), sweep_width(b), keys(n), perm(n),
        run_keys(n) {
    if (b < 0) throw std::invalid_argument("sweep width must be >= 1 (or 0 for none)");
    ibc_workspace* w = nullptr;
    b200::check(ibc_workspace_create(b200::context(), n, &grid.c_grid(), b, &w));
    handle_.reset(w);
  }

  // Overlay: the device workspace, and the hook a spread calls.
  ibc_workspace* handle() const { return handle_.get(); }
  void spread_done() {
    ibc_workspace* h = handle();
    const std::size_t n = point_count;
    keys.invalidate([h, n](std::vector<SortKey>& v) { b200::check(ibc_workspace_get_keys(h, v.data(), n)); });
    perm.invalidate([h, n](std::vector<std::uint32_t>& v) { b200::check(ibc_workspace_get_perm(h, v.data(), n)); });
    run_keys.invalidate([h](std::vector<SortKey>& v) {
      std::size_t q = 0;
      b200::check(ibc_workspace_get_run_keys(h, v.data(), v.size(), &q));
    });
    run_count.invalidate([h] {
      std::size_t q = 0;
      b200::check(ibc_workspace_run_count(h, &q));
      return q;
    });
  }

 private:
  struct Release {
    void operator()(ibc_workspace* w) const { ibc_workspace_destroy(w); }
  };
  std::unique_ptr<ibc_workspace, Release> handle_;
};

namespace detail {

// spread.hpp:58-77 (the C ABI repeats these checks; kept for callers).
template <std::size_t D>
void check_spread_args(std::size_t n_points, std::size_t n_values, int support) {
  if (n_values != n_points) throw std::invalid_argument("one value per point required");
  if (support < 1 || support > max_support)
    throw std::invalid_argument("unsupported kernel support size");
}

template <std::size_t D>
void check_workspace(const SpreadWorkspace<D>& ws, std::size_t n_points,
                     const StaggeredGrid<D>& grid, bool needs_buffers) {
  if (ws.point_count != n_points)
    throw std::invalid_argument("workspace sized for a different point count");
  if (ws.grid_points != grid.point_count())
    throw std::invalid_argument("workspace sized for a different grid");
  if (needs_buffers && ws.sweep_width < 1)
    throw std::invalid_argument("workspace has no sweep buffers");
}

}  // namespace detail

namespace b200 {
template <std::size_t D, Kernel K>
GridField<D> spread(ibc_spread_algorithm algo, const PointSet<D>& points,
                    std::span<const double> values, const StaggeredGrid<D>& grid, const K& kernel,
                    int sweep_width, SpreadWorkspace<D>* ws, int workers) {
  GridField<D> out(grid);
  check(ibc_spread(context(), &grid.c_grid(), kernel_id(kernel), algo, flat(points), values.data(),
                   points.size(), values.size(), sweep_width, ws ? ws->handle() : nullptr, workers,
                   out.values.data()));
  if (ws) ws->spread_done();
  return out;
}
}  // namespace b200

// Algorithm 2 (spread.hpp:125-159).
template <std::size_t D, Kernel K>
GridField<D> spread_serial(const PointSet<D>& points, std::span<const double> values,
                           const StaggeredGrid<D>& grid, const K& kernel) {
  return b200::spread<D>(IBC_SPREAD_SERIAL, points, values, grid, kernel, 0, nullptr, 1);
}

// Algorithm 4 (spread.hpp:161-216).
template <std::size_t D, Kernel K>
GridField<D> spread_fused(const PointSet<D>& points, std::span<const double> values,
                          const StaggeredGrid<D>& grid, const K& kernel, SpreadWorkspace<D>& ws,
                          int workers) {
  return b200::spread<D>(IBC_SPREAD_FUSED, points, values, grid, kernel, 0, &ws, workers);
}

// Algorithm 5 (spread.hpp:218-303).
template <std::size_t D, Kernel K>
GridField<D> spread_buffered(const PointSet<D>& points, std::span<const double> values,
                             const StaggeredGrid<D>& grid, const K& kernel, SpreadWorkspace<D>& ws,
                             int workers) {
  return b200::spread<D>(IBC_SPREAD_BUFFERED, points, values, grid, kernel, 0, &ws, workers);
}

// Algorithm 6 (spread.hpp:305-317).
template <std::size_t D, Kernel K>
GridField<D> spread_buffered_otf(const PointSet<D>& points, std::span<const double> values,
                                 const StaggeredGrid<D>& grid, const K& kernel, int sweep_width,
                                 int workers) {
  return b200::spread<D>(IBC_SPREAD_OTF, points, values, grid, kernel, sweep_width, nullptr,
                         workers);
}

// One spread per MAC component (spread.hpp:319-350).  The reference runs the
// components one after the other, each checking its arguments first; here
// the checks run first, in the same order and with the same messages, and
// the components that would have run before the first failing one run
// concurrently (b200::for_components), then its exception is thrown.  With
// a workspace (fused / buffered) the last component spreads through it, so
// it ends up holding that component's sort as in the reference, and the
// others run the same device operator on context scratch.
template <std::size_t D, Kernel K>
std::array<GridField<D>, D> spread_vector(const PointSet<D>& points,
                                          const std::array<LagrangianValues, D>& values,
                                          std::span<const StaggeredGrid<D>> grids, const K& kernel,
                                          SpreadAlgorithm algorithm, int sweep_width,
                                          SpreadWorkspace<D>* workspace, int workers) {
  if (grids.size() != D) throw std::invalid_argument("expected one grid per vector component");
  // The first component whose call would throw, and its exception.
  std::size_t ok = D;
  std::exception_ptr fail;
  for (std::size_t c = 0; c < D && !fail; ++c) {
    try {
      switch (algorithm) {
        case SpreadAlgorithm::serial:
          detail::check_spread_args<D>(points.size(), values[c].size(), kernel.support());
          break;
        case SpreadAlgorithm::fused:
        case SpreadAlgorithm::buffered: {
          const bool buffered = algorithm == SpreadAlgorithm::buffered;
          if (!workspace)
            throw std::invalid_argument(buffered ? "buffered spreading needs a workspace"
                                                 : "fused spreading needs a workspace");
          detail::check_spread_args<D>(points.size(), values[c].size(), kernel.support());
          detail::check_workspace(*workspace, points.size(), grids[c], buffered);
          break;
        }
        case SpreadAlgorithm::otf:
          if (sweep_width < 1) throw std::invalid_argument("sweep width must be >= 1");
          detail::check_spread_args<D>(points.size(), values[c].size(), kernel.support());
          break;
        default:
          throw std::invalid_argument("unknown spreading algorithm");
      }
    } catch (...) {
      ok = c;
      fail = std::current_exception();
    }
  }
  std::array<std::optional<GridField<D>>, D> res;
  auto component = [&](std::size_t c) {
    const std::span<const double> v(values[c]);
    const bool last = c + 1 == D;
    if (algorithm == SpreadAlgorithm::serial || (!last && algorithm != SpreadAlgorithm::otf))
      res[c].emplace(spread_serial(points, v, grids[c], kernel));
    else if (algorithm == SpreadAlgorithm::fused)
      res[c].emplace(spread_fused(points, v, grids[c], kernel, *workspace, workers));
    else if (algorithm == SpreadAlgorithm::buffered)
      res[c].emplace(spread_buffered(points, v, grids[c], kernel, *workspace, workers));
    else
      res[c].emplace(spread_buffered_otf(points, v, grids[c], kernel, sweep_width, workers));
  };
  b200::for_components<D>(ok, component);
  if (fail) std::rethrow_exception(fail);
  if constexpr (D == 1) return {std::move(*res[0])};
  else if constexpr (D == 2) return {std::move(*res[0]), std::move(*res[1])};
  else return {std::move(*res[0]), std::move(*res[1]), std::move(*res[2])};
}

}  // namespace ib
