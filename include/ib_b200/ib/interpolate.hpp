// ib_b200/ib/interpolate.hpp -- overlay of the reference's ib/interpolate.hpp:
// Algorithm 3 on the B200 through ibc_interpolate.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>

#include "b200.hpp"
#include "detail/support_window.hpp"
#include "grid.hpp"
#include "kernel.hpp"
#include "parallel.hpp"
#include "stats.hpp"

namespace ib {

// E_i = h^d sum_k delta_h(x_k - X_i) e_k, off-grid support skipped
// (interpolate.hpp:16-58).
template <std::size_t D, Kernel K>
LagrangianValues interpolate(const GridField<D>& field, const PointSet<D>& points, const K& kernel,
                             int workers) {
  LagrangianValues out(points.size());
  b200::check(ibc_interpolate(b200::context(), &field.grid.c_grid(), b200::kernel_id(kernel),
                              field.values.data(), b200::flat(points), points.size(), workers,
                              out.data()));
  return out;
}

// interpolate.hpp:60-72; the components run concurrently.
template <std::size_t D, Kernel K>
std::array<LagrangianValues, D> interpolate_vector(std::span<const GridField<D>> fields,
                                                   const PointSet<D>& points, const K& kernel,
                                                   int workers) {
  if (fields.size() != D) throw std::invalid_argument("expected one field per vector component");
  // The components concurrently, one host thread each (b200::for_components);
  // each call checks its arguments before any work, like the reference's.
  std::array<LagrangianValues, D> out;
  b200::for_components<D>(D, [&](std::size_t c) { out[c] = interpolate(fields[c], points, kernel, workers); });
  return out;
}

}  // namespace ib
