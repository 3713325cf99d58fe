// ib_b200/ib/stats.hpp -- overlay of the reference's ib/stats.hpp: the
// kernel-evaluation counter lives in libibcuda.so, which adds
// n_points * support^d per operation exactly as the reference does
// (stats.hpp:9-25, spread.hpp:158, interpolate.hpp:55).
#pragma once

#include <cstdint>

#include "ibcuda.h"

namespace ib::stats {

inline std::uint64_t delta_evaluations() { return ibc_delta_evaluations(); }
inline void reset_delta_evaluations() { ibc_reset_delta_evaluations(); }
inline void add_delta_evaluations(std::uint64_t n) { ibc_add_delta_evaluations(n); }

}  // namespace ib::stats
