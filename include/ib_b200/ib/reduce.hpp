// ib_b200/ib/reduce.hpp -- overlay of the reference's ib/reduce.hpp: run
// counting and the segmented reduction run on the device
// (ibc_count_unique / ibc_collect_unique_keys / ibc_segmented_reduce_rows).
// Each run is summed as a left fold in index order: the reference's result
// at workers == 1, bit for bit, and within its 1e-12 at any worker count.
// Decreasing keys raise std::invalid_argument (the reference asserts).
#pragma once

#include <algorithm>
#include <cassert>
#include <cstdint>
#include <span>
#include <vector>

#include "b200.hpp"
#include "grid.hpp"

namespace ib {

namespace detail {

template <int = 0>
bool keys_sorted(std::span<const SortKey> keys) {  // reduce.hpp:16-19
  return std::is_sorted(keys.begin(), keys.end());
}

// Runs that start inside [begin, end) (reduce.hpp:21-28).
inline std::size_t count_run_starts(std::span<const SortKey> keys, std::size_t begin,
                                    std::size_t end) {
  std::size_t starts = 0;
  for (std::size_t i = begin; i < end; ++i) starts += (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  return starts;
}

// First key of every run -> out_keys; returns q (reduce.hpp:34-52).
inline std::size_t collect_unique_keys(std::span<const SortKey> sorted_keys,
                                       std::span<SortKey> out_keys, int /*workers*/) {
  std::size_t q = 0;
  b200::check(ibc_collect_unique_keys(b200::context(), sorted_keys.data(), sorted_keys.size(),
                                      out_keys.data(), out_keys.size(), &q));
  return q;
}

}  // namespace detail

// reduce.hpp:54-69.
inline std::size_t count_unique(std::span<const SortKey> sorted_keys, int workers = 1) {
  std::size_t q = 0;
  b200::check(ibc_count_unique(b200::context(), sorted_keys.data(), sorted_keys.size(), workers, &q));
  return q;
}

// reduce.hpp:70-137: sums consecutive rows of `width` doubles while their
// keys match; one key and one row per run; returns q.
inline std::size_t segmented_reduce_rows(std::span<const SortKey> sorted_keys,
                                         std::span<const double> values, std::size_t width,
                                         std::span<SortKey> out_keys, std::span<double> out_values,
                                         int workers) {
  assert(width >= 1);
  assert(values.size() == sorted_keys.size() * width);
  std::size_t q = 0;
  b200::check(ibc_segmented_reduce_rows(b200::context(), sorted_keys.data(), values.data(),
                                        sorted_keys.size(), width, out_keys.data(), out_keys.size(),
                                        out_values.data(), out_values.size(), workers, &q));
  return q;
}

// reduce.hpp:139-145.
inline std::size_t segmented_reduce(std::span<const SortKey> sorted_keys,
                                    std::span<const double> values, std::span<SortKey> out_keys,
                                    std::span<double> out_sums, int workers) {
  return segmented_reduce_rows(sorted_keys, values, 1, out_keys, out_sums, workers);
}

}  // namespace ib
