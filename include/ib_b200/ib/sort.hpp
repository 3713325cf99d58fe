// ib_b200/ib/sort.hpp -- overlay of the reference's ib/sort.hpp: the stable
// 32-bit key-value sort runs on the device (onesweep LSD radix sort,
// ibc_key_value_sort), bit-identical to the reference's (sort.hpp:12-71:
// equal keys keep their input order, so the result is unique).
#pragma once

#include <cassert>
#include <cstdint>
#include <span>
#include <type_traits>

#include "b200.hpp"
#include "grid.hpp"

namespace ib {

template <class Payload>
void key_value_sort(std::span<SortKey> keys, std::span<Payload> payload, int workers) {
  static_assert(std::is_trivially_copyable_v<Payload>, "payload is moved as raw bytes");
  assert(keys.size() == payload.size());
  b200::check(ibc_key_value_sort(b200::context(), keys.data(), payload.data(), sizeof(Payload),
                                 keys.size(), workers));
}

}  // namespace ib
