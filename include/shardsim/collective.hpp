// Byte-splitting rules for evenly sharded bulk-synchronous collectives.
//
// Reference: proj/include/shardsim/collective.hpp:8-33.  Every byte count the
// cost model reports - and every byte counter the B200 NIC emulator keeps -
// is defined through these two helpers, so parity is integer equality.
#pragma once

#include <cassert>
#include <cstdint>

namespace shardsim {

inline constexpr std::uint64_t kKiB = std::uint64_t{1} << 10;
inline constexpr std::uint64_t kMiB = std::uint64_t{1} << 20;
inline constexpr std::uint64_t kGiB = std::uint64_t{1} << 30;

namespace detail {
// floor(x * (k - 1) / k) without forming the (possibly overflowing) product.
inline std::uint64_t all_but_one_share(std::uint64_t x, std::uint64_t k) {
  const std::uint64_t q = x / k, r = x % k;
  return q * (k - 1) + (r * (k - 1)) / k;
}
}  // namespace detail

/// Bytes through one node's NIC when `payload` bytes, sharded over
/// `scope_nodes` nodes, are all-gathered (or reduce-scattered).
inline std::uint64_t ag_inter_bytes(std::uint64_t payload, int scope_nodes) {
  assert(scope_nodes >= 1);
  return scope_nodes > 1 ? detail::all_but_one_share(payload, std::uint64_t(scope_nodes)) : 0;
}

/// Bytes each GPU moves in a ring all-gather of `payload` over `ring_gpus`.
inline std::uint64_t ring_intra_bytes(std::uint64_t payload, int ring_gpus) {
  assert(ring_gpus >= 1);
  return ring_gpus > 1 ? detail::all_but_one_share(payload, std::uint64_t(ring_gpus)) : 0;
}

}  // namespace shardsim
