// How many bytes an evenly sharded all-gather / reduce-scatter moves - the
// unit of every count in this project (cost model, NIC emulator counters,
// bench).  Same two functions and constants as the reference header
// (proj/include/shardsim/collective.hpp:8-33), so byte parity is an integer
// comparison.
#pragma once

#include <cassert>
#include <cstdint>

namespace shardsim {

inline constexpr std::uint64_t kKiB = 1024ull;
inline constexpr std::uint64_t kMiB = 1024ull * kKiB;
inline constexpr std::uint64_t kGiB = 1024ull * kMiB;

namespace detail {
// (k - 1) / k of x, rounded down, computed without x * (k - 1) overflowing.
inline std::uint64_t share_of_peers(std::uint64_t x, std::uint64_t k) {
  return (x / k) * (k - 1) + ((x % k) * (k - 1)) / k;
}
}  // namespace detail

// One node's NIC bytes for a collective over `nodes` nodes of a `bytes` payload
// (zero for a single node).
inline std::uint64_t ag_inter_bytes(std::uint64_t bytes, int nodes) {
  assert(nodes >= 1);
  return nodes <= 1 ? 0 : detail::share_of_peers(bytes, static_cast<std::uint64_t>(nodes));
}

// One GPU's bytes in a ring all-gather of `bytes` over `gpus` GPUs.
inline std::uint64_t ring_intra_bytes(std::uint64_t bytes, int gpus) {
  assert(gpus >= 1);
  return gpus <= 1 ? 0 : detail::share_of_peers(bytes, static_cast<std::uint64_t>(gpus));
}

}  // namespace shardsim
