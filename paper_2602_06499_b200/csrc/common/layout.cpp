#include "common/layout.hpp"

#include <algorithm>
#include <stdexcept>

namespace fcdp {

Layout build_layout(std::int64_t chunks, const std::uint8_t* mask, int elem_bytes, int nodes,
                    int local) {
  if (chunks <= 0) throw std::invalid_argument("layout: a layer needs at least one 16-byte chunk");
  if (elem_bytes != 2 && elem_bytes != 4) throw std::invalid_argument("layout: elem_bytes must be 2 or 4");
  if (nodes < 1 || nodes > kMaxNodes || local < 1 || local > kMaxLocal)
    throw std::invalid_argument("layout: unsupported emulated-node geometry");

  Layout L;
  L.dev.chunks = chunks;
  L.dev.words = (chunks + 31) / 32;
  L.dev.nodes = nodes;
  L.dev.local = local;
  L.dev.elem_bytes = elem_bytes;
  L.bits.assign(static_cast<std::size_t>(L.dev.words), 0u);
  L.tpre.assign(static_cast<std::size_t>(L.dev.words), 0u);

  std::int64_t t = 0;
  for (std::int64_t w = 0; w < L.dev.words; ++w) {
    L.tpre[w] = static_cast<std::uint32_t>(t);
    std::uint32_t b = 0;
    for (int i = 0; i < 32; ++i) {
      const std::int64_t c = w * 32 + i;
      if (c < chunks && (mask == nullptr || mask[c] != 0)) b |= 1u << i;
    }
    L.bits[w] = b;
    t += __builtin_popcount(b);
  }
  if (t > 0xffffffffll) throw std::invalid_argument("layout: layer too large for 32-bit chunk ranks");
  L.dev.pt = t;
  L.dev.pf = chunks - t;

  const std::int64_t G = static_cast<std::int64_t>(nodes) * local;
  auto padded = [G](std::int64_t p) { return (p + G - 1) / G * G; };
  L.dev.shard_t = padded(L.dev.pt) / G;
  L.dev.shard_f = padded(L.dev.pf) / G;
  L.dev.slice_t = L.dev.shard_t * nodes;
  L.dev.slice_f = L.dev.shard_f * nodes;

  // Word ranges per slice for the trainable reduce-scatter.
  L.rs_word_begin.assign(local, 0);
  L.rs_word_end.assign(local, 0);
  std::int64_t w = 0;
  for (int j = 0; j < local; ++j) {
    const std::int64_t k0 = j * L.dev.slice_t;
    const std::int64_t k1 = std::min<std::int64_t>((j + 1) * L.dev.slice_t, L.dev.pt);
    if (k0 >= k1) {
      L.rs_word_begin[j] = L.rs_word_end[j] = 0;
      continue;
    }
    // first word whose trainable range reaches rank k0
    while (w + 1 < L.dev.words && L.tpre[w + 1] <= k0) ++w;
    L.rs_word_begin[j] = w;
    std::int64_t we = w;
    while (we < L.dev.words && L.tpre[we] < k1) ++we;
    L.rs_word_end[j] = we;
  }
  for (std::int64_t i = 0; i < L.dev.words; ++i)
    if (L.bits[i]) L.twords.push_back(static_cast<std::uint32_t>(i));
  L.rs_tw_begin.assign(local, 0);
  L.rs_tw_end.assign(local, 0);
  for (int j = 0; j < local; ++j) {
    auto lo = std::lower_bound(L.twords.begin(), L.twords.end(), static_cast<std::uint32_t>(L.rs_word_begin[j]));
    auto hi = std::lower_bound(L.twords.begin(), L.twords.end(), static_cast<std::uint32_t>(L.rs_word_end[j]));
    L.rs_tw_begin[j] = lo - L.twords.begin();
    L.rs_tw_end[j] = hi - L.twords.begin();
  }
  return L;
}

}  // namespace fcdp
