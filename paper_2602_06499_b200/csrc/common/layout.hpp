// Layer layout shared by the kernels and the runtime.
//
// A layer is E elements in natural (model) order, viewed as C 16-byte chunks.
// The chunk mask splits it into a trainable and a frozen portion (shardsim's
// two ParamState portions, reference schedule.hpp:43-50).  Each portion is the
// mask-order compaction of its chunks, padded to a multiple of G chunks and
// split G ways; global shard r = j*N + n lives on (node n, local GPU j), so
// the intra-node slice j (p^intra) is contiguous.
#pragma once

#include <cstdint>
#include <vector>

namespace fcdp {

inline constexpr int kChunkBytes = 16;
inline constexpr int kMaxLocal = 8;  // GPUs per emulated node (NVLink peers)
inline constexpr int kMaxNodes = 8;

// What the kernels need, by value.  Device pointers only.
struct LayoutDev {
  std::int64_t chunks = 0;        // C
  std::int64_t words = 0;         // ceil(C / 32) mask words
  const std::uint32_t* bits = nullptr;  // trainable bit per chunk
  const std::uint32_t* tpre = nullptr;  // exclusive prefix of trainable chunks per word
  std::int64_t pt = 0, pf = 0;    // trainable / frozen chunk counts
  std::int64_t shard_t = 0, shard_f = 0;  // chunks per shard (padded / G)
  std::int64_t slice_t = 0, slice_f = 0;  // chunks per intra slice (N shards)
  int nodes = 1, local = 1;       // N, g
  int elem_bytes = 2;
  // Sparse trainable mask (e.g. LoRA: 0.26% of a Llama-7B block): the mask
  // words holding at least one trainable chunk, ascending.  ntwords > 0 only
  // when they are under half of all words; the trainable-only gather and the
  // reduce-scatter then walk this list, so their work follows the trainable
  // bytes instead of the layer size.
  const std::uint32_t* twords = nullptr;
  std::int64_t ntwords = 0;
};

// Host-side layout: owns the mask metadata and its device copy.
struct Layout {
  LayoutDev dev;                        // device pointers filled by upload()
  std::vector<std::uint32_t> bits, tpre;
  // For the reduce-scatter: mask-word range [word_begin[j], word_end[j]) that
  // holds every trainable chunk of intra slice j.
  std::vector<std::int64_t> rs_word_begin, rs_word_end;
  // Active trainable words (see LayoutDev::twords) and, per slice j, the
  // index range [rs_tw_begin[j], rs_tw_end[j]) of them it covers.
  std::vector<std::uint32_t> twords;
  std::vector<std::int64_t> rs_tw_begin, rs_tw_end;
  bool sparse_t() const { return !twords.empty() && 2 * static_cast<std::int64_t>(twords.size()) < dev.words; }

  bool dense_trainable() const { return dev.pt == dev.chunks; }
  bool dense_frozen() const { return dev.pf == dev.chunks; }
  // Real (unpadded) chunks of portion shard r.
  std::int64_t real_chunks(bool frozen, int r) const {
    const std::int64_t per = frozen ? dev.shard_f : dev.shard_t;
    const std::int64_t total = frozen ? dev.pf : dev.pt;
    const std::int64_t lo = per * r;
    return lo >= total ? 0 : (total - lo < per ? total - lo : per);
  }
  std::int64_t real_slice_chunks(bool frozen, int j) const {
    std::int64_t s = 0;
    for (int n = 0; n < dev.nodes; ++n) s += real_chunks(frozen, j * dev.nodes + n);
    return s;
  }
};

// Builds bits / prefix / shard geometry from a per-chunk byte mask.
Layout build_layout(std::int64_t chunks, const std::uint8_t* mask, int elem_bytes, int nodes,
                    int local);

}  // namespace fcdp
