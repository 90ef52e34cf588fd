// sm_100a data-plane kernels for the FCDP parameter-movement hot path.
//
// Every kernel here is bandwidth-bound byte movement (HBM, NVLink peer reads):
//   * 16-byte vector loads/stores (one 16 B "chunk" per lane),
//   * mask handled per warp: 32 chunks = one mask word; the per-lane trainable
//     predicate is turned into ranks with __ballot_sync + __popc and a
//     per-word exclusive prefix precomputed once (the mask is static),
//   * kUnroll independent chunks in flight per lane (loads issued before
//     stores) to cover NVLink latency (~2 us) and HBM latency,
//   * grid = a multiple of the SM count, grid-stride loops.
// Reference semantics: the data plane is described, not implemented, by the
// reference (Algorithm 1); the CPU restatement these kernels
// are checked against bit-for-bit is oracle/fcdp_oracle.c.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "kernels/kernels.hpp"

namespace fcdp {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;
constexpr unsigned kFull = 0xffffffffu;

int g_sm_count = 0;

int grid_for(std::int64_t work_items, int per_block) {
  const std::int64_t want = (work_items + per_block - 1) / per_block;
  const std::int64_t cap = static_cast<std::int64_t>(sm_count()) * 8;
  return static_cast<int>(std::max<std::int64_t>(1, std::min(want, cap)));
}

__device__ __forceinline__ int slice_of(std::int64_t k, std::int64_t per, int local) {
  int j = 0;
#pragma unroll
  for (int i = 1; i < kMaxLocal; ++i) j += (i < local && k >= i * per) ? 1 : 0;
  return j;
}

__device__ __forceinline__ const uint4* pick(const SlicePtrs& s, int j) {
  // Unrolled select keeps the pointer table in registers (no local-memory spill).
  const void* p = s.p[0];
#pragma unroll
  for (int i = 1; i < kMaxLocal; ++i)
    if (j == i) p = s.p[i];
  return static_cast<const uint4*>(p);
}

// ------------------------------------------------------------------ expand
// Intra-node all-gather fused with the PEFT expansion: natural chunk c takes
// its value from rank k of its portion, which lives in slice k / slice_size
// (that GPU's memory, local or NVLink peer).
// Slice lookup with the local GPU count as a compile-time constant: for g = 1
// it vanishes, for g > 1 it is g - 1 predicated compares (no division).
template <int kG>
__device__ __forceinline__ int slice_of_g(int k, int per) {
  int j = 0;
#pragma unroll
  for (int i = 1; i < kG; ++i) j += k >= i * per ? 1 : 0;
  return j;
}

template <int kG>
__device__ __forceinline__ const uint4* pick_g(const SlicePtrs& s, int j) {
  const void* p = s.p[0];
#pragma unroll
  for (int i = 1; i < kG; ++i)
    if (j == i) p = s.p[i];
  return static_cast<const uint4*>(p);
}

// 32-bit chunk indices (the launcher rejects layers of >= 2^31 chunks, 32 GiB):
// this loop is issue-bound as much as memory-bound, and 64-bit index math
// doubled its instruction count.
// kSparse (trainable-only gathers of a sparse mask): warps walk the active
// trainable words L.twords instead of every mask word.
template <bool kWriteT, bool kWriteF, int kG, bool kSparse = false>
__global__ void __launch_bounds__(kThreads) expand_kernel(LayoutDev L, SlicePtrs ts, SlicePtrs fs,
                                                          uint4* __restrict__ out) {
  static_assert(!kSparse || (kWriteT && !kWriteF), "the active-word list covers trainable chunks only");
  const int lane = threadIdx.x & 31;
  const int warp = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const unsigned below = (1u << lane) - 1u;
  const int words = static_cast<int>(kSparse ? L.ntwords : L.words), chunks = static_cast<int>(L.chunks);
  const int per_t = static_cast<int>(L.slice_t), per_f = static_cast<int>(L.slice_f);
  for (int w0 = warp; w0 < words; w0 += nwarps * kUnroll) {
    // phase 1: the mask words and prefixes of all kUnroll groups (independent loads)
    unsigned bits[kUnroll];
    int pre[kUnroll], wid[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int i = w0 + u * nwarps;
      const int w = i < words ? (kSparse ? static_cast<int>(__ldg(L.twords + i)) : i) : 0;
      wid[u] = w;
      bits[u] = i < words ? __ldg(L.bits + w) : 0u;
      pre[u] = i < words ? static_cast<int>(__ldg(L.tpre + w)) : 0;
    }
    // phase 2: ranks -> source addresses; phase 3: all data loads in flight
    uint4 v[kUnroll];
    int dst[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int c = (w0 + u * nwarps < words) ? wid[u] * 32 + lane : chunks;
      const bool valid = c < chunks;
      const bool tr = valid && ((bits[u] >> lane) & 1u);
      // the mask word's own bits are the ballot of the lanes' predicates
      const int kt = pre[u] + __popc(bits[u] & below);
      dst[u] = -1;
      if (valid && (tr ? kWriteT : kWriteF)) {
        const int k = tr ? kt : c - kt;
        const int per = tr ? per_t : per_f;
        const int j = slice_of_g<kG>(k, per);
        v[u] = pick_g<kG>(tr ? ts : fs, j)[k - j * per];
        dst[u] = c;
      }
    }
    // phase 4: stores
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dst[u] >= 0) out[dst[u]] = v[u];
  }
}

// Dense portion (no mask): natural = concat of the g slices (each trimmed to
// the real chunk count).  blockIdx.y selects the source slice.
__global__ void __launch_bounds__(kThreads) concat_kernel(SlicePtrs src, std::int64_t per,
                                                          std::int64_t total, uint4* __restrict__ out) {
  // Block-contiguous tiles of kThreads*kUnroll chunks (16 KiB): a warp's kUnroll
  // loads hit consecutive 512 B segments of one tile, so DRAM pages stay open.
  const int j = blockIdx.y;
  const std::int64_t lo = j * per;
  if (lo >= total) return;
  const std::int64_t n = std::min(per, total - lo);
  const uint4* __restrict__ s = pick(src, j);
  uint4* __restrict__ d = out + lo;
  constexpr std::int64_t kTile = static_cast<std::int64_t>(kThreads) * kUnroll;
  const std::int64_t tiles = (n + kTile - 1) / kTile;
  for (std::int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const std::int64_t base = t * kTile + threadIdx.x;
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + u * kThreads < n) v[u] = __ldcs(s + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + u * kThreads < n) d[base + u * kThreads] = v[u];
  }
}

// ---------------------------------------------------------- TMA bulk copy
// Dense gathers and the own-shard pack are pure copies: one elected thread per
// CTA drives the Tensor Memory Accelerator with 1-D bulk copies
// (cp.async.bulk global->shared with an mbarrier transaction count, then
// shared->global), kStages 32 KiB tiles in flight per SM.  One warp per SM
// moves the bytes, so the copy leaves the SMs to the concurrently running
// GEMMs of the driving model.  Sources may be NVLink peer mappings.
constexpr int kBulkTile = 32 * 1024;
constexpr int kBulkStages = 4;

struct BulkSegs {
  const unsigned char* src[kMaxLocal + 1];
  unsigned char* dst[kMaxLocal + 1];
  std::int64_t bytes[kMaxLocal + 1];
  std::int64_t tile_base[kMaxLocal + 2];  // exclusive prefix of tiles per segment
  int n;
};

__device__ __forceinline__ void bulk_tile(const BulkSegs& s, std::int64_t t, const unsigned char*& src,
                                          unsigned char*& dst, unsigned& bytes) {
  int k = 0;
#pragma unroll
  for (int i = 1; i <= kMaxLocal; ++i)
    if (i < s.n && t >= s.tile_base[i]) k = i;
  const std::int64_t off = (t - s.tile_base[k]) * kBulkTile;
  const std::int64_t rem = s.bytes[k] - off;
  bytes = static_cast<unsigned>(rem < kBulkTile ? rem : kBulkTile);
  src = s.src[k] + off;
  dst = s.dst[k] + off;
}

__global__ void __launch_bounds__(32) bulk_copy_kernel(BulkSegs segs) {
  extern __shared__ __align__(1024) unsigned char bulk_smem[];
  auto stage = reinterpret_cast<unsigned char(*)[kBulkTile]>(bulk_smem);
  auto bar = reinterpret_cast<unsigned long long*>(bulk_smem + kBulkStages * kBulkTile);
  if (threadIdx.x != 0) return;
  const std::int64_t total = segs.tile_base[segs.n];
  const std::int64_t n = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (n == 0) return;
  for (int i = 0; i < kBulkStages; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(&bar[i]))));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  auto issue_load = [&](std::int64_t i) {
    const int st = static_cast<int>(i % kBulkStages);
    const unsigned char* src;
    unsigned char* dst;
    unsigned bytes;
    bulk_tile(segs, blockIdx.x + i * gridDim.x, src, dst, bytes);
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[st]));
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(&stage[st][0]));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
  };
  for (std::int64_t i = 0; i < kBulkStages - 1 && i < n; ++i) issue_load(i);
  for (std::int64_t i = 0; i < n; ++i) {
    // the stage refilled below last held tile i-1, whose store must have read it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (i + kBulkStages - 1 < n) issue_load(i + kBulkStages - 1);
    const int st = static_cast<int>(i % kBulkStages);
    const unsigned phase = static_cast<unsigned>((i / kBulkStages) & 1);
    const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(&bar[st]));
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(b), "r"(phase)
          : "memory");
    const unsigned char* src;
    unsigned char* dst;
    unsigned bytes;
    bulk_tile(segs, blockIdx.x + i * gridDim.x, src, dst, bytes);
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&stage[st][0]));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA copies keep 128 KiB of shared memory per CTA, which cannot co-reside
// with the driving model's GEMM CTAs; the SM copy (no smem, 32 registers)
// slots in beside them.  FCDP_COPY=tma selects the TMA path.
bool use_tma_copy() {
  static const bool on = [] {
    const char* v = std::getenv("FCDP_COPY");
    return v && std::string(v) == "tma";
  }();
  return on;
}

cudaError_t launch_bulk(const BulkSegs& segs_in, cudaStream_t s) {
  BulkSegs segs = segs_in;
  std::int64_t tiles = 0;
  for (int i = 0; i < segs.n; ++i) {
    segs.tile_base[i] = tiles;
    tiles += (segs.bytes[i] + kBulkTile - 1) / kBulkTile;
  }
  segs.tile_base[segs.n] = tiles;
  if (tiles == 0) return cudaSuccess;
  constexpr int kSmem = kBulkStages * kBulkTile + kBulkStages * 8;
  static bool configured = false;
  if (!configured) {
    const cudaError_t e = cudaFuncSetAttribute(bulk_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int grid = static_cast<int>(std::min<std::int64_t>(tiles, static_cast<std::int64_t>(sm_count())));
  bulk_copy_kernel<<<grid, 32, kSmem, s>>>(segs);
  return cudaGetLastError();
}

// --------------------------------------------------------------- partition
// natural -> (trainable, frozen) portion vectors: warp-ballot compaction.
__global__ void __launch_bounds__(kThreads) partition_kernel(LayoutDev L, const uint4* __restrict__ in,
                                                             uint4* __restrict__ t, uint4* __restrict__ f) {
  const int lane = threadIdx.x & 31;
  const std::int64_t warp = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
  const unsigned below = (1u << lane) - 1u;
  for (std::int64_t w = warp; w < L.words; w += nwarps) {
    const std::int64_t c = w * 32 + lane;
    const bool valid = c < L.chunks;
    const bool tr = valid && ((__ldg(L.bits + w) >> lane) & 1u);
    const unsigned ballot = __ballot_sync(kFull, tr);
    const std::int64_t kt = static_cast<std::int64_t>(__ldg(L.tpre + w)) + __popc(ballot & below);
    if (!valid) continue;
    const uint4 v = in[c];
    if (tr)
      t[kt] = v;
    else
      f[c - kt] = v;
  }
}

// ------------------------------------------------------------ reduce-scatter
template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int kN = 8;
  __device__ static void add(float* acc, const uint4& q) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] = __fadd_rn(acc[2 * i], f.x);
      acc[2 * i + 1] = __fadd_rn(acc[2 * i + 1], f.y);
    }
  }
  __device__ static uint4 pack(const float* a) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(a[2 * i], a[2 * i + 1]);
    return q;
  }
  __device__ static float load1(const void* p, std::int64_t i) {
    return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  }
  __device__ static void store1(void* p, std::int64_t i, float x) {
    static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
  }
};
template <>
struct Vec<float> {
  static constexpr int kN = 4;
  __device__ static void add(float* acc, const uint4& q) {
    acc[0] = __fadd_rn(acc[0], __uint_as_float(q.x));
    acc[1] = __fadd_rn(acc[1], __uint_as_float(q.y));
    acc[2] = __fadd_rn(acc[2], __uint_as_float(q.z));
    acc[3] = __fadd_rn(acc[3], __uint_as_float(q.w));
  }
  __device__ static uint4 pack(const float* a) {
    return make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]),
                      __float_as_uint(a[3]));
  }
  __device__ static float load1(const void* p, std::int64_t i) { return static_cast<const float*>(p)[i]; }
  __device__ static void store1(void* p, std::int64_t i, float x) { static_cast<float*>(p)[i] = x; }
};

struct RsArgs {
  std::int64_t k0, k1;          // trainable ranks of this slice
  std::int64_t own_lo, own_hi;  // slice-relative chunk range of this rank's shard
  float scale;
  int final_scale;
  int local;
};

template <typename T, int kG>
__device__ __forceinline__ void rs_emit_q(const RsArgs& a, const uint4 (&q)[kG], std::int64_t rel,
                                          float* own_out, uint4* wire_out) {
  constexpr int V = Vec<T>::kN;
  float acc[V];
#pragma unroll
  for (int e = 0; e < V; ++e) acc[e] = 0.0f;
#pragma unroll
  for (int i = 0; i < kG; ++i)  // fixed order 0..g-1: deterministic
    Vec<T>::add(acc, q[i]);
  if (rel >= a.own_lo && rel < a.own_hi) {
    float4* o = reinterpret_cast<float4*>(own_out + (rel - a.own_lo) * V);
#pragma unroll
    for (int e = 0; e < V; e += 4) {
      float4 r = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
      if (a.final_scale) {
        r.x = __fmul_rn(r.x, a.scale);
        r.y = __fmul_rn(r.y, a.scale);
        r.z = __fmul_rn(r.z, a.scale);
        r.w = __fmul_rn(r.w, a.scale);
      }
      __stcs(o + e / 4, r);
    }
  } else {
    __stcs(wire_out + rel, Vec<T>::pack(acc));
  }
}

template <typename T, int kG>
__device__ __forceinline__ void rs_emit(const RsArgs& a, const GradPtrs& g, std::int64_t c,
                                        std::int64_t rel, float* own_out, uint4* wire_out) {
  uint4 q[kG];
#pragma unroll
  for (int i = 0; i < kG; ++i) q[i] = static_cast<const uint4*>(g.p[i])[c];
  rs_emit_q<T, kG>(a, q, rel, own_out, wire_out);
}

// [wb, we): mask words, or (sparse mask) indices into the active-word list L.twords
template <typename T, int kG, bool kSparse = false>
__global__ void __launch_bounds__(kThreads) rs_masked_kernel(LayoutDev L, GradPtrs g, RsArgs a,
                                                             std::int64_t wb, std::int64_t we,
                                                             float* __restrict__ own_out,
                                                             uint4* __restrict__ wire_out) {
  const int lane = threadIdx.x & 31;
  const std::int64_t warp = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
  const unsigned below = (1u << lane) - 1u;
  for (std::int64_t i = wb + warp; i < we; i += nwarps) {
    const std::int64_t w = kSparse ? static_cast<std::int64_t>(__ldg(L.twords + i)) : i;
    const std::int64_t c = w * 32 + lane;
    const bool valid = c < L.chunks;
    const bool tr = valid && ((__ldg(L.bits + w) >> lane) & 1u);
    const unsigned ballot = __ballot_sync(kFull, tr);
    const std::int64_t kt = static_cast<std::int64_t>(__ldg(L.tpre + w)) + __popc(ballot & below);
    if (tr && kt >= a.k0 && kt < a.k1) rs_emit<T, kG>(a, g, c, kt - a.k0, own_out, wire_out);
  }
}

// Dense slice: kU chunks per lane per trip with every one of the kU * g
// gradient loads (local HBM or NVLink peer) issued before any add or store -
// 8 independent 16-byte loads in flight per lane whatever g is (the loads of
// chunk u+1 no longer wait behind chunk u's stores, which may alias them).
template <typename T, int kG>
__global__ void __launch_bounds__(kThreads) rs_dense_kernel(GradPtrs g, RsArgs a, float* __restrict__ own_out,
                                                            uint4* __restrict__ wire_out) {
  constexpr int kU = kG >= 8 ? 1 : 8 / kG;
  const std::int64_t n = a.k1 - a.k0;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if constexpr (kG == 1) {
    // g = 1 (kU = 8): a layer launch is only ~2.6 trips per thread, so the last,
    // partial trip is predicated instead of a one-load-at-a-time tail
    // (kernel bench: 0.66 -> 0.71 of HBM; for g > 1 the plain loop measured better)
    for (; i < n; i += kU * stride) {
      uint4 q[kU][1];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i + u * stride < n) q[u][0] = __ldcs(static_cast<const uint4*>(g.p[0]) + a.k0 + i + u * stride);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (i + u * stride < n) rs_emit_q<T, 1>(a, q[u], i + u * stride, own_out, wire_out);
    }
    return;
  }
  for (; i + (kU - 1) * stride < n; i += kU * stride) {
    uint4 q[kU][kG];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int k = 0; k < kG; ++k) q[u][k] = __ldcs(static_cast<const uint4*>(g.p[k]) + a.k0 + i + u * stride);
#pragma unroll
    for (int u = 0; u < kU; ++u) rs_emit_q<T, kG>(a, q[u], i + u * stride, own_out, wire_out);
  }
  for (; i < n; i += stride) rs_emit<T, kG>(a, g, a.k0 + i, i, own_out, wire_out);
}

template <typename T>
__device__ __forceinline__ float4 load4(const void* p, std::int64_t i4);
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const void* p, std::int64_t i4) {
  const uint2 q = __ldcs(static_cast<const uint2*>(p) + i4);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
template <>
__device__ __forceinline__ float4 load4<float>(const void* p, std::int64_t i4) {
  return __ldcs(static_cast<const float4*>(p) + i4);
}

// Inter-node epilogue, 4 elements per lane (n is a multiple of 4: whole chunks).
template <typename T>
__global__ void __launch_bounds__(kThreads) rs_finalize_kernel(std::int64_t n, int nodes, int node,
                                                               const float* __restrict__ own,
                                                               const void* __restrict__ wire,
                                                               std::int64_t stride, float scale,
                                                               float* __restrict__ out) {
  const std::int64_t n4 = n / 4, s4 = stride / 4;
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += step) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int m = 0; m < nodes; ++m) {  // fixed node order
      const float4 x = m == node ? __ldcs(reinterpret_cast<const float4*>(own) + i) : load4<T>(wire, m * s4 + i);
      acc.x = __fadd_rn(acc.x, x.x);
      acc.y = __fadd_rn(acc.y, x.y);
      acc.z = __fadd_rn(acc.z, x.z);
      acc.w = __fadd_rn(acc.w, x.w);
    }
    __stcs(reinterpret_cast<float4*>(out) + i,
           make_float4(__fmul_rn(acc.x, scale), __fmul_rn(acc.y, scale), __fmul_rn(acc.z, scale),
                       __fmul_rn(acc.w, scale)));
  }
}

// -------------------------------------------------------------------- Adam
__device__ __forceinline__ float adam_one(const AdamParams& p, float omb1, float omb2, float g, float& w,
                                          float& m, float& v) {
  const float mi = __fmaf_rn(p.beta1, m, __fmul_rn(omb1, g));
  const float vi = __fmaf_rn(p.beta2, v, __fmul_rn(__fmul_rn(omb2, g), g));
  const float mhat = __fdiv_rn(mi, p.bias_c1);
  const float vhat = __fdiv_rn(vi, p.bias_c2);
  const float denom = __fadd_rn(__fsqrt_rn(vhat), p.eps);
  const float upd = __fadd_rn(__fdiv_rn(mhat, denom), __fmul_rn(p.weight_decay, w));
  w = __fsub_rn(w, __fmul_rn(p.lr, upd));
  m = mi;
  v = vi;
  return w;
}

template <typename T>
__device__ __forceinline__ void store4(void* param, std::int64_t i4, const float4& w);
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(void* param, std::int64_t i4, const float4& w) {
  uint2 q;
  __nv_bfloat162 a = __floats2bfloat162_rn(w.x, w.y), b = __floats2bfloat162_rn(w.z, w.w);
  q.x = *reinterpret_cast<unsigned*>(&a);
  q.y = *reinterpret_cast<unsigned*>(&b);
  __stcs(static_cast<uint2*>(param) + i4, q);
}
template <>
__device__ __forceinline__ void store4<float>(void* param, std::int64_t i4, const float4& w) {
  __stcs(static_cast<float4*>(param) + i4, w);
}

// AdamW over the fp32 trainable arena: 16-byte vectors (4 elements per lane),
// streaming cache hints (every byte is touched once per step).
template <typename T>
__global__ void __launch_bounds__(kThreads) adam_kernel(std::int64_t n, AdamParams p, float* __restrict__ master,
                                                        float* __restrict__ m, float* __restrict__ v,
                                                        const float* __restrict__ grad, void* __restrict__ param) {
  const float omb1 = __fsub_rn(1.0f, p.beta1), omb2 = __fsub_rn(1.0f, p.beta2);
  const std::int64_t n4 = n / 4;
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  const std::int64_t tid = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  float4* W4 = reinterpret_cast<float4*>(master);
  float4* M4 = reinterpret_cast<float4*>(m);
  float4* V4 = reinterpret_cast<float4*>(v);
  const float4* G4 = reinterpret_cast<const float4*>(grad);
  for (std::int64_t i = tid; i < n4; i += step) {
    const float4 g = __ldcs(G4 + i);
    float4 w = __ldcs(W4 + i), mm = __ldcs(M4 + i), vv = __ldcs(V4 + i);
    adam_one(p, omb1, omb2, g.x, w.x, mm.x, vv.x);
    adam_one(p, omb1, omb2, g.y, w.y, mm.y, vv.y);
    adam_one(p, omb1, omb2, g.z, w.z, mm.z, vv.z);
    adam_one(p, omb1, omb2, g.w, w.w, mm.w, vv.w);
    __stcs(W4 + i, w);
    __stcs(M4 + i, mm);
    __stcs(V4 + i, vv);
    store4<T>(param, i, w);
  }
  for (std::int64_t i = n4 * 4 + tid; i < n; i += step) {
    float w = master[i], mm = m[i], vv = v[i];
    adam_one(p, omb1, omb2, grad[i], w, mm, vv);
    master[i] = w;
    m[i] = mm;
    v[i] = vv;
    Vec<T>::store1(param, i, w);
  }
}

// G = 1 (one GPU holds the whole dense layer): the reduce-scatter is the
// identity up to its fp32 widen + 1/G scale, so it is fused into AdamW, which
// reads the gradient straight from where backward left it - the engine's
// natural gradient slot or the autograd buffers themselves (segments) - in the
// parameter dtype.  Per 16-byte gradient chunk (V elements):
//   g = (0 + x) * scale      exactly the rs_dense_kernel<T, 1> arithmetic
//   AdamW(g)                 exactly adam_kernel's arithmetic
// so results are bit-identical to RS-then-AdamW; the fp32 gradient shard is
// written only when asked (keep_grad: readback for tests), saving 8 B/param of
// HBM traffic and the separate RS pass.  Chunks no segment covers have g = 0.
// The launcher turns the caller's segments into a cover of the whole layer
// (gaps become zero-gradient segments) and gives every segment a share of the
// grid proportional to its size, so a block finds its segment once and then
// streams it like adam_kernel: 4 elements per lane, 2 groups per trip.
constexpr int kMaxCover = 2 * kMaxGradSegs + 1;
struct AdamCover {
  int n;
  int block0[kMaxCover + 1];         // first block of each segment; block0[n] = grid
  std::int64_t elem0[kMaxCover];     // first element of the segment in the layer
  std::int64_t count[kMaxCover];     // elements (multiple of 4)
  const void* src[kMaxCover];        // gradient (param dtype), nullptr: zero gradient
};

template <typename T>
__device__ __forceinline__ float4 grad4(const void* src, std::int64_t i4) {
  if (!src) return make_float4(0.f, 0.f, 0.f, 0.f);
  return load4<T>(src, i4);
}

template <typename T>
__device__ __forceinline__ void adam_grad4(const AdamParams& p, float omb1, float omb2, float scale, float4 g,
                                           float4 w, float4 mm, float4 vv, std::int64_t e4, float* master, float* m,
                                           float* v, void* param, float* keep) {
  // g = (0 + x) * scale: exactly the rs_dense_kernel<T, 1> final-scale arithmetic
  g = make_float4(__fmul_rn(__fadd_rn(0.0f, g.x), scale), __fmul_rn(__fadd_rn(0.0f, g.y), scale),
                  __fmul_rn(__fadd_rn(0.0f, g.z), scale), __fmul_rn(__fadd_rn(0.0f, g.w), scale));
  if (keep) __stcs(reinterpret_cast<float4*>(keep) + e4, g);
  adam_one(p, omb1, omb2, g.x, w.x, mm.x, vv.x);
  adam_one(p, omb1, omb2, g.y, w.y, mm.y, vv.y);
  adam_one(p, omb1, omb2, g.z, w.z, mm.z, vv.z);
  adam_one(p, omb1, omb2, g.w, w.w, mm.w, vv.w);
  __stcs(reinterpret_cast<float4*>(master) + e4, w);
  __stcs(reinterpret_cast<float4*>(m) + e4, mm);
  __stcs(reinterpret_cast<float4*>(v) + e4, vv);
  store4<T>(param, e4, w);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) adam_grad_kernel(AdamCover cv, AdamParams p, float scale,
                                                             float* __restrict__ master, float* __restrict__ m,
                                                             float* __restrict__ v, void* __restrict__ param,
                                                             float* __restrict__ keep) {
  int s = 0;
  while (s + 1 < cv.n && static_cast<int>(blockIdx.x) >= cv.block0[s + 1]) ++s;
  const float omb1 = __fsub_rn(1.0f, p.beta1), omb2 = __fsub_rn(1.0f, p.beta2);
  const std::int64_t groups = cv.count[s] / 4, base4 = cv.elem0[s] / 4;
  const void* src = cv.src[s];
  const std::int64_t step = static_cast<std::int64_t>(cv.block0[s + 1] - cv.block0[s]) * blockDim.x;
  std::int64_t i = static_cast<std::int64_t>(blockIdx.x - cv.block0[s]) * blockDim.x + threadIdx.x;
  const float4* W4 = reinterpret_cast<const float4*>(master);
  const float4* M4 = reinterpret_cast<const float4*>(m);
  const float4* V4 = reinterpret_cast<const float4*>(v);
  for (; i + step < groups; i += 2 * step) {
    const std::int64_t a = base4 + i, b = base4 + i + step;
    const float4 ga = grad4<T>(src, i), gb = grad4<T>(src, i + step);
    const float4 wa = __ldcs(W4 + a), ma = __ldcs(M4 + a), va = __ldcs(V4 + a);
    const float4 wb = __ldcs(W4 + b), mb = __ldcs(M4 + b), vb = __ldcs(V4 + b);
    adam_grad4<T>(p, omb1, omb2, scale, ga, wa, ma, va, a, master, m, v, param, keep);
    adam_grad4<T>(p, omb1, omb2, scale, gb, wb, mb, vb, b, master, m, v, param, keep);
  }
  for (; i < groups; i += step) {
    const std::int64_t a = base4 + i;
    adam_grad4<T>(p, omb1, omb2, scale, grad4<T>(src, i), __ldcs(W4 + a), __ldcs(M4 + a), __ldcs(V4 + a), a, master,
                  m, v, param, keep);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) widen_kernel(std::int64_t n, const void* __restrict__ src,
                                                         float* __restrict__ dst) {
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += step)
    dst[i] = Vec<T>::load1(src, i);
}

// --------------------------------------------------------------------- init
__device__ __forceinline__ std::uint64_t splitmix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <typename T>
__global__ void __launch_bounds__(kThreads) init_kernel(std::int64_t n, std::uint64_t seed, int layer,
                                                        const InitRange* __restrict__ ranges, int nr,
                                                        void* __restrict__ out) {
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t e = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += step) {
    float x = 0.0f;
    for (int r = 0; r < nr; ++r) {
      if (e < ranges[r].begin || e >= ranges[r].end) continue;
      if (ranges[r].kind == 1) {
        x = ranges[r].scale;
      } else {
        const std::uint64_t z =
            splitmix64(seed ^ (static_cast<std::uint64_t>(layer) << 40) ^ static_cast<std::uint64_t>(e));
        const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f);  // exact
        x = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), ranges[r].scale);
      }
      break;
    }
    Vec<T>::store1(out, e, x);
  }
}

// rows x (row_bytes) strided copy, 16-byte vectors (one third of a joint
// [tokens x 3h] projection to or from a dense [tokens x h] tensor).
__global__ void __launch_bounds__(kThreads) copy_rows_kernel(std::int64_t rows, int rv, const uint4* __restrict__ src,
                                                             std::int64_t ss, uint4* __restrict__ dst,
                                                             std::int64_t ds) {
  const std::int64_t n = rows * rv;
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += step) {
    const std::int64_t r = i / rv, c = i - r * rv;
    dst[r * ds + c] = __ldcs(src + r * ss + c);
  }
}

// Gradient hand-off of a masked (LoRA) layer: up to kMaxCopySegs small
// tensors copied into their places in the natural gradient slot by ONE launch
// (blockIdx.y = segment) instead of one memcpy each (launch-bound: 12 per layer).
struct CopySegs {
  const uint4* src[kMaxCopySegs];
  uint4* dst[kMaxCopySegs];
  std::int64_t chunks[kMaxCopySegs];
};

__global__ void __launch_bounds__(kThreads) seg_copy_kernel(CopySegs c) {
  const int k = blockIdx.y;
  const std::int64_t n = c.chunks[k];
  const uint4* __restrict__ src = c.src[k];
  uint4* __restrict__ dst = c.dst[k];
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + step < n; i += 2 * step) {
    const uint4 a = __ldcs(src + i), b = __ldcs(src + i + step);
    dst[i] = a;
    dst[i + step] = b;
  }
  for (; i < n; i += step) dst[i] = __ldcs(src + i);
}

__global__ void __launch_bounds__(kThreads) copy_kernel(const uint4* __restrict__ s, uint4* __restrict__ d,
                                                        std::int64_t n) {
  constexpr std::int64_t kTile = static_cast<std::int64_t>(kThreads) * kUnroll;
  const std::int64_t tiles = (n + kTile - 1) / kTile;
  for (std::int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const std::int64_t base = t * kTile + threadIdx.x;
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + u * kThreads < n) v[u] = __ldcs(s + base + u * kThreads);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (base + u * kThreads < n) d[base + u * kThreads] = v[u];
  }
}

}  // namespace

int sm_count() {
  if (g_sm_count == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      g_sm_count = n;
    else
      return 148;
  }
  return g_sm_count;
}

cudaError_t launch_partition(const Layout& L, const void* natural, void* t, void* f, cudaStream_t s) {
  const std::int64_t bytes = L.dev.chunks * kChunkBytes;
  if (L.dense_trainable()) return cudaMemcpyAsync(t, natural, bytes, cudaMemcpyDeviceToDevice, s);
  if (L.dense_frozen()) return cudaMemcpyAsync(f, natural, bytes, cudaMemcpyDeviceToDevice, s);
  partition_kernel<<<grid_for(L.dev.words * 32, kThreads), kThreads, 0, s>>>(
      L.dev, static_cast<const uint4*>(natural), static_cast<uint4*>(t), static_cast<uint4*>(f));
  return cudaGetLastError();
}

cudaError_t launch_expand(const Layout& L, const SlicePtrs& ts, const SlicePtrs& fs, void* natural,
                          int set, cudaStream_t s) {
  const bool want_t = set != kSetFrozen, want_f = set != kSetTrainable;
  uint4* out = static_cast<uint4*>(natural);
  if (L.dense_trainable() || L.dense_frozen()) {
    const bool tr = L.dense_trainable();
    if (tr ? !want_t : !want_f) return cudaSuccess;
    const std::int64_t per = tr ? L.dev.slice_t : L.dev.slice_f;
    if (!use_tma_copy()) {
      dim3 grid(std::max(1, grid_for(per, kThreads * kUnroll) / L.dev.local), L.dev.local);
      concat_kernel<<<grid, kThreads, 0, s>>>(tr ? ts : fs, per, L.dev.chunks, out);
      return cudaGetLastError();
    }
    BulkSegs segs{};
    for (int j = 0; j < L.dev.local; ++j) {
      const std::int64_t lo = j * per;
      if (lo >= L.dev.chunks) break;
      segs.src[segs.n] = static_cast<const unsigned char*>((tr ? ts : fs).p[j]);
      segs.dst[segs.n] = reinterpret_cast<unsigned char*>(out + lo);
      segs.bytes[segs.n] = std::min(per, L.dev.chunks - lo) * kChunkBytes;
      ++segs.n;
    }
    return launch_bulk(segs, s);
  }
  if (L.dev.words * 32 >= (std::int64_t{1} << 31) - (std::int64_t{1} << 24))
    return cudaErrorInvalidValue;  // 32-bit chunk indices (+ grid-stride headroom)
  const bool sparse = want_t && !want_f && L.dev.ntwords > 0;
  const int grid = grid_for((sparse ? L.dev.ntwords : L.dev.words) * 32, kThreads * kUnroll);
  auto go = [&](auto tag_g) {
    constexpr int G = decltype(tag_g)::value;
    if (want_t && want_f)
      expand_kernel<true, true, G><<<grid, kThreads, 0, s>>>(L.dev, ts, fs, out);
    else if (sparse)
      expand_kernel<true, false, G, true><<<grid, kThreads, 0, s>>>(L.dev, ts, fs, out);
    else if (want_t)
      expand_kernel<true, false, G><<<grid, kThreads, 0, s>>>(L.dev, ts, fs, out);
    else
      expand_kernel<false, true, G><<<grid, kThreads, 0, s>>>(L.dev, ts, fs, out);
  };
  switch (L.dev.local) {
    case 1: go(std::integral_constant<int, 1>{}); break;
    case 2: go(std::integral_constant<int, 2>{}); break;
    case 3: go(std::integral_constant<int, 3>{}); break;
    case 4: go(std::integral_constant<int, 4>{}); break;
    case 5: go(std::integral_constant<int, 5>{}); break;
    case 6: go(std::integral_constant<int, 6>{}); break;
    case 7: go(std::integral_constant<int, 7>{}); break;
    default: go(std::integral_constant<int, 8>{}); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_rs_slice(const Layout& L, const GradPtrs& grads, int j, int n, float scale,
                            bool final_scale, float* own_out, void* wire_out, cudaStream_t s,
                            int max_blocks) {
  RsArgs a;
  a.k0 = j * L.dev.slice_t;
  a.k1 = std::min<std::int64_t>((j + 1) * L.dev.slice_t, L.dev.pt);
  if (a.k0 >= a.k1) return cudaSuccess;
  a.own_lo = n * L.dev.shard_t;
  a.own_hi = a.own_lo + L.dev.shard_t;
  a.scale = scale;
  a.final_scale = final_scale ? 1 : 0;
  a.local = L.dev.local;
  uint4* wire = static_cast<uint4*>(wire_out);
  const bool bf16 = L.dev.elem_bytes == 2;
  const bool dense = L.dense_trainable();
  const bool sparse = !dense && L.dev.ntwords > 0;
  const std::int64_t wb = dense ? 0 : (sparse ? L.rs_tw_begin[j] : L.rs_word_begin[j]);
  const std::int64_t we = dense ? 0 : (sparse ? L.rs_tw_end[j] : L.rs_word_end[j]);
  int grid = dense ? grid_for(a.k1 - a.k0, kThreads * std::max(1, 8 / L.dev.local))
                   : grid_for((we - wb) * 32, kThreads);
  if (max_blocks > 0) grid = std::min(grid, max_blocks);
  auto go = [&](auto tag_t, auto tag_g) {
    using T = decltype(tag_t);
    constexpr int G = decltype(tag_g)::value;
    if (dense)
      rs_dense_kernel<T, G><<<grid, kThreads, 0, s>>>(grads, a, own_out, wire);
    else if (sparse)
      rs_masked_kernel<T, G, true><<<grid, kThreads, 0, s>>>(L.dev, grads, a, wb, we, own_out, wire);
    else
      rs_masked_kernel<T, G><<<grid, kThreads, 0, s>>>(L.dev, grads, a, wb, we, own_out, wire);
  };
  auto by_g = [&](auto tag_t) {
    switch (L.dev.local) {
      case 1: go(tag_t, std::integral_constant<int, 1>{}); break;
      case 2: go(tag_t, std::integral_constant<int, 2>{}); break;
      case 4: go(tag_t, std::integral_constant<int, 4>{}); break;
      case 8: go(tag_t, std::integral_constant<int, 8>{}); break;
      case 3: go(tag_t, std::integral_constant<int, 3>{}); break;
      case 5: go(tag_t, std::integral_constant<int, 5>{}); break;
      case 6: go(tag_t, std::integral_constant<int, 6>{}); break;
      default: go(tag_t, std::integral_constant<int, 7>{}); break;
    }
  };
  if (bf16)
    by_g(__nv_bfloat16{});
  else
    by_g(float{});
  return cudaGetLastError();
}

cudaError_t launch_rs_finalize(std::int64_t n_elems, int nodes, int node, int elem_bytes,
                               const float* own, const void* wire, std::int64_t wire_stride,
                               float scale, float* out, cudaStream_t s) {
  if (n_elems <= 0) return cudaSuccess;
  if (n_elems % 4 || wire_stride % 4) return cudaErrorInvalidValue;
  const int grid = grid_for(n_elems / 4, kThreads);
  if (elem_bytes == 2)
    rs_finalize_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(n_elems, nodes, node, own, wire,
                                                                wire_stride, scale, out);
  else
    rs_finalize_kernel<float><<<grid, kThreads, 0, s>>>(n_elems, nodes, node, own, wire, wire_stride,
                                                        scale, out);
  return cudaGetLastError();
}

cudaError_t launch_adam(std::int64_t n, const AdamParams& p, float* master, float* m, float* v,
                        const float* grad, void* param, int param_elem_bytes, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = grid_for(n / 4 + 1, kThreads);
  if (param_elem_bytes == 2)
    adam_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(n, p, master, m, v, grad, param);
  else
    adam_kernel<float><<<grid, kThreads, 0, s>>>(n, p, master, m, v, grad, param);
  return cudaGetLastError();
}

cudaError_t launch_adam_grad(std::int64_t chunks, const GradSegs& segs, const AdamParams& p, float scale,
                             float* master, float* m, float* v, void* param, int param_elem_bytes, float* keep_grad,
                             cudaStream_t s, int max_blocks) {
  if (chunks <= 0) return cudaSuccess;
  if (segs.n < 0 || segs.n > kMaxGradSegs) return cudaErrorInvalidValue;
  const std::int64_t V = kChunkBytes / param_elem_bytes;
  AdamCover cv{};
  std::int64_t at = 0;  // chunks covered so far
  auto push = [&](std::int64_t c0, std::int64_t nc, const void* src) {
    if (nc <= 0) return;
    cv.elem0[cv.n] = c0 * V;
    cv.count[cv.n] = nc * V;
    cv.src[cv.n] = src;
    ++cv.n;
  };
  for (int i = 0; i < segs.n; ++i) {
    if (reinterpret_cast<std::uintptr_t>(segs.src[i]) % 16) return cudaErrorMisalignedAddress;
    if (segs.dst_chunk[i] < at || segs.dst_chunk[i] + segs.nchunks[i] > chunks) return cudaErrorInvalidValue;
    push(at, segs.dst_chunk[i] - at, nullptr);  // gap: zero gradient
    push(segs.dst_chunk[i], segs.nchunks[i], segs.src[i]);
    at = segs.dst_chunk[i] + segs.nchunks[i];
  }
  push(at, chunks - at, nullptr);
  // grid shares proportional to segment size (at least one block each)
  int total = grid_for(chunks * V / 4, kThreads * 2);
  if (max_blocks > 0) total = std::max(std::min(total, max_blocks - cv.n), 1);  // each segment adds >= 1 block
  int b = 0;
  for (int i = 0; i < cv.n; ++i) {
    cv.block0[i] = b;
    const std::int64_t share = (cv.count[i] * total + chunks * V - 1) / (chunks * V);
    b += static_cast<int>(std::max<std::int64_t>(1, share));
  }
  cv.block0[cv.n] = b;
  if (param_elem_bytes == 2)
    adam_grad_kernel<__nv_bfloat16><<<b, kThreads, 0, s>>>(cv, p, scale, master, m, v, param, keep_grad);
  else
    adam_grad_kernel<float><<<b, kThreads, 0, s>>>(cv, p, scale, master, m, v, param, keep_grad);
  return cudaGetLastError();
}

cudaError_t launch_init_natural(std::int64_t n_elems, int elem_bytes, std::uint64_t seed, int layer,
                                const InitRange* ranges_dev, int num_ranges, void* natural,
                                cudaStream_t s) {
  if (n_elems <= 0) return cudaSuccess;
  const int grid = grid_for(n_elems, kThreads);
  if (elem_bytes == 2)
    init_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(n_elems, seed, layer, ranges_dev, num_ranges, natural);
  else
    init_kernel<float><<<grid, kThreads, 0, s>>>(n_elems, seed, layer, ranges_dev, num_ranges, natural);
  return cudaGetLastError();
}

cudaError_t launch_widen(std::int64_t n, const void* src, int elem_bytes, float* dst, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = grid_for(n, kThreads);
  if (elem_bytes == 2)
    widen_kernel<__nv_bfloat16><<<grid, kThreads, 0, s>>>(n, src, dst);
  else
    widen_kernel<float><<<grid, kThreads, 0, s>>>(n, src, dst);
  return cudaGetLastError();
}

cudaError_t launch_copy_rows(std::int64_t rows, std::int64_t row_bytes, const void* src, std::int64_t src_pitch,
                             void* dst, std::int64_t dst_pitch, cudaStream_t s) {
  if (row_bytes % kChunkBytes || src_pitch % kChunkBytes || dst_pitch % kChunkBytes || rows < 0 ||
      reinterpret_cast<std::uintptr_t>(src) % 16 || reinterpret_cast<std::uintptr_t>(dst) % 16)
    return cudaErrorInvalidValue;
  const std::int64_t n = rows * (row_bytes / kChunkBytes);
  if (n == 0) return cudaSuccess;
  copy_rows_kernel<<<grid_for(n, kThreads * 2), kThreads, 0, s>>>(
      rows, static_cast<int>(row_bytes / kChunkBytes), static_cast<const uint4*>(src), src_pitch / kChunkBytes,
      static_cast<uint4*>(dst), dst_pitch / kChunkBytes);
  return cudaGetLastError();
}

cudaError_t launch_copy_segments(int n, const void* const* src, void* const* dst, const std::int64_t* bytes,
                                 cudaStream_t s) {
  for (int base = 0; base < n; base += kMaxCopySegs) {
    CopySegs c{};
    const int m = std::min(kMaxCopySegs, n - base);
    std::int64_t most = 0;
    for (int k = 0; k < m; ++k) {
      const auto sp = reinterpret_cast<std::uintptr_t>(src[base + k]);
      const auto dp = reinterpret_cast<std::uintptr_t>(dst[base + k]);
      if (bytes[base + k] % kChunkBytes || sp % 16 || dp % 16 || bytes[base + k] < 0) return cudaErrorInvalidValue;
      c.src[k] = static_cast<const uint4*>(src[base + k]);
      c.dst[k] = static_cast<uint4*>(dst[base + k]);
      c.chunks[k] = bytes[base + k] / kChunkBytes;
      most = std::max(most, c.chunks[k]);
    }
    if (most == 0) continue;
    const dim3 grid(static_cast<unsigned>(std::max<std::int64_t>(
                        1, std::min<std::int64_t>((most + 2 * kThreads - 1) / (2 * kThreads), sm_count()))),
                    static_cast<unsigned>(m));
    seg_copy_kernel<<<grid, kThreads, 0, s>>>(c);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_copy(const void* src, void* dst, std::int64_t bytes, cudaStream_t s) {
  if (use_tma_copy() && bytes % kChunkBytes == 0 && reinterpret_cast<std::uintptr_t>(src) % 16 == 0 &&
      reinterpret_cast<std::uintptr_t>(dst) % 16 == 0) {
    BulkSegs segs{};
    segs.src[0] = static_cast<const unsigned char*>(src);
    segs.dst[0] = static_cast<unsigned char*>(dst);
    segs.bytes[0] = bytes;
    segs.n = 1;
    return launch_bulk(segs, s);
  }
  const std::int64_t n = bytes / kChunkBytes;
  if (n > 0)
    copy_kernel<<<grid_for(n, kThreads * kUnroll), kThreads, 0, s>>>(static_cast<const uint4*>(src),
                                                                      static_cast<uint4*>(dst), n);
  const std::int64_t tail = bytes - n * kChunkBytes;
  if (tail > 0)
    return cudaMemcpyAsync(static_cast<char*>(dst) + n * kChunkBytes,
                           static_cast<const char*>(src) + n * kChunkBytes, tail,
                           cudaMemcpyDeviceToDevice, s);
  return cudaGetLastError();
}

}  // namespace fcdp
