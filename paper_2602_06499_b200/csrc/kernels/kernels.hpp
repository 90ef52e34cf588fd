// Launchers for the sm_100a data-plane kernels (kernels.cu).
//
// All kernels are HBM- or link-bound byte movers: 16-byte vector accesses,
// warp-granular mask handling (ballot + popc over 32 chunks), grid sized as a
// multiple of the SM count.  None of them reshapes work into GEMMs.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "common/layout.hpp"

namespace fcdp {

struct SlicePtrs {
  const void* p[kMaxLocal];
};
struct GradPtrs {
  const void* p[kMaxLocal];
};

enum PortionSet : int { kSetAll = 0, kSetTrainable = 1, kSetFrozen = 2 };

// natural -> (t, f) compaction.  Dense layers degrade to a copy.
cudaError_t launch_partition(const Layout& L, const void* natural, void* t, void* f, cudaStream_t s);

// g slice pointers per portion -> natural layer (fused gather + PEFT expand).
cudaError_t launch_expand(const Layout& L, const SlicePtrs& ts, const SlicePtrs& fs, void* natural,
                          int set, cudaStream_t s);

// Intra-node reduce-scatter of the trainable gradient for slice `j`.
// max_blocks > 0 caps the grid (the RS then streams beside concurrently running GEMM CTAs).
cudaError_t launch_rs_slice(const Layout& L, const GradPtrs& grads, int j, int n, float scale,
                            bool final_scale, float* own_out, void* wire_out, cudaStream_t s, int max_blocks = 0);

// Inter-node epilogue: out = scale * sum_m part_m (fixed order).
cudaError_t launch_rs_finalize(std::int64_t n_elems, int nodes, int node, int elem_bytes,
                               const float* own, const void* wire, std::int64_t wire_stride,
                               float scale, float* out, cudaStream_t s);

struct AdamParams {
  float lr, beta1, beta2, eps, weight_decay;
  float bias_c1, bias_c2;  // 1 - beta^t, computed on the host in double
};
cudaError_t launch_adam(std::int64_t n, const AdamParams& p, float* master, float* m, float* v,
                        const float* grad, void* param, int param_elem_bytes, cudaStream_t s);

// G = 1 fused reduce-scatter (widen + scale) + AdamW of a dense trainable layer,
// reading the gradient in the parameter dtype from up to kMaxGradSegs
// segments (16-byte aligned; chunk offsets within the layer; chunks no segment
// covers have gradient 0).  keep_grad (nullable) receives the fp32 gradient.
inline constexpr int kMaxGradSegs = 24;
struct GradSegs {
  int n = 0;
  std::int64_t dst_chunk[kMaxGradSegs];
  std::int64_t nchunks[kMaxGradSegs];
  const void* src[kMaxGradSegs];
};
// max_blocks > 0 caps the grid (e.g. one CTA per SM, so each SM keeps room for
// a concurrently running GEMM CTA beside it).
cudaError_t launch_adam_grad(std::int64_t chunks, const GradSegs& segs, const AdamParams& p, float scale,
                             float* master, float* m, float* v, void* param, int param_elem_bytes, float* keep_grad,
                             cudaStream_t s, int max_blocks = 0);

// Deterministic init of a natural layer; `ranges` is a device array.
struct InitRange {
  std::int64_t begin, end;
  std::int32_t kind;
  float scale;
};
cudaError_t launch_init_natural(std::int64_t n_elems, int elem_bytes, std::uint64_t seed, int layer,
                                const InitRange* ranges_dev, int num_ranges, void* natural,
                                cudaStream_t s);

// Widen a portion shard (param dtype) to fp32 (master init).
cudaError_t launch_widen(std::int64_t n, const void* src, int elem_bytes, float* dst, cudaStream_t s);

// rows x row_bytes strided device copy (pitches in bytes; all multiples of 16).
cudaError_t launch_copy_rows(std::int64_t rows, std::int64_t row_bytes, const void* src, std::int64_t src_pitch,
                             void* dst, std::int64_t dst_pitch, cudaStream_t s);
// Up to any number of 16-byte aligned (src, dst, bytes) copies, kMaxCopySegs per launch.
inline constexpr int kMaxCopySegs = 32;
cudaError_t launch_copy_segments(int n, const void* const* src, void* const* dst, const std::int64_t* bytes,
                                 cudaStream_t s);

// Dense 16B-vector copy kernel (SM-driven; used for peer pulls when CE is off).
cudaError_t launch_copy(const void* src, void* dst, std::int64_t bytes, cudaStream_t s);

int sm_count();

}  // namespace fcdp
