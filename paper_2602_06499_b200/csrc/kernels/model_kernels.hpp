// Kernels of the driving model (bf16): LayerNorm (h a multiple of 256, h <= 2048),
// bias gradients, bias + GELU, fused cross-entropy.
// Not part of the parameter-movement path; see model_kernels.cu.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fcdp {

bool layernorm_supported(int h);
// r / s_out (both or neither): normalise the residual sum s = x + r (bf16), written to s_out
cudaError_t launch_layernorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* w, const void* b,
                                 void* y, float* mean, float* rstd, cudaStream_t s, const void* r = nullptr,
                                 void* s_out = nullptr);
// part: 2 * splits * h floats of scratch (column partials of dgamma, dbeta)
// dres (nullable): gradient reaching the residual sum from downstream, added to dx
cudaError_t launch_layernorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                                 const float* mean, const float* rstd, void* dx, void* dw, void* db, float* part,
                                 int splits, cudaStream_t s, const void* dres = nullptr);

// bias gradient: out[c] = sum_r dy[r, c] (cols a multiple of 8); part: splits * cols floats
int colsum_splits(std::int64_t rows, int cols);
cudaError_t launch_colsum(std::int64_t rows, int cols, const void* dy, void* out, float* part, int splits,
                          cudaStream_t s);
// y = gelu_tanh(h + b) and its backward dh = dy * gelu'(h + b), db = sum_r dh
cudaError_t launch_bias_gelu_fwd(std::int64_t rows, int cols, const void* h, const void* b, void* y, cudaStream_t s);
cudaError_t launch_bias_gelu_bwd(std::int64_t rows, int cols, const void* dy, const void* h, const void* b, void* dh,
                                 void* db, float* part, int splits, cudaStream_t s);
// cross-entropy over bf16 logits rows (label < 0: ignored): loss[r], lse[r]; backward
// dlogits = (softmax - onehot) * scale[0] (a separate buffer; scale is a device scalar)
cudaError_t launch_xent_fwd(std::int64_t rows, int V, const void* logits, const std::int64_t* labels, float* loss,
                            float* lse, cudaStream_t s);
cudaError_t launch_xent_bwd(std::int64_t rows, int V, const void* logits, const std::int64_t* labels,
                            const float* lse, const float* scale, void* dlogits, cudaStream_t s);

// RoPE of x [batch, seq, heads, dim] with fp32 cos / sin tables [seq, dim / 2]; inverse: the backward.
// x_stride / y_stride: elements between consecutive tokens (>= heads * dim, multiples of 8).
cudaError_t launch_rope(std::int64_t batch, int seq, int heads, int dim, const void* x, std::int64_t x_stride,
                        const float* cs, const float* sn, bool inverse, void* y, std::int64_t y_stride,
                        cudaStream_t s);
// SwiGLU y = silu(g) * u, [rows x f]; strides in elements (multiples of 8)
cudaError_t launch_swiglu_fwd(std::int64_t rows, int f, const void* g, std::int64_t g_stride, const void* u,
                              std::int64_t u_stride, void* y, cudaStream_t s);
cudaError_t launch_swiglu_bwd(std::int64_t rows, int f, const void* dy, const void* g, std::int64_t g_stride,
                              const void* u, std::int64_t u_stride, void* dg, std::int64_t dg_stride, void* du,
                              std::int64_t du_stride, cudaStream_t s);

// Llama RMSNorm (h a multiple of 1024, <= 8192): y = x * rstd * w (r / s_out: residual sum first)
bool rmsnorm_supported(int h);
cudaError_t launch_rmsnorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* r, const void* w,
                               void* s_out, void* y, float* rstd, cudaStream_t s);
cudaError_t launch_rmsnorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                               const float* rstd, const void* dres, void* dx, void* dw, float* part, int splits,
                               cudaStream_t s);

}  // namespace fcdp
