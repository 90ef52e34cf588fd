// LayerNorm kernels of the driving model (bf16 rows, h a multiple of 256, h <= 2048).
// Not part of the parameter-movement path; see model_kernels.cu.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fcdp {

bool layernorm_supported(int h);
cudaError_t launch_layernorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* w, const void* b,
                                 void* y, float* mean, float* rstd, cudaStream_t s);
// part: 2 * splits * h floats of scratch (column partials of dgamma, dbeta)
cudaError_t launch_layernorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                                 const float* mean, const float* rstd, void* dx, void* dw, void* db, float* part,
                                 int splits, cudaStream_t s);

}  // namespace fcdp
