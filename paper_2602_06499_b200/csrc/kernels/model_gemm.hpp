// cuBLASLt GEMMs of the driving model's GPT-2 MLP with fused epilogues (see model_gemm.cpp).
#pragma once

#include <cstdint>
#include <string>

#include <cuda_runtime.h>

namespace fcdp {

bool mlp_gemm_available(std::string* why);
// act = gelu_tanh(x W^T + b), aux = x W^T + b; x [rows x in], W [out x in], all bf16 row-major
cudaError_t launch_fc_gelu_fwd(std::int64_t rows, std::int64_t in, std::int64_t out, const void* x, const void* w,
                               const void* b, void* act, void* aux, cudaStream_t s, std::string* err);
// dpre = (dy W2) * gelu'(aux), db1 = sum over rows of dpre; dy [rows x hidden], W2 [hidden x ffn], aux [rows x ffn]
cudaError_t launch_fc2_dgrad_dgelu(std::int64_t rows, std::int64_t hidden, std::int64_t ffn, const void* dy,
                                   const void* w2, const void* aux, void* dpre, void* db1, cudaStream_t s,
                                   std::string* err);

}  // namespace fcdp
