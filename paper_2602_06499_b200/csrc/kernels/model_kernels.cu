// LayerNorm forward / backward for the driving model (GPT-2 blocks, bf16).
//
// Not part of the parameter-movement path: the driving model is its consumer.
// PyTorch's LayerNorm kernels ran at ~2 TB/s forward and the backward's
// gamma/beta column reduction dominated its 94 us per [8192 x 2048] call
// (profiles/r02_model_profile.txt), ~6 ms of a 79 ms GPT-2 1.3B step.  These
// are plain bandwidth kernels:
//   fwd     one warp per row, the row in registers (16-byte vectors), fp32
//           two-pass mean / variance, y and the per-row (mean, rstd) written
//   bwd dx  one warp per row: dx = rstd * (g - mean(g) - xhat * mean(g*xhat)),
//           g = dy * gamma, xhat recomputed from (mean, rstd)
//   bwd dw  column partials of dgamma = sum dy*xhat and dbeta = sum dy over
//           row blocks (fixed split), then a fixed-order sum of the partials:
//           deterministic, no atomics.
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels/model_kernels.hpp"

namespace fcdp {
namespace {

constexpr int kWarps = 4;          // rows per block (fwd, bwd dx): more resident blocks at ~150 registers
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return q;
}

// kV = 16-byte vectors per lane (h = 256 * kV)
template <int kV>
__global__ void __launch_bounds__(kWarps * 32) ln_fwd_kernel(std::int64_t rows, int h, float eps,
                                                             const uint4* __restrict__ x, const uint4* __restrict__ w,
                                                             const uint4* __restrict__ b, uint4* __restrict__ y,
                                                             float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  const int lane = threadIdx.x & 31;
  const std::int64_t row = static_cast<std::int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const std::int64_t base = row * (h / 8);
  float v[kV][8];
#pragma unroll
  for (int k = 0; k < kV; ++k) unpack8(__ldcs(x + base + k * 32 + lane), v[k]);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) s += v[k][e];
  const float mean = warp_sum(s) / h;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float d = v[k][e] - mean;
      q += d * d;
    }
  const float rstd = rsqrtf(warp_sum(q) / h + eps);
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float wf[8], bf[8], o[8];
    unpack8(__ldg(w + k * 32 + lane), wf);
    unpack8(__ldg(b + k * 32 + lane), bf);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = (v[k][e] - mean) * rstd * wf[e] + bf[e];
    __stcs(y + base + k * 32 + lane, pack8(o));
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

template <int kV>
__global__ void __launch_bounds__(kWarps * 32) ln_bwd_dx_kernel(std::int64_t rows, int h, const uint4* __restrict__ dy,
                                                                const uint4* __restrict__ x,
                                                                const uint4* __restrict__ w,
                                                                const float* __restrict__ mean_in,
                                                                const float* __restrict__ rstd_in,
                                                                uint4* __restrict__ dx) {
  const int lane = threadIdx.x & 31;
  const std::int64_t row = static_cast<std::int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const std::int64_t base = row * (h / 8);
  const float mean = __ldg(mean_in + row), rstd = __ldg(rstd_in + row);
  float xh[kV][8], g[kV][8];
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float xf[8], df[8], wf[8];
    unpack8(__ldg(x + base + k * 32 + lane), xf);
    unpack8(__ldcs(dy + base + k * 32 + lane), df);
    unpack8(__ldg(w + k * 32 + lane), wf);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      xh[k][e] = (xf[e] - mean) * rstd;
      g[k][e] = df[e] * wf[e];
    }
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      s1 += g[k][e];
      s2 += g[k][e] * xh[k][e];
    }
  const float c2 = warp_sum(s1) / h, c1 = warp_sum(s2) / h;
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = rstd * (g[k][e] - c2 - xh[k][e] * c1);
    __stcs(dx + base + k * 32 + lane, pack8(o));
  }
}

// dgamma / dbeta partials: block (column group of 256 columns, row split r);
// each thread owns 8 columns (one 16-byte vector), a warp covers the block's
// 256 columns of one row (512 contiguous bytes), and the block's 8 warps walk
// the split's rows 8 apart; the 8 row-lane sums are added in fixed order.
constexpr int kColThreads = 32;  // column vectors per block = 256 columns
constexpr int kRowLanes = 8;     // rows processed concurrently per block
__global__ void __launch_bounds__(kColThreads * kRowLanes) ln_bwd_dw_partial_kernel(
    std::int64_t rows, int h, int splits, const uint4* __restrict__ dy, const uint4* __restrict__ x,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, float* __restrict__ part_w,
    float* __restrict__ part_b) {
  __shared__ float red_w[kRowLanes][kColThreads * 8 + 1];
  __shared__ float red_b[kRowLanes][kColThreads * 8 + 1];
  const int cv = blockIdx.x * kColThreads + (threadIdx.x % kColThreads);  // column vector index
  const int rl = threadIdx.x / kColThreads;
  const int split = blockIdx.y;
  const std::int64_t per = (rows + splits - 1) / splits;
  const std::int64_t r0 = split * per, r1 = min(rows, r0 + per);
  float aw[8], ab[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) aw[e] = ab[e] = 0.f;
  const bool valid = cv < h / 8;
  if (valid)
    for (std::int64_t r = r0 + rl; r < r1; r += kRowLanes) {
      float xf[8], df[8];
      unpack8(__ldg(x + r * (h / 8) + cv), xf);
      unpack8(__ldg(dy + r * (h / 8) + cv), df);
      const float mean = __ldg(mean_in + r), rstd = __ldg(rstd_in + r);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        aw[e] += df[e] * ((xf[e] - mean) * rstd);
        ab[e] += df[e];
      }
    }
  const int c = threadIdx.x % kColThreads;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    red_w[rl][c * 8 + e] = aw[e];
    red_b[rl][c * 8 + e] = ab[e];
  }
  __syncthreads();
  // fixed-order sum over the row lanes, one column per thread
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    float sw = 0.f, sb = 0.f;
#pragma unroll
    for (int l = 0; l < kRowLanes; ++l) {
      sw += red_w[l][col];
      sb += red_b[l][col];
    }
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol < h) {
      part_w[static_cast<std::int64_t>(split) * h + gcol] = sw;
      part_b[static_cast<std::int64_t>(split) * h + gcol] = sb;
    }
  }
}

__global__ void ln_bwd_dw_final_kernel(int h, int splits, const float* __restrict__ part_w,
                                       const float* __restrict__ part_b, __nv_bfloat16* __restrict__ dw,
                                       __nv_bfloat16* __restrict__ db) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= h) return;
  float sw = 0.f, sb = 0.f;
  for (int s = 0; s < splits; ++s) {  // fixed order: deterministic
    sw += part_w[static_cast<std::int64_t>(s) * h + col];
    sb += part_b[static_cast<std::int64_t>(s) * h + col];
  }
  dw[col] = __float2bfloat16_rn(sw);
  db[col] = __float2bfloat16_rn(sb);
}

}  // namespace

// the row lives in registers: 8 x h/256 floats per lane (h <= 2048)
bool layernorm_supported(int h) { return h % 256 == 0 && h / 256 >= 1 && h / 256 <= 8; }

cudaError_t launch_layernorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* w, const void* b,
                                 void* y, float* mean, float* rstd, cudaStream_t s) {
  if (!layernorm_supported(h)) return cudaErrorInvalidValue;
  const int grid = static_cast<int>((rows + kWarps - 1) / kWarps);
  auto X = static_cast<const uint4*>(x);
  auto W = static_cast<const uint4*>(w);
  auto B = static_cast<const uint4*>(b);
  auto Y = static_cast<uint4*>(y);
  switch (h / 256) {
#define FCDP_LN_FWD(V) \
  case V: ln_fwd_kernel<V><<<grid, kWarps * 32, 0, s>>>(rows, h, eps, X, W, B, Y, mean, rstd); break;
    FCDP_LN_FWD(1) FCDP_LN_FWD(2) FCDP_LN_FWD(3) FCDP_LN_FWD(4) FCDP_LN_FWD(5) FCDP_LN_FWD(6) FCDP_LN_FWD(7)
    FCDP_LN_FWD(8)
#undef FCDP_LN_FWD
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_layernorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                                 const float* mean, const float* rstd, void* dx, void* dw, void* db, float* part,
                                 int splits, cudaStream_t s) {
  if (!layernorm_supported(h) || splits < 1) return cudaErrorInvalidValue;
  const int grid = static_cast<int>((rows + kWarps - 1) / kWarps);
  auto DY = static_cast<const uint4*>(dy);
  auto X = static_cast<const uint4*>(x);
  auto W = static_cast<const uint4*>(w);
  auto DX = static_cast<uint4*>(dx);
  switch (h / 256) {
#define FCDP_LN_BWD(V) \
  case V: ln_bwd_dx_kernel<V><<<grid, kWarps * 32, 0, s>>>(rows, h, DY, X, W, mean, rstd, DX); break;
    FCDP_LN_BWD(1) FCDP_LN_BWD(2) FCDP_LN_BWD(3) FCDP_LN_BWD(4) FCDP_LN_BWD(5) FCDP_LN_BWD(6) FCDP_LN_BWD(7)
    FCDP_LN_BWD(8)
#undef FCDP_LN_BWD
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (dw && db) {
    const dim3 g2((h / 8 + kColThreads - 1) / kColThreads, splits);
    ln_bwd_dw_partial_kernel<<<g2, kColThreads * kRowLanes, 0, s>>>(rows, h, splits, DY, X, mean, rstd, part,
                                                                     part + static_cast<std::int64_t>(splits) * h);
    ln_bwd_dw_final_kernel<<<(h + 255) / 256, 256, 0, s>>>(h, splits, part,
                                                           part + static_cast<std::int64_t>(splits) * h,
                                                           static_cast<__nv_bfloat16*>(dw),
                                                           static_cast<__nv_bfloat16*>(db));
  }
  return cudaGetLastError();
}

}  // namespace fcdp
