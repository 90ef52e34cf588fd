// Driving-model kernels (GPT-2 blocks and the LM head, bf16): LayerNorm
// forward / backward, bias gradients (column sums), bias + GELU forward and
// GELU backward fused with the bias gradient, the fused cross-entropy, and
// the Llama blocks' rotary embedding and SwiGLU (forward / backward).
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

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
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

// kV = 16-byte vectors per lane (h = 256 * kV).  kRes: the input is the
// residual sum s = x + r (rounded to bf16 as the unfused add would, and
// written out for the residual stream), normalised in the same pass.
template <int kV, bool kRes = false>
__global__ void __launch_bounds__(kWarps * 32) ln_fwd_kernel(std::int64_t rows, int h, float eps,
                                                             const uint4* __restrict__ x, const uint4* __restrict__ w,
                                                             const uint4* __restrict__ b, uint4* __restrict__ y,
                                                             float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                             const uint4* __restrict__ r = nullptr,
                                                             uint4* __restrict__ s_out = nullptr) {
  const int lane = threadIdx.x & 31;
  const std::int64_t row = static_cast<std::int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const std::int64_t base = row * (h / 8);
  float v[kV][8];
#pragma unroll
  for (int k = 0; k < kV; ++k) unpack8(__ldcs(x + base + k * 32 + lane), v[k]);
  if constexpr (kRes) {
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      float rf[8];
      unpack8(__ldcs(r + base + k * 32 + lane), rf);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[k][e] += rf[e];
      const uint4 q = pack8(v[k]);
      __stcs(s_out + base + k * 32 + lane, q);
      unpack8(q, v[k]);  // normalise the stored (bf16) sum
    }
  }
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

// kRes: dx += dres (the gradient reaching the residual sum from downstream)
template <int kV, bool kRes = false>
__global__ void __launch_bounds__(kWarps * 32) ln_bwd_dx_kernel(std::int64_t rows, int h, const uint4* __restrict__ dy,
                                                                const uint4* __restrict__ x,
                                                                const uint4* __restrict__ w,
                                                                const float* __restrict__ mean_in,
                                                                const float* __restrict__ rstd_in,
                                                                uint4* __restrict__ dx,
                                                                const uint4* __restrict__ dres = nullptr) {
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
    if constexpr (kRes) {
      float rf[8];
      unpack8(__ldcs(dres + base + k * 32 + lane), rf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += rf[e];
    }
    __stcs(dx + base + k * 32 + lane, pack8(o));
  }
}

// Split-sum epilogue shared by the column reductions: every (column group,
// row split) block writes its partial row, and the LAST block of a column group
// to finish (an arrival counter per group, threadfence-published partials)
// sums that group's partials over the splits in split order and writes the
// result.  The sum order is fixed whatever order the blocks ran in, so the
// result is deterministic, and no second launch is needed.  The counters come
// from a small per-device pool (one slot range per launch) and are reset to 0
// by the block that consumes them.
__device__ __forceinline__ bool last_split_block(unsigned int* counter) {
  __shared__ bool last;
  __threadfence();  // this block's partials are visible before it arrives
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter + blockIdx.x, 1u) == gridDim.y - 1;
  __syncthreads();
  if (last) __threadfence();  // and the others' before it reads them
  return last;
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
    float* __restrict__ part_b, unsigned int* __restrict__ counter, __nv_bfloat16* __restrict__ dw,
    __nv_bfloat16* __restrict__ db) {
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
  if (!last_split_block(counter)) return;
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol >= h) continue;
    float sw = 0.f, sb = 0.f;
    for (int k = 0; k < splits; ++k) {  // fixed order: deterministic
      sw += __ldcg(part_w + static_cast<std::int64_t>(k) * h + gcol);
      sb += __ldcg(part_b + static_cast<std::int64_t>(k) * h + gcol);
    }
    dw[gcol] = __float2bfloat16_rn(sw);
    db[gcol] = __float2bfloat16_rn(sb);
  }
  if (threadIdx.x == 0) counter[blockIdx.x] = 0;
}

// ------------------------------------------------- column sums (bias grads)
// out[c] = sum_r dy[r, c] for a bf16 [rows x cols] matrix (the bias gradient
// of a linear layer).  Same two-stage, fixed-order scheme as the LayerNorm
// dgamma/dbeta: block (256-column group, row split), 32 column vectors x 8 row
// lanes, kRowUnroll rows in flight per lane; the split partials are summed in
// split order.  kGelu: the tensor summed is the GELU backward of the MLP's
// first linear, computed here and written out as well:
//   pre = h + b (fp32), dh = dy * gelu'(pre) rounded to bf16, sum the rounded dh
// (torch's gelu_backward + bias-grad arithmetic, tanh approximation).
constexpr int kRowUnroll = 4;
constexpr float kGeluBeta = 0.7978845608028654f;  // sqrt(2 / pi)
constexpr float kGeluKappa = 0.044715f;

// tanh on the SFU: one tanh.approx.f32 (max relative error 2^-10.99, under a
// quarter of a bf16 ulp of the outputs).  libm tanhf made these kernels
// issue-bound (2.9 TB/s), and exp + rcp still cost two SFU ops per element.
__device__ __forceinline__ float fast_tanh(float u) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return t;
}

__device__ __forceinline__ float gelu_tanh(float x) {
  const float inner = kGeluBeta * (x + kGeluKappa * x * x * x);
  return 0.5f * x * (1.0f + fast_tanh(inner));
}

__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float x2 = x * x;
  const float t = fast_tanh(kGeluBeta * (x + kGeluKappa * x2 * x));
  const float left = 0.5f * x, right = 1.0f + t;
  return 0.5f * right + left * (1.0f - t * t) * kGeluBeta * (1.0f + 3.0f * kGeluKappa * x2);
}

template <bool kGelu>
__global__ void __launch_bounds__(kColThreads * kRowLanes) colsum_partial_kernel(
    std::int64_t rows, int cols, int splits, const uint4* __restrict__ dy, const uint4* __restrict__ h,
    const uint4* __restrict__ bias, uint4* __restrict__ dh, float* __restrict__ part,
    unsigned int* __restrict__ counter, __nv_bfloat16* __restrict__ out) {
  __shared__ float red[kRowLanes][kColThreads * 8 + 1];
  const int cv = blockIdx.x * kColThreads + (threadIdx.x % kColThreads);
  const int rl = threadIdx.x / kColThreads;
  const int vpr = cols / 8;  // 16-byte vectors per row
  const std::int64_t per = (rows + splits - 1) / splits;
  const std::int64_t r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  float bf[8];
  if (kGelu && cv < vpr) unpack8(__ldg(bias + cv), bf);
  if (cv < vpr) {
    std::int64_t r = r0 + rl;
    for (; r + (kRowUnroll - 1) * kRowLanes < r1; r += kRowUnroll * kRowLanes) {
      uint4 q[kRowUnroll], hq[kRowUnroll];
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        const std::int64_t i = (r + u * kRowLanes) * vpr + cv;
        q[u] = __ldcs(dy + i);
        if (kGelu) hq[u] = __ldcs(h + i);
      }
#pragma unroll
      for (int u = 0; u < kRowUnroll; ++u) {
        float d[8];
        unpack8(q[u], d);
        if (kGelu) {
          float hf[8];
          unpack8(hq[u], hf);
#pragma unroll
          for (int e = 0; e < 8; ++e) d[e] *= gelu_tanh_grad(hf[e] + bf[e]);
          const uint4 o = pack8(d);
          __stcs(dh + (r + u * kRowLanes) * vpr + cv, o);
          unpack8(o, d);  // sum what was stored (bf16-rounded), like gelu_backward then sum
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += d[e];
      }
    }
    for (; r < r1; r += kRowLanes) {
      const std::int64_t i = r * vpr + cv;
      float d[8];
      unpack8(__ldcs(dy + i), d);
      if (kGelu) {
        float hf[8];
        unpack8(__ldcs(h + i), hf);
#pragma unroll
        for (int e = 0; e < 8; ++e) d[e] *= gelu_tanh_grad(hf[e] + bf[e]);
        const uint4 o = pack8(d);
        __stcs(dh + i, o);
        unpack8(o, d);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += d[e];
    }
  }
  const int c = threadIdx.x % kColThreads;
#pragma unroll
  for (int e = 0; e < 8; ++e) red[rl][c * 8 + e] = acc[e];
  __syncthreads();
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    float sacc = 0.f;
#pragma unroll
    for (int l = 0; l < kRowLanes; ++l) sacc += red[l][col];
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol < cols) part[static_cast<std::int64_t>(blockIdx.y) * cols + gcol] = sacc;
  }
  if (!last_split_block(counter)) return;
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol >= cols) continue;
    float sacc = 0.f;
    for (int k = 0; k < splits; ++k) sacc += __ldcg(part + static_cast<std::int64_t>(k) * cols + gcol);  // fixed order
    out[gcol] = __float2bfloat16_rn(sacc);
  }
  if (threadIdx.x == 0) counter[blockIdx.x] = 0;
}

// RMSNorm dgamma = sum_r dy * x * rstd: column partials + last-block split sum.
__global__ void __launch_bounds__(kColThreads * kRowLanes) rms_bwd_dw_partial_kernel(
    std::int64_t rows, int h, int splits, const uint4* __restrict__ dy, const uint4* __restrict__ x,
    const float* __restrict__ rstd_in, float* __restrict__ part_w, unsigned int* __restrict__ counter,
    __nv_bfloat16* __restrict__ dw) {
  __shared__ float red_w[kRowLanes][kColThreads * 8 + 1];
  const int cv = blockIdx.x * kColThreads + (threadIdx.x % kColThreads);
  const int rl = threadIdx.x / kColThreads;
  const std::int64_t per = (rows + splits - 1) / splits;
  const std::int64_t r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float aw[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) aw[e] = 0.f;
  if (cv < h / 8)
    for (std::int64_t r = r0 + rl; r < r1; r += kRowLanes) {
      float xf[8], df[8];
      unpack8(__ldg(x + r * (h / 8) + cv), xf);
      unpack8(__ldg(dy + r * (h / 8) + cv), df);
      const float rstd = __ldg(rstd_in + r);
#pragma unroll
      for (int e = 0; e < 8; ++e) aw[e] += df[e] * (xf[e] * rstd);
    }
  const int c = threadIdx.x % kColThreads;
#pragma unroll
  for (int e = 0; e < 8; ++e) red_w[rl][c * 8 + e] = aw[e];
  __syncthreads();
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    float sw = 0.f;
#pragma unroll
    for (int l = 0; l < kRowLanes; ++l) sw += red_w[l][col];
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol < h) part_w[static_cast<std::int64_t>(blockIdx.y) * h + gcol] = sw;
  }
  if (!last_split_block(counter)) return;
  for (int col = threadIdx.x; col < kColThreads * 8; col += blockDim.x) {
    const int gcol = blockIdx.x * kColThreads * 8 + col;
    if (gcol >= h) continue;
    float sw = 0.f;
    for (int k = 0; k < splits; ++k) sw += __ldcg(part_w + static_cast<std::int64_t>(k) * h + gcol);
    dw[gcol] = __float2bfloat16_rn(sw);
  }
  if (threadIdx.x == 0) counter[blockIdx.x] = 0;
}

// y = gelu(h + b): the MLP's first linear runs without its bias epilogue and the
// bias add is fused here (one read of h, one write of y).  A thread owns one
// column vector (its bias loaded once) and walks rows gridDim.y apart, 4 in
// flight: no per-element index division.
constexpr int kGeluRows = 4;
__global__ void __launch_bounds__(256) bias_gelu_fwd_kernel(std::int64_t rows, int vpr,
                                                            const uint4* __restrict__ h,
                                                            const uint4* __restrict__ bias,
                                                            uint4* __restrict__ y) {
  const int cv = blockIdx.x * blockDim.x + threadIdx.x;
  if (cv >= vpr) return;
  float bf[8];
  unpack8(__ldg(bias + cv), bf);
  std::int64_t r = blockIdx.y;
  const std::int64_t step = gridDim.y;
  for (; r + (kGeluRows - 1) * step < rows; r += kGeluRows * step) {
    uint4 q[kGeluRows];
#pragma unroll
    for (int u = 0; u < kGeluRows; ++u) q[u] = __ldcs(h + (r + u * step) * vpr + cv);
#pragma unroll
    for (int u = 0; u < kGeluRows; ++u) {
      float a[8];
      unpack8(q[u], a);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = gelu_tanh(a[e] + bf[e]);
      __stcs(y + (r + u * step) * vpr + cv, pack8(a));
    }
  }
  for (; r < rows; r += step) {
    float a[8];
    unpack8(__ldcs(h + r * vpr + cv), a);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = gelu_tanh(a[e] + bf[e]);
    __stcs(y + r * vpr + cv, pack8(a));
  }
}

// ------------------------------------------------------------ cross-entropy
// Mean cross-entropy over rows of bf16 logits [rows x V] (V a multiple of 8),
// fp32 arithmetic.  One block per row, kXentThreads threads:
//   fwd  one read of the row: per-thread online (max, sum exp) over 16-byte
//        vectors, merged across the block; lse[row] and loss[row] = lse - x[label]
//   bwd  one read + one write: dx = (exp(x - lse) - [c == label]) * scale[0]
// label < 0 = ignored row (loss 0, gradient 0).  Replaces logits.float() +
// log_softmax + nll (fp32 copies of the whole logits matrix) of the head.
constexpr int kXentThreads = 512;

__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * __expf(m - mn) + s2 * __expf(m2 - mn);
  m = mn;
}

__global__ void __launch_bounds__(kXentThreads) xent_fwd_kernel(int vpr, const uint4* __restrict__ x,
                                                                const std::int64_t* __restrict__ labels,
                                                                float* __restrict__ loss, float* __restrict__ lse) {
  __shared__ float sm[kXentThreads / 32], ss[kXentThreads / 32];
  const std::int64_t row = blockIdx.x;
  const uint4* xr = x + row * vpr;
  float m = -INFINITY, s = 0.f;
  int i = threadIdx.x;
  for (; i + kXentThreads < vpr; i += 2 * kXentThreads) {
    float a[8], b[8];
    unpack8(__ldcs(xr + i), a);
    unpack8(__ldcs(xr + i + kXentThreads), b);
    float lm = a[0];
#pragma unroll
    for (int e = 0; e < 8; ++e) lm = fmaxf(lm, fmaxf(a[e], b[e]));
    const float mn = fmaxf(m, lm);
    float t = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) t += __expf(a[e] - mn) + __expf(b[e] - mn);
    s = s * __expf(m - mn) + t;
    m = mn;
  }
  for (; i < vpr; i += kXentThreads) {
    float a[8];
    unpack8(__ldcs(xr + i), a);
    float lm = a[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, a[e]);
    const float mn = fmaxf(m, lm);
    float t = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) t += __expf(a[e] - mn);
    s = s * __expf(m - mn) + t;
    m = mn;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(kFull, m, o), s2 = __shfl_xor_sync(kFull, s, o);
    ms_merge(m, s, m2, s2);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], Ssum = ss[0];
    for (int w = 1; w < kXentThreads / 32; ++w) ms_merge(M, Ssum, sm[w], ss[w]);  // fixed order
    const float l = M + logf(Ssum);
    lse[row] = l;
    const std::int64_t lab = labels[row];
    const float xl = lab >= 0 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xr)[lab]) : 0.f;
    loss[row] = lab >= 0 ? l - xl : 0.f;
  }
}

__global__ void __launch_bounds__(kXentThreads) xent_bwd_kernel(int vpr, const uint4* __restrict__ x,
                                                                const std::int64_t* __restrict__ labels,
                                                                const float* __restrict__ lse,
                                                                const float* __restrict__ scale,
                                                                uint4* __restrict__ dx) {
  const std::int64_t row = blockIdx.x;
  const std::int64_t lab = labels[row];
  const float l = lse[row], sc = lab >= 0 ? __ldg(scale) : 0.f;
  const uint4* xr = x + row * vpr;
  uint4* dr = dx + row * vpr;
  for (int i = threadIdx.x; i < vpr; i += kXentThreads) {
    float a[8];
    unpack8(__ldcs(xr + i), a);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float p = __expf(a[e] - l);
      a[e] = (p - (static_cast<std::int64_t>(i) * 8 + e == lab ? 1.0f : 0.0f)) * sc;
    }
    __stcs(dr + i, pack8(a));
  }
}

// ------------------------------------------------------------- Llama: RMSNorm
// One block of kRmsThreads threads per row (h = kRmsThreads * 8 * kV, i.e. a
// multiple of 1024: Llama-7B 4096, 13B 5120), the row in registers, fp32
// statistics.  kRes: the input is the residual sum s = x + r (bf16, written
// out) - the Llama block's second norm takes its residual add in the same pass.
// Backward: dx = rstd * (g - xh * mean(g * xh)) with g = dy * w, xh = x * rstd,
// (+ dres: the residual's downstream gradient); dw as column partials summed by
// the last block of each column group (as the LayerNorm's).
constexpr int kRmsThreads = 128;

__device__ __forceinline__ float block_sum_rms(float v, float* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < kRmsThreads / 32; ++i) t += red[i];  // fixed order
  __syncthreads();
  return t;
}

template <int kV, bool kRes>
__global__ void __launch_bounds__(kRmsThreads) rms_fwd_kernel(int h, float eps, const uint4* __restrict__ x,
                                                              const uint4* __restrict__ r, const uint4* __restrict__ w,
                                                              uint4* __restrict__ s_out, uint4* __restrict__ y,
                                                              float* __restrict__ rstd_out) {
  __shared__ float red[kRmsThreads / 32];
  const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * (h / 8);
  float v[kV][8];
#pragma unroll
  for (int k = 0; k < kV; ++k) unpack8(__ldcs(x + base + k * kRmsThreads + threadIdx.x), v[k]);
  if constexpr (kRes) {
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      float rf[8];
      unpack8(__ldcs(r + base + k * kRmsThreads + threadIdx.x), rf);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[k][e] += rf[e];
      const uint4 q = pack8(v[k]);
      __stcs(s_out + base + k * kRmsThreads + threadIdx.x, q);
      unpack8(q, v[k]);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k)
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += v[k][e] * v[k][e];
  const float rstd = rsqrtf(block_sum_rms(ss, red) / h + eps);
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float wf[8], o[8];
    unpack8(__ldg(w + k * kRmsThreads + threadIdx.x), wf);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = v[k][e] * rstd * wf[e];
    __stcs(y + base + k * kRmsThreads + threadIdx.x, pack8(o));
  }
  if (threadIdx.x == 0) rstd_out[blockIdx.x] = rstd;
}

template <int kV, bool kRes>
__global__ void __launch_bounds__(kRmsThreads) rms_bwd_dx_kernel(int h, const uint4* __restrict__ dy,
                                                                 const uint4* __restrict__ x,
                                                                 const uint4* __restrict__ w,
                                                                 const float* __restrict__ rstd_in,
                                                                 const uint4* __restrict__ dres,
                                                                 uint4* __restrict__ dx) {
  __shared__ float red[kRmsThreads / 32];
  const std::int64_t base = static_cast<std::int64_t>(blockIdx.x) * (h / 8);
  const float rstd = __ldg(rstd_in + blockIdx.x);
  float xh[kV][8], g[kV][8];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float xf[8], df[8], wf[8];
    unpack8(__ldg(x + base + k * kRmsThreads + threadIdx.x), xf);
    unpack8(__ldcs(dy + base + k * kRmsThreads + threadIdx.x), df);
    unpack8(__ldg(w + k * kRmsThreads + threadIdx.x), wf);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      xh[k][e] = xf[e] * rstd;
      g[k][e] = df[e] * wf[e];
      s += g[k][e] * xh[k][e];
    }
  }
  const float c = block_sum_rms(s, red) / h;
#pragma unroll
  for (int k = 0; k < kV; ++k) {
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = rstd * (g[k][e] - xh[k][e] * c);
    if constexpr (kRes) {
      float rf[8];
      unpack8(__ldcs(dres + base + k * kRmsThreads + threadIdx.x), rf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] += rf[e];
    }
    __stcs(dx + base + k * kRmsThreads + threadIdx.x, pack8(o));
  }
}

// --------------------------------------------------------- Llama: RoPE, SwiGLU
// Rotary embedding of x [batch, seq, heads, dim] (bf16, contiguous): pairs
// (2i, 2i+1) rotated by pos * base^(-2i/dim), angles from fp32 cos / sin tables
// [seq, dim/2]; sign = -1 applies the inverse rotation (the backward).  One
// 16-byte vector (4 pairs) per thread, fp32 arithmetic, one rounding.
// xs / ys: token strides of x and y in 16-byte vectors (heads * dim / 8 when
// contiguous; larger for one third of a joint [tokens x 3h] q|k|v projection).
// Grid: x over a token's vectors, y over tokens (a grid-stride loop past 65535):
// no per-element 64-bit index division (which made the flat version issue-bound).
__global__ void __launch_bounds__(256) rope_kernel(std::int64_t tokens, int seq, int vrow, int vdim,
                                                   const uint4* __restrict__ x, std::int64_t xs,
                                                   const float* __restrict__ cs, const float* __restrict__ sn,
                                                   float sign, uint4* __restrict__ y, std::int64_t ys) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= vrow) return;
  const int d0 = (col % vdim) * 4;  // first rotated pair of this vector
  const int half = vdim * 4;        // dim / 2
  for (std::int64_t tok = blockIdx.y; tok < tokens; tok += gridDim.y) {
    const int pos = static_cast<int>(tok % seq);
    const float4 c = __ldg(reinterpret_cast<const float4*>(cs + static_cast<std::int64_t>(pos) * half + d0));
    const float4 s4 = __ldg(reinterpret_cast<const float4*>(sn + static_cast<std::int64_t>(pos) * half + d0));
    const float cc[4] = {c.x, c.y, c.z, c.w};
    const float ss[4] = {sign * s4.x, sign * s4.y, sign * s4.z, sign * s4.w};
    float v[8], o[8];
    unpack8(__ldcs(x + tok * xs + col), v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o[2 * k] = v[2 * k] * cc[k] - v[2 * k + 1] * ss[k];
      o[2 * k + 1] = v[2 * k] * ss[k] + v[2 * k + 1] * cc[k];
    }
    __stcs(y + tok * ys + col, pack8(o));
  }
}

// SwiGLU y = silu(g) * u over [rows x f] (g, u with their own row strides, in
// 16-byte vectors, so one [rows x 2f] gate|up GEMM output feeds it directly).
__device__ __forceinline__ float sigmoid_fast(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

__global__ void __launch_bounds__(256) swiglu_fwd_kernel(std::int64_t rows, int fv, const uint4* __restrict__ g,
                                                         std::int64_t gs, const uint4* __restrict__ u,
                                                         std::int64_t us, uint4* __restrict__ y) {
  const std::int64_t n = rows * fv;
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += step) {
    const std::int64_t r = i / fv, c = i % fv;
    float a[8], b[8];
    unpack8(__ldcs(g + r * gs + c), a);
    unpack8(__ldcs(u + r * us + c), b);
#pragma unroll
    for (int e = 0; e < 8; ++e) a[e] = a[e] * sigmoid_fast(a[e]) * b[e];
    __stcs(y + i, pack8(a));
  }
}

// dg = dy * u * silu'(g), du = dy * silu(g);  silu'(g) = s (1 + g (1 - s)), s = sigmoid(g)
__global__ void __launch_bounds__(256) swiglu_bwd_kernel(std::int64_t rows, int fv, const uint4* __restrict__ dy,
                                                         const uint4* __restrict__ g, std::int64_t gs,
                                                         const uint4* __restrict__ u, std::int64_t us,
                                                         uint4* __restrict__ dg, std::int64_t dgs,
                                                         uint4* __restrict__ du, std::int64_t dus) {
  const std::int64_t n = rows * fv;
  const std::int64_t step = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += step) {
    const std::int64_t r = i / fv, c = i % fv;
    float d[8], a[8], b[8], og[8], ou[8];
    unpack8(__ldcs(dy + i), d);
    unpack8(__ldcs(g + r * gs + c), a);
    unpack8(__ldcs(u + r * us + c), b);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float sg = sigmoid_fast(a[e]);
      ou[e] = d[e] * a[e] * sg;
      og[e] = d[e] * b[e] * sg * (1.0f + a[e] * (1.0f - sg));
    }
    __stcs(dg + r * dgs + c, pack8(og));
    __stcs(du + r * dus + c, pack8(ou));
  }
}

}  // namespace


namespace {
// Arrival counters of the split-sum epilogue: a zeroed per-device pool, a
// fresh slot range per launch (consumers reset their slots to 0).
constexpr unsigned kCounterPool = 1u << 16;
constexpr unsigned kCounterSlots = 64;  // column groups per launch (cols <= 64 * 256)
unsigned int* counter_slots() {
  static unsigned int* pool[64] = {};
  static std::atomic<unsigned> cursor{0};
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!pool[dev]) {
    unsigned int* p = nullptr;
    if (cudaMalloc(&p, kCounterPool * sizeof(unsigned)) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, kCounterPool * sizeof(unsigned)) != cudaSuccess) return nullptr;  // before any stream uses it
    pool[dev] = p;
  }
  const unsigned slot = (cursor.fetch_add(kCounterSlots) % kCounterPool);
  return pool[dev] + slot;
}
}  // namespace

// the row lives in registers: 8 x h/256 floats per lane (h <= 2048)
bool layernorm_supported(int h) { return h % 256 == 0 && h / 256 >= 1 && h / 256 <= 8; }

cudaError_t launch_layernorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* w, const void* b,
                                 void* y, float* mean, float* rstd, cudaStream_t s, const void* r, void* s_out) {
  if (!layernorm_supported(h) || (r == nullptr) != (s_out == nullptr)) return cudaErrorInvalidValue;
  const int grid = static_cast<int>((rows + kWarps - 1) / kWarps);
  auto X = static_cast<const uint4*>(x);
  auto W = static_cast<const uint4*>(w);
  auto B = static_cast<const uint4*>(b);
  auto Y = static_cast<uint4*>(y);
  auto R = static_cast<const uint4*>(r);
  auto SO = static_cast<uint4*>(s_out);
  switch (h / 256) {
#define FCDP_LN_FWD(V)                                                                                     \
  case V:                                                                                                  \
    if (r)                                                                                                 \
      ln_fwd_kernel<V, true><<<grid, kWarps * 32, 0, s>>>(rows, h, eps, X, W, B, Y, mean, rstd, R, SO);     \
    else                                                                                                   \
      ln_fwd_kernel<V><<<grid, kWarps * 32, 0, s>>>(rows, h, eps, X, W, B, Y, mean, rstd);                  \
    break;
    FCDP_LN_FWD(1) FCDP_LN_FWD(2) FCDP_LN_FWD(3) FCDP_LN_FWD(4) FCDP_LN_FWD(5) FCDP_LN_FWD(6) FCDP_LN_FWD(7)
    FCDP_LN_FWD(8)
#undef FCDP_LN_FWD
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_layernorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                                 const float* mean, const float* rstd, void* dx, void* dw, void* db, float* part,
                                 int splits, cudaStream_t s, const void* dres) {
  if (!layernorm_supported(h) || splits < 1) return cudaErrorInvalidValue;
  const int grid = static_cast<int>((rows + kWarps - 1) / kWarps);
  auto DY = static_cast<const uint4*>(dy);
  auto X = static_cast<const uint4*>(x);
  auto W = static_cast<const uint4*>(w);
  auto DX = static_cast<uint4*>(dx);
  switch (h / 256) {
#define FCDP_LN_BWD(V)                                                                                   \
  case V:                                                                                                \
    if (dres)                                                                                            \
      ln_bwd_dx_kernel<V, true><<<grid, kWarps * 32, 0, s>>>(rows, h, DY, X, W, mean, rstd, DX,           \
                                                             static_cast<const uint4*>(dres));            \
    else                                                                                                 \
      ln_bwd_dx_kernel<V><<<grid, kWarps * 32, 0, s>>>(rows, h, DY, X, W, mean, rstd, DX);                \
    break;
    FCDP_LN_BWD(1) FCDP_LN_BWD(2) FCDP_LN_BWD(3) FCDP_LN_BWD(4) FCDP_LN_BWD(5) FCDP_LN_BWD(6) FCDP_LN_BWD(7)
    FCDP_LN_BWD(8)
#undef FCDP_LN_BWD
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (dw && db) {
    const dim3 g2((h / 8 + kColThreads - 1) / kColThreads, splits);
    unsigned int* ctr = counter_slots();
    if (!ctr || g2.x > kCounterSlots) return cudaErrorInvalidValue;
    ln_bwd_dw_partial_kernel<<<g2, kColThreads * kRowLanes, 0, s>>>(
        rows, h, splits, DY, X, mean, rstd, part, part + static_cast<std::int64_t>(splits) * h, ctr,
        static_cast<__nv_bfloat16*>(dw), static_cast<__nv_bfloat16*>(db));
  }
  return cudaGetLastError();
}

int colsum_splits(std::int64_t rows, int cols) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int groups = (cols / 8 + kColThreads - 1) / kColThreads;
  const std::int64_t want = (4LL * sms + groups - 1) / groups;
  const std::int64_t cap = std::max<std::int64_t>(1, rows / (kRowLanes * kRowUnroll));
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>({want, cap, 1024})));
}

cudaError_t launch_colsum(std::int64_t rows, int cols, const void* dy, void* out, float* part, int splits,
                          cudaStream_t s) {
  if (cols % 8 || splits < 1 || rows < 1) return cudaErrorInvalidValue;
  const dim3 g((cols / 8 + kColThreads - 1) / kColThreads, splits);
  unsigned int* ctr = counter_slots();
  if (!ctr || g.x > kCounterSlots) return cudaErrorInvalidValue;
  colsum_partial_kernel<false><<<g, kColThreads * kRowLanes, 0, s>>>(
      rows, cols, splits, static_cast<const uint4*>(dy), nullptr, nullptr, nullptr, part, ctr,
      static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

cudaError_t launch_bias_gelu_fwd(std::int64_t rows, int cols, const void* h, const void* b, void* y,
                                 cudaStream_t s) {
  if (cols % 8 || rows < 1) return cudaErrorInvalidValue;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int vpr = cols / 8;
  const int gx = (vpr + 255) / 256;
  // about 8 resident blocks of 256 per SM over the whole grid, each row group >= 4 rows deep
  const std::int64_t gy = std::max<std::int64_t>(
      1, std::min<std::int64_t>((8LL * sms + gx - 1) / gx, (rows + kGeluRows - 1) / kGeluRows));
  bias_gelu_fwd_kernel<<<dim3(gx, static_cast<unsigned>(std::min<std::int64_t>(gy, 65535))), 256, 0, s>>>(
      rows, vpr, static_cast<const uint4*>(h), static_cast<const uint4*>(b), static_cast<uint4*>(y));
  return cudaGetLastError();
}

cudaError_t launch_bias_gelu_bwd(std::int64_t rows, int cols, const void* dy, const void* h, const void* b, void* dh,
                                 void* db, float* part, int splits, cudaStream_t s) {
  if (cols % 8 || splits < 1 || rows < 1) return cudaErrorInvalidValue;
  const dim3 g((cols / 8 + kColThreads - 1) / kColThreads, splits);
  unsigned int* ctr = counter_slots();
  if (!ctr || g.x > kCounterSlots) return cudaErrorInvalidValue;
  colsum_partial_kernel<true><<<g, kColThreads * kRowLanes, 0, s>>>(
      rows, cols, splits, static_cast<const uint4*>(dy), static_cast<const uint4*>(h),
      static_cast<const uint4*>(b), static_cast<uint4*>(dh), part, ctr, static_cast<__nv_bfloat16*>(db));
  return cudaGetLastError();
}

cudaError_t launch_xent_fwd(std::int64_t rows, int V, const void* logits, const std::int64_t* labels, float* loss,
                            float* lse, cudaStream_t s) {
  if (V % 8 || rows < 1 || rows > 0x7fffffff) return cudaErrorInvalidValue;
  xent_fwd_kernel<<<static_cast<unsigned>(rows), kXentThreads, 0, s>>>(V / 8, static_cast<const uint4*>(logits),
                                                                       labels, loss, lse);
  return cudaGetLastError();
}

cudaError_t launch_xent_bwd(std::int64_t rows, int V, const void* logits, const std::int64_t* labels,
                            const float* lse, const float* scale, void* dlogits, cudaStream_t s) {
  if (V % 8 || rows < 1 || rows > 0x7fffffff) return cudaErrorInvalidValue;
  xent_bwd_kernel<<<static_cast<unsigned>(rows), kXentThreads, 0, s>>>(
      V / 8, static_cast<const uint4*>(logits), labels, lse, scale, static_cast<uint4*>(dlogits));
  return cudaGetLastError();
}

namespace {
int elementwise_grid(std::int64_t nvec) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  return static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((nvec + 255) / 256, 8LL * sms)));
}
}  // namespace

cudaError_t launch_rope(std::int64_t batch, int seq, int heads, int dim, const void* x, std::int64_t x_stride,
                        const float* cs, const float* sn, bool inverse, void* y, std::int64_t y_stride,
                        cudaStream_t s) {
  const std::int64_t row = static_cast<std::int64_t>(heads) * dim;
  if (dim % 8 || batch < 1 || seq < 1 || heads < 1 || x_stride % 8 || y_stride % 8 || x_stride < row ||
      y_stride < row)
    return cudaErrorInvalidValue;
  const std::int64_t tokens = batch * seq;
  const int vrow = static_cast<int>(row / 8);
  const dim3 grid((vrow + 255) / 256, static_cast<unsigned>(std::min<std::int64_t>(tokens, 65535)));
  rope_kernel<<<grid, 256, 0, s>>>(tokens, seq, vrow, dim / 8, static_cast<const uint4*>(x), x_stride / 8, cs, sn,
                                   inverse ? -1.0f : 1.0f, static_cast<uint4*>(y), y_stride / 8);
  return cudaGetLastError();
}

cudaError_t launch_swiglu_fwd(std::int64_t rows, int f, const void* g, std::int64_t g_stride, const void* u,
                              std::int64_t u_stride, void* y, cudaStream_t s) {
  if (f % 8 || g_stride % 8 || u_stride % 8 || rows < 1) return cudaErrorInvalidValue;
  swiglu_fwd_kernel<<<elementwise_grid(rows * (f / 8)), 256, 0, s>>>(
      rows, f / 8, static_cast<const uint4*>(g), g_stride / 8, static_cast<const uint4*>(u), u_stride / 8,
      static_cast<uint4*>(y));
  return cudaGetLastError();
}

cudaError_t launch_swiglu_bwd(std::int64_t rows, int f, const void* dy, const void* g, std::int64_t g_stride,
                              const void* u, std::int64_t u_stride, void* dg, std::int64_t dg_stride, void* du,
                              std::int64_t du_stride, cudaStream_t s) {
  if (f % 8 || g_stride % 8 || u_stride % 8 || dg_stride % 8 || du_stride % 8 || rows < 1)
    return cudaErrorInvalidValue;
  swiglu_bwd_kernel<<<elementwise_grid(rows * (f / 8)), 256, 0, s>>>(
      rows, f / 8, static_cast<const uint4*>(dy), static_cast<const uint4*>(g), g_stride / 8,
      static_cast<const uint4*>(u), u_stride / 8, static_cast<uint4*>(dg), dg_stride / 8, static_cast<uint4*>(du),
      du_stride / 8);
  return cudaGetLastError();
}

bool rmsnorm_supported(int h) { return h % 1024 == 0 && h / 1024 >= 1 && h / 1024 <= 8; }

cudaError_t launch_rmsnorm_fwd(std::int64_t rows, int h, float eps, const void* x, const void* r, const void* w,
                               void* s_out, void* y, float* rstd, cudaStream_t s) {
  if (!rmsnorm_supported(h) || rows < 1 || rows > 0x7fffffff || (r == nullptr) != (s_out == nullptr))
    return cudaErrorInvalidValue;
  const unsigned grid = static_cast<unsigned>(rows);
  auto X = static_cast<const uint4*>(x);
  auto R = static_cast<const uint4*>(r);
  auto W = static_cast<const uint4*>(w);
  auto SO = static_cast<uint4*>(s_out);
  auto Y = static_cast<uint4*>(y);
  switch (h / 1024) {
#define FCDP_RMS_FWD(V)                                                                           \
  case V:                                                                                         \
    if (r)                                                                                        \
      rms_fwd_kernel<V, true><<<grid, kRmsThreads, 0, s>>>(h, eps, X, R, W, SO, Y, rstd);         \
    else                                                                                          \
      rms_fwd_kernel<V, false><<<grid, kRmsThreads, 0, s>>>(h, eps, X, nullptr, W, nullptr, Y, rstd); \
    break;
    FCDP_RMS_FWD(1) FCDP_RMS_FWD(2) FCDP_RMS_FWD(3) FCDP_RMS_FWD(4) FCDP_RMS_FWD(5) FCDP_RMS_FWD(6) FCDP_RMS_FWD(7)
    FCDP_RMS_FWD(8)
#undef FCDP_RMS_FWD
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_bwd(std::int64_t rows, int h, const void* dy, const void* x, const void* w,
                               const float* rstd, const void* dres, void* dx, void* dw, float* part, int splits,
                               cudaStream_t s) {
  if (!rmsnorm_supported(h) || rows < 1 || rows > 0x7fffffff || splits < 1) return cudaErrorInvalidValue;
  const unsigned grid = static_cast<unsigned>(rows);
  auto DY = static_cast<const uint4*>(dy);
  auto X = static_cast<const uint4*>(x);
  auto W = static_cast<const uint4*>(w);
  auto DR = static_cast<const uint4*>(dres);
  auto DX = static_cast<uint4*>(dx);
  switch (h / 1024) {
#define FCDP_RMS_BWD(V)                                                                       \
  case V:                                                                                     \
    if (dres)                                                                                 \
      rms_bwd_dx_kernel<V, true><<<grid, kRmsThreads, 0, s>>>(h, DY, X, W, rstd, DR, DX);      \
    else                                                                                      \
      rms_bwd_dx_kernel<V, false><<<grid, kRmsThreads, 0, s>>>(h, DY, X, W, rstd, nullptr, DX); \
    break;
    FCDP_RMS_BWD(1) FCDP_RMS_BWD(2) FCDP_RMS_BWD(3) FCDP_RMS_BWD(4) FCDP_RMS_BWD(5) FCDP_RMS_BWD(6) FCDP_RMS_BWD(7)
    FCDP_RMS_BWD(8)
#undef FCDP_RMS_BWD
    default: return cudaErrorInvalidValue;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !dw) return e;
  const dim3 g2((h / 8 + kColThreads - 1) / kColThreads, splits);
  unsigned int* ctr = counter_slots();
  if (!ctr || g2.x > kCounterSlots) return cudaErrorInvalidValue;
  rms_bwd_dw_partial_kernel<<<g2, kColThreads * kRowLanes, 0, s>>>(rows, h, splits, DY, X, rstd, part, ctr,
                                                                   static_cast<__nv_bfloat16*>(dw));
  return cudaGetLastError();
}

}  // namespace fcdp
