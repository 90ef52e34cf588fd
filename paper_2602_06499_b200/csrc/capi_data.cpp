// C ABI over the stateless data-plane kernels (include/fcdp.h, "data plane").
#include <cmath>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "capi_util.hpp"
#include "common/layout.hpp"
#include <atomic>

#include "fcdp.h"
#include "kernels/kernels.hpp"
#include "kernels/model_gemm.hpp"
#include "kernels/model_kernels.hpp"

struct fcdp_layout {
  fcdp::Layout host;
  std::uint32_t* d_bits = nullptr;
  std::uint32_t* d_tpre = nullptr;
  ~fcdp_layout() {
    if (d_bits) cudaFree(d_bits);
    if (d_tpre) cudaFree(d_tpre);
  }
};

namespace fcdp {

namespace {
thread_local std::string g_last_error;
}

// kernels launched through the stateless driving-model / copy entry points
// (the engine counts its own); read by bench.py for its gpu_launches claim
std::atomic<std::uint64_t> g_model_launches{0};

void set_last_error(const std::string& msg) { g_last_error = msg; }

void check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();  // clear sticky-free errors
  if (e == cudaErrorMemoryAllocation) throw OomError(std::string(what) + ": " + cudaGetErrorString(e));
  throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void upload_layout(Layout& L, std::uint32_t** d_bits, std::uint32_t** d_tpre) {
  const std::size_t bytes = L.bits.size() * sizeof(std::uint32_t);
  const std::size_t tw = L.sparse_t() ? L.twords.size() * sizeof(std::uint32_t) : 0;
  check_cuda(cudaMalloc(d_bits, bytes), "cudaMalloc(layout bits)");
  check_cuda(cudaMalloc(d_tpre, bytes + tw), "cudaMalloc(layout prefix)");
  check_cuda(cudaMemcpy(*d_bits, L.bits.data(), bytes, cudaMemcpyHostToDevice), "upload layout bits");
  check_cuda(cudaMemcpy(*d_tpre, L.tpre.data(), bytes, cudaMemcpyHostToDevice), "upload layout prefix");
  L.dev.bits = *d_bits;
  L.dev.tpre = *d_tpre;
  if (tw) {  // the active trainable words ride behind the prefix
    check_cuda(cudaMemcpy(*d_tpre + L.bits.size(), L.twords.data(), tw, cudaMemcpyHostToDevice), "upload active words");
    L.dev.twords = *d_tpre + L.bits.size();
    L.dev.ntwords = static_cast<std::int64_t>(L.twords.size());
  }
}

}  // namespace fcdp

using fcdp::check_cuda;
using fcdp::guarded;

extern "C" {

const char* fcdp_last_error(void) { return fcdp::g_last_error.c_str(); }

int fcdp_layout_create(int64_t chunks, const uint8_t* mask, int32_t eb, int32_t N, int32_t g,
                       fcdp_layout** out) {
  return guarded([&] {
    auto* L = new fcdp_layout;
    try {
      L->host = fcdp::build_layout(chunks, mask, eb, N, g);
      fcdp::upload_layout(L->host, &L->d_bits, &L->d_tpre);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}

int fcdp_layout_info(const fcdp_layout* L, int64_t* pt, int64_t* pf, int64_t* st, int64_t* sf,
                     int64_t* lt, int64_t* lf) {
  return guarded([&] {
    const auto& d = L->host.dev;
    if (pt) *pt = d.pt;
    if (pf) *pf = d.pf;
    if (st) *st = d.shard_t;
    if (sf) *sf = d.shard_f;
    if (lt) *lt = d.slice_t;
    if (lf) *lf = d.slice_f;
  });
}

void fcdp_layout_destroy(fcdp_layout* L) { delete L; }

int fcdp_partition(const fcdp_layout* L, const void* natural, void* t, void* f, void* stream) {
  return guarded([&] {
    check_cuda(fcdp::launch_partition(L->host, natural, t, f, static_cast<cudaStream_t>(stream)),
               "fcdp_partition");
  });
}

int fcdp_expand(const fcdp_layout* L, const void* const* ts, const void* const* fs, void* natural,
                int32_t set, void* stream) {
  return guarded([&] {
    fcdp::SlicePtrs a{}, b{};
    for (int j = 0; j < L->host.dev.local; ++j) {
      a.p[j] = ts ? ts[j] : nullptr;
      b.p[j] = fs ? fs[j] : nullptr;
    }
    check_cuda(fcdp::launch_expand(L->host, a, b, natural, set, static_cast<cudaStream_t>(stream)),
               "fcdp_expand");
  });
}

int fcdp_rs_slice(const fcdp_layout* L, const void* const* grads, int32_t j, int32_t n, float scale,
                  int32_t final_scale, float* own, void* wire, void* stream) {
  return guarded([&] {
    fcdp::GradPtrs gp{};
    for (int i = 0; i < L->host.dev.local; ++i) gp.p[i] = grads[i];
    check_cuda(fcdp::launch_rs_slice(L->host, gp, j, n, scale, final_scale != 0, own, wire,
                                     static_cast<cudaStream_t>(stream)),
               "fcdp_rs_slice");
  });
}

int fcdp_rs_finalize(int64_t n, int32_t N, int32_t node, int32_t eb, const float* own, const void* wire,
                     int64_t stride, float scale, float* out, void* stream) {
  return guarded([&] {
    check_cuda(fcdp::launch_rs_finalize(n, N, node, eb, own, wire, stride, scale, out,
                                        static_cast<cudaStream_t>(stream)),
               "fcdp_rs_finalize");
  });
}

int fcdp_adam_step(int64_t n, const fcdp_adam_config* c, float* master, float* m, float* v,
                   const float* grad, void* param, int32_t eb, void* stream) {
  return guarded([&] {
    fcdp::AdamParams p{c->lr, c->beta1, c->beta2, c->eps, c->weight_decay,
                       static_cast<float>(1.0 - std::pow(static_cast<double>(c->beta1), c->step)),
                       static_cast<float>(1.0 - std::pow(static_cast<double>(c->beta2), c->step))};
    check_cuda(fcdp::launch_adam(n, p, master, m, v, grad, param, eb, static_cast<cudaStream_t>(stream)),
               "fcdp_adam_step");
  });
}

int fcdp_layernorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* w, const void* b, void* y,
                       float* mean, float* rstd, void* stream) {
  return guarded([&] {
    if (!fcdp::layernorm_supported(h)) throw shardsim::ConfigError("layernorm: h must be a multiple of 256, <= 2048");
    check_cuda(fcdp::launch_layernorm_fwd(rows, h, eps, x, w, b, y, mean, rstd, static_cast<cudaStream_t>(stream)),
               "fcdp_layernorm_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_layernorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* mean,
                       const float* rstd, void* dx, void* dw, void* db, float* scratch, int32_t splits, void* stream) {
  return guarded([&] {
    if (!fcdp::layernorm_supported(h)) throw shardsim::ConfigError("layernorm: h must be a multiple of 256, <= 2048");
    check_cuda(fcdp::launch_layernorm_bwd(rows, h, dy, x, w, mean, rstd, dx, dw, db, scratch, splits,
                                          static_cast<cudaStream_t>(stream)),
               "fcdp_layernorm_bwd");
    fcdp::g_model_launches += (dw && db) ? 2 : 1;
  });
}

int fcdp_add_layernorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* r, const void* w,
                           const void* b, void* s_out, void* y, float* mean, float* rstd, void* stream) {
  return guarded([&] {
    if (!fcdp::layernorm_supported(h)) throw shardsim::ConfigError("layernorm: h must be a multiple of 256, <= 2048");
    if (!r || !s_out) throw shardsim::ConfigError("add_layernorm: r and s_out are required");
    check_cuda(fcdp::launch_layernorm_fwd(rows, h, eps, x, w, b, y, mean, rstd, static_cast<cudaStream_t>(stream), r,
                                          s_out),
               "fcdp_add_layernorm_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_layernorm_bwd_res(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* mean,
                           const float* rstd, const void* dres, void* dx, void* dw, void* db, float* scratch,
                           int32_t splits, void* stream) {
  return guarded([&] {
    if (!fcdp::layernorm_supported(h)) throw shardsim::ConfigError("layernorm: h must be a multiple of 256, <= 2048");
    check_cuda(fcdp::launch_layernorm_bwd(rows, h, dy, x, w, mean, rstd, dx, dw, db, scratch, splits,
                                          static_cast<cudaStream_t>(stream), dres),
               "fcdp_layernorm_bwd_res");
    fcdp::g_model_launches += (dw && db) ? 2 : 1;
  });
}

int fcdp_rmsnorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* r, const void* w, void* s_out,
                     void* y, float* rstd, void* stream) {
  return guarded([&] {
    if (!fcdp::rmsnorm_supported(h)) throw shardsim::ConfigError("rmsnorm: h must be a multiple of 1024, <= 8192");
    if ((r == nullptr) != (s_out == nullptr)) throw shardsim::ConfigError("rmsnorm: r and s_out go together");
    check_cuda(fcdp::launch_rmsnorm_fwd(rows, h, eps, x, r, w, s_out, y, rstd, static_cast<cudaStream_t>(stream)),
               "fcdp_rmsnorm_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_rmsnorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* rstd,
                     const void* dres, void* dx, void* dw, float* scratch, int32_t splits, void* stream) {
  return guarded([&] {
    if (!fcdp::rmsnorm_supported(h)) throw shardsim::ConfigError("rmsnorm: h must be a multiple of 1024, <= 8192");
    check_cuda(fcdp::launch_rmsnorm_bwd(rows, h, dy, x, w, rstd, dres, dx, dw, scratch, splits,
                                        static_cast<cudaStream_t>(stream)),
               "fcdp_rmsnorm_bwd");
    fcdp::g_model_launches += dw ? 2 : 1;
  });
}

int fcdp_colsum_splits(int64_t rows, int32_t cols) { return fcdp::colsum_splits(rows, cols); }

int fcdp_bias_grad(int64_t rows, int32_t cols, const void* dy, void* db, float* scratch, int32_t splits,
                   void* stream) {
  return guarded([&] {
    if (cols % 8 || cols > 16384) throw shardsim::ConfigError("bias_grad: cols must be a multiple of 8 and <= 16384");
    check_cuda(fcdp::launch_colsum(rows, cols, dy, db, scratch, splits, static_cast<cudaStream_t>(stream)),
               "fcdp_bias_grad");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_bias_gelu_fwd(int64_t rows, int32_t cols, const void* h, const void* b, void* y, void* stream) {
  return guarded([&] {
    if (cols % 8) throw shardsim::ConfigError("bias_gelu: cols must be a multiple of 8");
    check_cuda(fcdp::launch_bias_gelu_fwd(rows, cols, h, b, y, static_cast<cudaStream_t>(stream)),
               "fcdp_bias_gelu_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_bias_gelu_bwd(int64_t rows, int32_t cols, const void* dy, const void* h, const void* b, void* dh, void* db,
                       float* scratch, int32_t splits, void* stream) {
  return guarded([&] {
    if (cols % 8 || cols > 16384) throw shardsim::ConfigError("bias_gelu: cols must be a multiple of 8 and <= 16384");
    check_cuda(fcdp::launch_bias_gelu_bwd(rows, cols, dy, h, b, dh, db, scratch, splits,
                                          static_cast<cudaStream_t>(stream)),
               "fcdp_bias_gelu_bwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_xent_fwd(int64_t rows, int32_t vocab, const void* logits, const int64_t* labels, float* loss, float* lse,
                  void* stream) {
  return guarded([&] {
    if (vocab % 8) throw shardsim::ConfigError("xent: vocab must be a multiple of 8");
    check_cuda(fcdp::launch_xent_fwd(rows, vocab, logits, labels, loss, lse, static_cast<cudaStream_t>(stream)),
               "fcdp_xent_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_xent_bwd(int64_t rows, int32_t vocab, const void* logits, const int64_t* labels, const float* lse,
                  const float* scale, void* dlogits, void* stream) {
  return guarded([&] {
    if (vocab % 8) throw shardsim::ConfigError("xent: vocab must be a multiple of 8");
    check_cuda(fcdp::launch_xent_bwd(rows, vocab, logits, labels, lse, scale, dlogits,
                                     static_cast<cudaStream_t>(stream)),
               "fcdp_xent_bwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_rope(int64_t batch, int32_t seq, int32_t heads, int32_t dim, const void* x, int64_t x_stride,
              const float* cos_table, const float* sin_table, int32_t inverse, void* y, int64_t y_stride,
              void* stream) {
  return guarded([&] {
    const int64_t row = static_cast<int64_t>(heads) * dim;
    if (dim % 8) throw shardsim::ConfigError("rope: head dim must be a multiple of 8");
    if (x_stride == 0) x_stride = row;
    if (y_stride == 0) y_stride = row;
    if (x_stride % 8 || y_stride % 8 || x_stride < row || y_stride < row)
      throw shardsim::ConfigError("rope: token strides must be multiples of 8 and >= heads * dim");
    check_cuda(fcdp::launch_rope(batch, seq, heads, dim, x, x_stride, cos_table, sin_table, inverse != 0, y, y_stride,
                                 static_cast<cudaStream_t>(stream)),
               "fcdp_rope");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_swiglu_fwd(int64_t rows, int32_t f, const void* g, int64_t g_stride, const void* u, int64_t u_stride, void* y,
                    void* stream) {
  return guarded([&] {
    if (f % 8 || g_stride % 8 || u_stride % 8) throw shardsim::ConfigError("swiglu: f and strides must be multiples of 8");
    check_cuda(fcdp::launch_swiglu_fwd(rows, f, g, g_stride, u, u_stride, y, static_cast<cudaStream_t>(stream)),
               "fcdp_swiglu_fwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_swiglu_bwd(int64_t rows, int32_t f, const void* dy, const void* g, int64_t g_stride, const void* u,
                    int64_t u_stride, void* dg, int64_t dg_stride, void* du, int64_t du_stride, void* stream) {
  return guarded([&] {
    if (f % 8 || g_stride % 8 || u_stride % 8 || dg_stride % 8 || du_stride % 8)
      throw shardsim::ConfigError("swiglu: f and strides must be multiples of 8");
    check_cuda(fcdp::launch_swiglu_bwd(rows, f, dy, g, g_stride, u, u_stride, dg, dg_stride, du, du_stride,
                                       static_cast<cudaStream_t>(stream)),
               "fcdp_swiglu_bwd");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_copy_rows(int64_t rows, int64_t row_bytes, const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                   void* stream) {
  return guarded([&] {
    check_cuda(fcdp::launch_copy_rows(rows, row_bytes, src, src_pitch, dst, dst_pitch,
                                      static_cast<cudaStream_t>(stream)),
               "fcdp_copy_rows (16-byte aligned pointers, row bytes and pitches)");
    fcdp::g_model_launches += 1;
  });
}

int fcdp_copy_segments(int32_t n, const void* const* src, void* const* dst, const int64_t* bytes, void* stream) {
  return guarded([&] {
    if (n < 0) throw shardsim::ConfigError("copy_segments: negative count");
    check_cuda(fcdp::launch_copy_segments(n, src, dst, bytes, static_cast<cudaStream_t>(stream)),
               "fcdp_copy_segments (16-byte aligned pointers and sizes)");
    fcdp::g_model_launches += static_cast<std::uint64_t>((n + fcdp::kMaxCopySegs - 1) / fcdp::kMaxCopySegs);
  });
}

int fcdp_mlp_gemm_available(void) { return fcdp::mlp_gemm_available(nullptr) ? 1 : 0; }

int fcdp_fc_gelu_fwd(int64_t rows, int64_t in, int64_t out, const void* x, const void* w, const void* b, void* act,
                     void* aux, void* stream) {
  return guarded([&] {
    std::string why;
    if (!fcdp::mlp_gemm_available(&why)) throw shardsim::ConfigError("fc_gelu: " + why);
    if (in % 8 || out % 8) throw shardsim::ConfigError("fc_gelu: in and out must be multiples of 8");
    std::string err;
    if (fcdp::launch_fc_gelu_fwd(rows, in, out, x, w, b, act, aux, static_cast<cudaStream_t>(stream), &err) !=
        cudaSuccess)
      throw fcdp::CudaError("fcdp_fc_gelu_fwd: " + err);
  });
}

int fcdp_fc2_dgrad_dgelu(int64_t rows, int64_t hidden, int64_t ffn, const void* dy, const void* w2, const void* aux,
                         void* dpre, void* db1, void* stream) {
  return guarded([&] {
    std::string why;
    if (!fcdp::mlp_gemm_available(&why)) throw shardsim::ConfigError("fc2_dgrad_dgelu: " + why);
    if (hidden % 8 || ffn % 8) throw shardsim::ConfigError("fc2_dgrad_dgelu: hidden and ffn must be multiples of 8");
    std::string err;
    if (fcdp::launch_fc2_dgrad_dgelu(rows, hidden, ffn, dy, w2, aux, dpre, db1, static_cast<cudaStream_t>(stream),
                                     &err) != cudaSuccess)
      throw fcdp::CudaError("fcdp_fc2_dgrad_dgelu: " + err);
  });
}

uint64_t fcdp_model_kernel_launches(int32_t reset) {
  return reset ? fcdp::g_model_launches.exchange(0) : fcdp::g_model_launches.load();
}

int fcdp_enable_peer_access(int32_t device, int32_t peer) {
  return guarded([&] {
    int can = 0;
    check_cuda(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
    if (!can) throw shardsim::ConfigError("device " + std::to_string(device) + " cannot access peer " +
                                         std::to_string(peer));
    int cur = 0;
    check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else check_cuda(e, "cudaDeviceEnablePeerAccess");
    check_cuda(cudaSetDevice(cur), "cudaSetDevice");
  });
}

int fcdp_adam_grad_step(int64_t n, const fcdp_adam_config* c, float scale, int32_t num_segs,
                        const int64_t* elem_offsets, const void* const* grads, const int64_t* counts,
                        float* master, float* m, float* v, void* param, int32_t eb, float* keep_grad,
                        void* stream) {
  return guarded([&] {
    if (eb != 2 && eb != 4) throw shardsim::ConfigError("adam_grad_step: element bytes must be 2 or 4");
    const int64_t V = fcdp::kChunkBytes / eb;
    if (n % V) throw shardsim::ConfigError("adam_grad_step: n must be whole 16-byte chunks");
    if (num_segs < 0 || num_segs > fcdp::kMaxGradSegs) throw shardsim::ConfigError("adam_grad_step: too many segments");
    fcdp::GradSegs sg;
    sg.n = num_segs;
    for (int i = 0; i < num_segs; ++i) {
      if (elem_offsets[i] % V || counts[i] % V) throw shardsim::ConfigError("adam_grad_step: unaligned segment");
      sg.dst_chunk[i] = elem_offsets[i] / V;
      sg.nchunks[i] = counts[i] / V;
      sg.src[i] = grads[i];
    }
    fcdp::AdamParams p{c->lr, c->beta1, c->beta2, c->eps, c->weight_decay,
                       static_cast<float>(1.0 - std::pow(static_cast<double>(c->beta1), c->step)),
                       static_cast<float>(1.0 - std::pow(static_cast<double>(c->beta2), c->step))};
    check_cuda(fcdp::launch_adam_grad(n / V, sg, p, scale, master, m, v, param, eb, keep_grad,
                                      static_cast<cudaStream_t>(stream)),
               "fcdp_adam_grad_step");
  });
}

int fcdp_init_natural(const fcdp_layout* L, uint64_t seed, int32_t layer, const fcdp_init_range* r,
                      int32_t nr, void* natural, void* stream) {
  return guarded([&] {
    auto s = static_cast<cudaStream_t>(stream);
    fcdp::InitRange* d = nullptr;
    if (nr > 0) {
      check_cuda(cudaMallocAsync(&d, sizeof(fcdp::InitRange) * nr, s), "init ranges alloc");
      static_assert(sizeof(fcdp::InitRange) == sizeof(fcdp_init_range), "init range ABI");
      check_cuda(cudaMemcpyAsync(d, r, sizeof(fcdp::InitRange) * nr, cudaMemcpyHostToDevice, s),
                 "init ranges upload");
    }
    const int64_t elems = L->host.dev.chunks * fcdp::kChunkBytes / L->host.dev.elem_bytes;
    check_cuda(fcdp::launch_init_natural(elems, L->host.dev.elem_bytes, seed, layer, d, nr, natural, s),
               "fcdp_init_natural");
    if (d) check_cuda(cudaFreeAsync(d, s), "init ranges free");
    check_cuda(cudaStreamSynchronize(s), "init sync");  // ranges live on the caller's stack
  });
}

}  // extern "C"
