// GPT-2 MLP GEMMs of the driving model with their elementwise neighbours fused
// into cuBLASLt epilogues (library GEMMs; not part of the parameter-movement
// path):
//   forward   act = gelu_tanh(x W1^T + b1), aux = x W1^T + b1        GELU_AUX_BIAS
//   backward  dpre = (dy W2) * gelu'(aux), db1 = sum_rows dpre        DGELU_BGRAD
// which replaces the separate bias + GELU pass and the GELU-backward + bias
// gradient pass (model_kernels.cu) around the fc / fc2-dgrad GEMMs.
//
// libcublasLt is resolved at run time (dlopen of the copy the process already
// has, normally torch's), so libfcdp.so keeps no link-time dependency on it;
// when it is absent the entry points answer FCDP_ERR_CONFIG and the caller
// keeps the unfused kernels.
//
// Row-major [rows x cols] tensors are column-major [cols x rows]: with W1 [out x in]
// row-major, act^T [out x rows] = op_T(W1 as col-major [in x out]) * x^T [in x rows].
#include "kernels/model_gemm.hpp"

#include <cublasLt.h>
#include <dlfcn.h>

#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>

namespace fcdp {
namespace {

struct LtApi {
  decltype(&cublasLtCreate) create = nullptr;
  decltype(&cublasLtMatmulDescCreate) desc_create = nullptr;
  decltype(&cublasLtMatmulDescDestroy) desc_destroy = nullptr;
  decltype(&cublasLtMatmulDescSetAttribute) desc_set = nullptr;
  decltype(&cublasLtMatrixLayoutCreate) layout_create = nullptr;
  decltype(&cublasLtMatrixLayoutDestroy) layout_destroy = nullptr;
  decltype(&cublasLtMatmulPreferenceCreate) pref_create = nullptr;
  decltype(&cublasLtMatmulPreferenceDestroy) pref_destroy = nullptr;
  decltype(&cublasLtMatmulPreferenceSetAttribute) pref_set = nullptr;
  decltype(&cublasLtMatmulAlgoGetHeuristic) heuristic = nullptr;
  decltype(&cublasLtMatmul) matmul = nullptr;
  bool ok = false;
  std::string why;
};

LtApi load_api() {
  LtApi a;
  void* h = dlopen("libcublasLt.so.12", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libcublasLt.so.12", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.why = "libcublasLt.so.12 not loadable (load torch / cuBLAS first)";
    return a;
  }
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn && a.why.empty()) a.why = std::string("missing symbol ") + name;
  };
  sym(a.create, "cublasLtCreate");
  sym(a.desc_create, "cublasLtMatmulDescCreate");
  sym(a.desc_destroy, "cublasLtMatmulDescDestroy");
  sym(a.desc_set, "cublasLtMatmulDescSetAttribute");
  sym(a.layout_create, "cublasLtMatrixLayoutCreate");
  sym(a.layout_destroy, "cublasLtMatrixLayoutDestroy");
  sym(a.pref_create, "cublasLtMatmulPreferenceCreate");
  sym(a.pref_destroy, "cublasLtMatmulPreferenceDestroy");
  sym(a.pref_set, "cublasLtMatmulPreferenceSetAttribute");
  sym(a.heuristic, "cublasLtMatmulAlgoGetHeuristic");
  sym(a.matmul, "cublasLtMatmul");
  a.ok = a.why.empty();
  return a;
}

constexpr std::size_t kWorkspace = 32u << 20;

// One plan per (device, shape, epilogue): descriptors + the heuristic's algorithm.
struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  cublasLtMatmulAlgo_t algo{};
};

struct State {
  std::mutex mu;
  LtApi api;
  bool loaded = false;
  std::map<int, cublasLtHandle_t> handle;
  std::map<int, void*> workspace;
  std::map<std::tuple<int, std::int64_t, std::int64_t, std::int64_t, int>, Plan> plans;
};

State& state() {
  static State s;
  return s;
}

void lt_check(cublasStatus_t st, const char* what) {
  if (st != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string(what) + ": cublasLt status " + std::to_string(st));
}

// D[m x n] = op(A) * B (col-major), bf16 in / out, fp32 accumulate; epilogue with
// bias (length m) and aux [m x n] (ld m).
cudaError_t run(int epi, bool trans_a, std::int64_t m, std::int64_t n, std::int64_t k, const void* A,
                std::int64_t lda, const void* B, std::int64_t ldb, void* D, const void* bias_in, void* bias_out,
                void* aux, cudaStream_t s, std::string* err) {
  State& st = state();
  std::lock_guard<std::mutex> g(st.mu);
  if (!st.loaded) {
    st.api = load_api();
    st.loaded = true;
  }
  const LtApi& L = st.api;
  if (!L.ok) {
    *err = L.why;
    return cudaErrorNotSupported;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  try {
    if (!st.handle.count(dev)) {
      cublasLtHandle_t h;
      lt_check(L.create(&h), "cublasLtCreate");
      st.handle[dev] = h;
      void* w = nullptr;
      if (cudaMalloc(&w, kWorkspace) != cudaSuccess) throw std::runtime_error("cudaMalloc(cublasLt workspace)");
      st.workspace[dev] = w;
    }
    const auto key = std::make_tuple(dev, m, n, k, epi * 2 + (trans_a ? 1 : 0));
    auto it = st.plans.find(key);
    if (it == st.plans.end()) {
      Plan p;
      lt_check(L.desc_create(&p.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F), "MatmulDescCreate");
      const cublasOperation_t ta = trans_a ? CUBLAS_OP_T : CUBLAS_OP_N, tb = CUBLAS_OP_N;
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)), "TRANSA");
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)), "TRANSB");
      const cublasLtEpilogue_t e = static_cast<cublasLtEpilogue_t>(epi);
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e)), "EPILOGUE");
      const cudaDataType_t bt = CUDA_R_16BF;
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt)), "BIAS_DATA_TYPE");
      const std::int64_t ld_aux = m;
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &ld_aux, sizeof(ld_aux)), "AUX_LD");
      // A is [k x m] col-major when transposed (ld = lda), else [m x k]
      lt_check(L.layout_create(&p.a, CUDA_R_16BF, trans_a ? k : m, trans_a ? m : k, lda), "layout A");
      lt_check(L.layout_create(&p.b, CUDA_R_16BF, k, n, ldb), "layout B");
      lt_check(L.layout_create(&p.d, CUDA_R_16BF, m, n, m), "layout D");
      cublasLtMatmulPreference_t pref;
      lt_check(L.pref_create(&pref), "PreferenceCreate");
      const std::uint64_t ws = kWorkspace;
      lt_check(L.pref_set(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws, sizeof(ws)), "workspace pref");
      // the pointers' alignment steers the heuristic: set representative ones
      const void* bias_probe = bias_out ? bias_out : bias_in;
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias_probe, sizeof(bias_probe)), "BIAS_POINTER");
      lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(void*)), "AUX_POINTER");
      cublasLtMatmulHeuristicResult_t r{};
      int found = 0;
      const cublasStatus_t hs = L.heuristic(st.handle[dev], p.desc, p.a, p.b, p.d, p.d, pref, 1, &r, &found);
      L.pref_destroy(pref);
      if (hs != CUBLAS_STATUS_SUCCESS || found == 0)
        throw std::runtime_error("cublasLt: no algorithm for epilogue " + std::to_string(epi));
      p.algo = r.algo;
      it = st.plans.emplace(key, p).first;
    }
    Plan& p = it->second;
    const void* bias_ptr = bias_out ? bias_out : bias_in;
    lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias_ptr, sizeof(bias_ptr)), "BIAS_POINTER");
    lt_check(L.desc_set(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER, &aux, sizeof(aux)), "AUX_POINTER");
    const float one = 1.0f, zero = 0.0f;
    lt_check(L.matmul(st.handle[dev], p.desc, &one, A, p.a, B, p.b, &zero, D, p.d, D, p.d, &p.algo,
                      st.workspace[dev], kWorkspace, s),
             "cublasLtMatmul");
  } catch (const std::exception& ex) {
    *err = ex.what();
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace

bool mlp_gemm_available(std::string* why) {
  State& st = state();
  std::lock_guard<std::mutex> g(st.mu);
  if (!st.loaded) {
    st.api = load_api();
    st.loaded = true;
  }
  if (!st.api.ok && why) *why = st.api.why;
  return st.api.ok;
}

cudaError_t launch_fc_gelu_fwd(std::int64_t rows, std::int64_t in, std::int64_t out, const void* x, const void* w,
                               const void* b, void* act, void* aux, cudaStream_t s, std::string* err) {
  // act^T [out x rows] = op_T(W as col-major [in x out]) * x^T [in x rows]
  return run(CUBLASLT_EPILOGUE_GELU_AUX_BIAS, true, out, rows, in, w, in, x, in, act, b, nullptr, aux, s, err);
}

cudaError_t launch_fc2_dgrad_dgelu(std::int64_t rows, std::int64_t hidden, std::int64_t ffn, const void* dy,
                                   const void* w2, const void* aux, void* dpre, void* db1, cudaStream_t s,
                                   std::string* err) {
  // dpre^T [ffn x rows] = (W2 as col-major [ffn x hidden]) * dy^T [hidden x rows], then * gelu'(aux)
  return run(CUBLASLT_EPILOGUE_DGELU_BGRAD, false, ffn, rows, hidden, w2, ffn, dy, hidden, dpre, nullptr, db1,
             const_cast<void*>(aux), s, err);
}

}  // namespace fcdp
