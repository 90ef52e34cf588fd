// Per-rank FCDP engine (see engine.hpp for the overall contract).
//
// Event semantics follow the reference builder (proj/src/schedule.cpp:107-292)
// and Algorithm 1; the data layout is the one in
// common/layout.hpp.  Cross-rank ordering uses monotone 32-bit flags in the
// shared control block, written and awaited by the GPU streams themselves
// (cuStreamWriteValue32 / cuStreamWaitValue32):
//   slice fill q :  [wait peers SliceFree >= q-K] fill X[q%K] [SliceReady=q]
//   pull       q :  [wait peers SliceReady >= q] expand/gather -> W [SliceFree=q]
//   NIC piece  p :  [wait receivers Consumed >= p-ring] D2H into ring slot (or
//                   straight into the host cache: write-once staging) [Staged=p]
//                   -> NIC thread paces the wire, then TxReady=p
//   receive    p :  [wait sender TxReady >= p] H2D from its slot [Consumed=p]
//   rs         u :  [GradReady=u] [wait peers GradReady >= u] pull-reduce [GradFree=u]
// Every rank walks the same program, so sequence numbers agree, and a rank
// enqueues a wait only after the producing write was posted by its peer's host
// (SharedBlock::await_posted), so no wait can close a cycle.
#include "runtime/engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>

#include <nvtx3/nvToolsExt.h>
#include <sys/mman.h>

#include "capi_util.hpp"
#include "runtime/streamops.hpp"

namespace fcdp {

void check_cuda(cudaError_t e, const char* what);

namespace {

#define CK(expr) check_cuda((expr), #expr)

using shardsim::Event;
using shardsim::EventKind;
using shardsim::ParamSet;

constexpr int kElided = -2;  // PendingSlice::slot of an elided (resident) reload
constexpr int kAliasW = 3;   // w_of_layer_: the layer is read in place from this GPU's shard (G = 1)
constexpr int kAliasX = -4;  // x_of_t_/x_of_f_: the gathered portion is the shard itself

std::size_t round_up(std::size_t x, std::size_t a) { return (x + a - 1) / a * a; }

template <typename T>
T* dalloc(std::size_t bytes, const char* what) {
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, std::max<std::size_t>(bytes, 256));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw OomError(std::string("cudaMalloc(") + what + ", " + std::to_string(bytes) + " B) failed: " +
                   cudaGetErrorString(e));
  }
  check_cuda(cudaMemset(p, 0, std::max<std::size_t>(bytes, 256)), what);
  return static_cast<T*>(p);
}

// NVTX: one host range per executed program event ("fcdp" domain, message
// "<kind> L<layer>"), so ncu can select an event's kernels
// (--nvtx --nvtx-include "fcdp@reduce_scatter*").  Header-only NVTX3: free when
// no tool is attached.
nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("fcdp");
  return d;
}

struct NvtxRange {
  explicit NvtxRange(const shardsim::Event& e) {
    char msg[64];
    std::snprintf(msg, sizeof(msg), "%s L%d", shardsim::to_string(e.kind), e.layer);
    nvtxEventAttributes_t a{};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = msg;
    nvtxDomainRangePushEx(nvtx_domain(), &a);
  }
  ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

bool wants_t(ParamSet s) { return s != ParamSet::FrozenOnly; }
bool wants_f(ParamSet s) { return s != ParamSet::TrainableOnly; }

}  // namespace

template <typename F>
void Engine::timed(int cls, cudaStream_t s, std::uint64_t alg_bytes, F&& launch, std::uint64_t link_bytes) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (timing_) {
    for (cudaEvent_t* e : {&a, &b}) {
      if (!timing_pool_.empty()) {
        *e = timing_pool_.back();
        timing_pool_.pop_back();
      } else {
        CK(cudaEventCreate(e));
      }
    }
    CK(cudaEventRecord(a, s));
  }
  CK(launch());
  kstats_.launches[cls] += 1;
  kstats_.alg_bytes[cls] += alg_bytes;
  kstats_.link_bytes[cls] += link_bytes;
  if (timing_) {
    CK(cudaEventRecord(b, s));
    timed_pending_.push_back({cls, a, b, alg_bytes});
  }
}

void Engine::kernel_stats(fcdp_kernel_stats* out, bool reset) {
  sync();
  for (const TimedLaunch& t : timed_pending_) {
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    kstats_.total_ms[t.cls] += ms;
    kstats_.timed_launches[t.cls] += 1;
    timing_pool_.push_back(t.a);
    timing_pool_.push_back(t.b);
  }
  timed_pending_.clear();
  *out = kstats_;
  if (reset) kstats_ = fcdp_kernel_stats{};
}

Engine::Engine(const fcdp_engine_config& cfg, const shardsim::ModelSpec& model,
               const shardsim::ClusterTopology& topo, const shardsim::StrategyPlan& plan,
               const std::uint8_t* const* chunk_masks)
    : cfg_(cfg), shm_name_(cfg.shm_name ? cfg.shm_name : ""), model_(model), topo_(topo), plan_(plan) {
  topo_.validate();
  plan_.validate(topo_);
  model_.validate();
  if (plan_.kind == shardsim::StrategyKind::Zero2)
    throw shardsim::ConfigError("engine: the B200 data plane executes zero3, mics, zeropp, fcdp and fcdp-comm programs");
  zeropp_ = plan_.kind == shardsim::StrategyKind::ZeroPP;
  mics_ = plan_.kind == shardsim::StrategyKind::MiCS;
  if (mics_ && plan_.effective_subgroup(topo_) != topo_.gpus_per_node)
    throw shardsim::ConfigError("engine: mics is executed with subgroup_size = gpus_per_node");
  if (shm_name_.empty()) throw shardsim::ConfigError("engine: shm_name is required");
  N_ = topo_.num_nodes;
  g_ = topo_.gpus_per_node;
  G_ = N_ * g_;
  if (g_ > kMaxLocal || N_ > kMaxNodes) throw shardsim::ConfigError("engine: at most 8 nodes x 8 GPUs");
  if (cfg.world_size != G_) throw shardsim::ConfigError("engine: world_size must equal num_nodes * gpus_per_node");
  rank_ = cfg.rank;
  n_ = rank_ / g_;
  j_ = rank_ % g_;
  Ns_ = mics_ ? 1 : N_;
  ns_ = mics_ ? 0 : n_;
  eb_ = model_.param_bytes_per_element;
  V_ = kChunkBytes / eb_;
  if (cfg_.x_slots < 2) cfg_.x_slots = 3;
  if (cfg_.inter_slots < 4) cfg_.inter_slots = 16;  // staging ring depth, in pieces
  if (cfg_.timeout_s <= 0) cfg_.timeout_s = 300.0;
  use_ce_ = cfg_.use_copy_engine != 0;
  chunk_bytes_ = cfg_.inter_chunk_bytes > 0 ? cfg_.inter_chunk_bytes : (4ll << 20);
  chunk_bytes_ = (chunk_bytes_ + kChunkBytes - 1) / kChunkBytes * kChunkBytes;

  CK(cudaSetDevice(cfg_.device));
  // NUMA: run this rank's host thread - and the NIC thread it starts - on the
  // GPU's socket, and place its pinned host tiers there (multi-socket hosts).
  numa_.num_nodes = numa_online_nodes();
  numa_.gpu_node = numa_node_of_gpu(cfg_.device);
  // The pin is temporary: it covers the first touch of the host tiers and the
  // start of the NIC thread (which keeps it); the caller's thread gets its own
  // affinity back at the end of the constructor.
  const char* numa_env = std::getenv("FCDP_NUMA");
  const SavedAffinity caller_affinity = numa_save_affinity();
  if (numa_.num_nodes > 1 && numa_.gpu_node >= 0 && !(numa_env && std::strcmp(numa_env, "0") == 0))
    numa_.cpus_bound = numa_pin_thread(numa_.gpu_node);
  build_layouts(chunk_masks);

  // staging ring: inter_slots pieces of chunk_bytes_ per class per rank
  shm_ = std::make_unique<SharedBlock>(shm_name_, rank_, G_, N_, g_, cfg_.inter_slots,
                                       static_cast<std::uint64_t>(chunk_bytes_), cfg_.timeout_s);
  CK(cudaHostRegister(shm_->base(), shm_->bytes(), cudaHostRegisterPortable | cudaHostRegisterMapped));
  CK(cudaHostGetDevicePointer(&shm_dev_base_, shm_->base(), 0));
  if (!StreamOps::available()) throw CudaError("engine: stream memory operations unavailable on this device");

  allocate();
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&s_comp_, cudaStreamNonBlocking, lo));
  CK(cudaStreamCreateWithPriority(&s_gather_, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_cache_, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_rs_, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_agsend_, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_rssend_, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&s_rsrecv_, cudaStreamNonBlocking, hi));
  // G = 1 fused RS + AdamW: on the compute stream by default (below);
  // FCDP_OPT_STREAM=rs keeps it on s_rs_, FCDP_OPT_PRIO=low moves it to s_opt_
  // at the compute stream's priority.
  CK(cudaStreamCreateWithPriority(&s_opt_, cudaStreamNonBlocking, lo));
  CK(cudaEventCreateWithFlags(&opt_fork_, cudaEventDisableTiming));
  {
    const char* e = std::getenv("FCDP_OPT_PRIO");
    opt_low_ = e && std::strcmp(e, "low") == 0;
    // Default: the fused update runs on the compute stream right after the
    // layer's backward, with its full grid (0.85 of the HBM copy rate per launch).
    // FCDP_OPT_STREAM=rs runs it on the high-priority RS stream with its grid
    // capped at ONE CTA per SM (16 K registers, no shared memory): the backward
    // GEMMs' CTAs (256 threads x 168 registers, 213 KB shared memory; ncu,
    // profiles/r02_gemm_resources.csv) leave exactly that much room per SM, so
    // it streams beside them.  A/B/C on one box (profiles/r02_ab_opt_stream.json):
    // 69.3 ms per step against 71.2 ms serialised, 71.3 ms with two CTAs per SM
    // (no longer fits beside a GEMM CTA); each launch then spans the GEMMs it
    // overlaps, about 0.37 of the roofline per launch.  FCDP_OPT_PRIO=low uses
    // the low-priority stream, FCDP_OPT_CTAS_PER_SM=k sets the cap (0 = full grid).
    const char* c = std::getenv("FCDP_OPT_STREAM");
    opt_on_compute_ = !opt_low_ && !(c && std::strcmp(c, "rs") == 0);
    const char* k = std::getenv("FCDP_OPT_CTAS_PER_SM");
    opt_ctas_per_sm_ = k ? std::atoi(k) : (opt_on_compute_ ? 0 : 1);
    const char* r = std::getenv("FCDP_RS_CTAS_PER_SM");
    rs_ctas_per_sm_ = r ? std::atoi(r) : 0;
    const char* rsx = std::getenv("FCDP_RS_STREAM");
    rs_on_compute_ = rsx && std::strcmp(rsx, "compute") == 0;
  }
  for (auto& e : fin_done_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : rs_kernel_done_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : rs_staged_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  x_reader_.assign(static_cast<std::size_t>(cfg_.x_slots), nullptr);
  for (auto& e : x_reader_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : rs_done_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&iter_done_, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&alias_fence_, cudaEventDisableTiming));
  for (auto& e : join_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));

  exchange_handles();
  nic_ = std::make_unique<NicEmulator>(*shm_, rank_, n_, topo_.inter_node.bandwidth_bytes_per_s,
                                       cfg_.nic_pacing != 0);
  if (numa_.cpus_bound) numa_restore_affinity(caller_affinity);
  shm_->barrier(cfg_.timeout_s);
}

Engine::~Engine() {
  try {
    sync();
    if (shm_) shm_->barrier(cfg_.timeout_s, false);  // no peer still reads our memory (even after an abort)
  } catch (...) {
  }
  nic_.reset();
  for (int jj = 0; jj < g_; ++jj)
    if (jj != j_ && peer_base_[jj]) cudaIpcCloseMemHandle(peer_base_[jj]);
  for (cudaEvent_t e : ev_done_) cudaEventDestroy(e);
  for (cudaEvent_t e : x_reader_) cudaEventDestroy(e);
  for (cudaEvent_t e : rs_done_) cudaEventDestroy(e);
  for (cudaEvent_t e : timing_pool_) cudaEventDestroy(e);
  for (cudaEvent_t e : trace_begin_) cudaEventDestroy(e);
  for (cudaEvent_t e : trace_end_) cudaEventDestroy(e);
  if (trace_start_) cudaEventDestroy(trace_start_);
  for (const TimedLaunch& t : timed_pending_) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (iter_done_) cudaEventDestroy(iter_done_);
  if (alias_fence_) cudaEventDestroy(alias_fence_);
  for (cudaEvent_t e : join_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : rs_kernel_done_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : rs_staged_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : fin_done_)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {s_comp_, s_gather_, s_cache_, s_rs_, s_agsend_, s_rssend_, s_rsrecv_, s_opt_})
    if (s) cudaStreamDestroy(s);
  if (opt_fork_) cudaEventDestroy(opt_fork_);
  for (void* p : {static_cast<void*>(param_t_), static_cast<void*>(param_f_), static_cast<void*>(master_),
                  static_cast<void*>(adam_m_), static_cast<void*>(adam_v_), static_cast<void*>(grad32_),
                  static_cast<void*>(w_slots_[0]), static_cast<void*>(w_slots_[1]),
                  static_cast<void*>(peer_arena_), static_cast<void*>(own32_[0]), static_cast<void*>(own32_[1]),
                  static_cast<void*>(wire_[0]), static_cast<void*>(wire_[1]), static_cast<void*>(rx_[0]),
                  static_cast<void*>(rx_[1])})
    if (p) cudaFree(p);
  for (unsigned char* p : retained_)
    if (p) cudaFree(p);  // cudaMallocAsync memory; cudaFree synchronises
  for (LayerRt& l : layers_) {
    if (l.d_bits) cudaFree(l.d_bits);
    if (l.d_tpre) cudaFree(l.d_tpre);
  }
  for (auto& ev : cache_staged_)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : ag_staged_)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : d2h_done_)
    if (ev) cudaEventDestroy(ev);
  for (int nn = 0; nn < kMaxNodes; ++nn)
    if (hc_peer_[nn]) {
      cudaHostUnregister(hc_peer_[nn]->base());
      hc_peer_[nn].reset();
    }
  if (hc_own_) {
    cudaHostUnregister(hc_own_->base());
    hc_own_.reset();
  } else if (host_cache_) {
    cudaHostUnregister(host_cache_);
    munmap(host_cache_, host_cache_map_bytes_);
  }
  if (shm_) cudaHostUnregister(shm_->base());
  shm_.reset();
}

// ------------------------------------------------------------------- setup

void Engine::build_layouts(const std::uint8_t* const* masks) {
  const int L = model_.num_layers();
  layers_.resize(static_cast<std::size_t>(L));
  const int r = j_ * Ns_ + ns_;  // shard index of this GPU in its sharding scope
  for (int l = 0; l < L; ++l) {
    LayerRt& lr = layers_[l];
    const std::int64_t E = model_.layers[l].param_count;
    if ((E * eb_) % kChunkBytes != 0)
      throw shardsim::ConfigError("layer " + std::to_string(l) + ": " + std::to_string(E) +
                                  " params is not a whole number of 16-byte chunks");
    lr.elems = E;
    lr.chunks = E * eb_ / kChunkBytes;
    const std::int64_t trainable = shardsim::layer_trainable_params(model_.layers[l]);
    std::vector<std::uint8_t> derived;
    const std::uint8_t* mask = masks ? masks[l] : nullptr;
    if (!mask) {
      if ((trainable * eb_) % kChunkBytes != 0)
        throw shardsim::ConfigError("layer " + std::to_string(l) +
                                    ": trainable_fraction does not select whole 16-byte chunks; pass a chunk mask");
      derived.assign(static_cast<std::size_t>(lr.chunks), 0);
      std::fill_n(derived.begin(), trainable * eb_ / kChunkBytes, 1);
      mask = derived.data();
    }
    lr.L = build_layout(lr.chunks, mask, eb_, Ns_, g_);
    if (lr.L.dev.pt * V_ != trainable)
      throw shardsim::ConfigError("layer " + std::to_string(l) + ": chunk mask selects " +
                                  std::to_string(lr.L.dev.pt * V_) + " trainable params, trainable_fraction gives " +
                                  std::to_string(trainable));
    const std::size_t wb = lr.L.bits.size() * sizeof(std::uint32_t);
    const std::size_t tw = lr.L.sparse_t() ? lr.L.twords.size() * sizeof(std::uint32_t) : 0;
    CK(cudaMalloc(&lr.d_bits, wb));
    CK(cudaMalloc(&lr.d_tpre, wb + tw));  // prefix, then the active trainable words (sparse masks)
    CK(cudaMemcpy(lr.d_bits, lr.L.bits.data(), wb, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lr.d_tpre, lr.L.tpre.data(), wb, cudaMemcpyHostToDevice));
    lr.L.dev.bits = lr.d_bits;
    lr.L.dev.tpre = lr.d_tpre;
    if (tw) {
      CK(cudaMemcpy(lr.d_tpre + lr.L.bits.size(), lr.L.twords.data(), tw, cudaMemcpyHostToDevice));
      lr.L.dev.twords = lr.d_tpre + lr.L.bits.size();
      lr.L.dev.ntwords = static_cast<std::int64_t>(lr.L.twords.size());
    }
    lr.has_t = lr.L.dev.pt > 0;
    lr.has_f = lr.L.dev.pf > 0;
    lr.off_t = arena_t_;
    arena_t_ += lr.L.dev.shard_t;
    lr.off_f = arena_f_;
    arena_f_ += lr.L.dev.shard_f;
    lr.host_off = host_chunks_;
    host_chunks_ += lr.L.dev.slice_t + lr.L.dev.slice_f;
    lr.my_real_t = lr.L.real_chunks(false, r);
    lr.my_real_f = lr.L.real_chunks(true, r);
    lr.slice_real_t = lr.L.real_slice_chunks(false, j_);
    lr.slice_real_f = lr.L.real_slice_chunks(true, j_);
    max_chunks_ = std::max(max_chunks_, lr.chunks);
    max_slice_ = std::max(max_slice_, lr.L.dev.slice_t + lr.L.dev.slice_f);
    max_shard_t_ = std::max(max_shard_t_, lr.L.dev.shard_t);
    max_slice_t_ = std::max(max_slice_t_, lr.L.dev.slice_t);
  }
  pending_h2d_.assign(static_cast<std::size_t>(L), {});
  x_of_t_.assign(static_cast<std::size_t>(L), -1);
  x_of_f_.assign(static_cast<std::size_t>(L), -1);
  w_of_layer_.assign(static_cast<std::size_t>(L), -1);
  grad_slot_of_layer_.assign(static_cast<std::size_t>(L), -1);
  u_of_layer_.assign(static_cast<std::size_t>(L), 0);
  retained_.assign(static_cast<std::size_t>(L), nullptr);
  retained_content_.assign(static_cast<std::size_t>(L), {});
}

void Engine::allocate() {
  const std::size_t C = kChunkBytes;
  param_t_ = dalloc<unsigned char>(arena_t_ * C, "trainable shards");
  param_f_ = dalloc<unsigned char>(arena_f_ * C, "frozen shards");
  const std::size_t nt = static_cast<std::size_t>(arena_t_) * V_ * sizeof(float);
  master_ = dalloc<float>(nt, "fp32 master");
  adam_m_ = dalloc<float>(nt, "adam m");
  adam_v_ = dalloc<float>(nt, "adam v");
  grad32_ = dalloc<float>(nt, "fp32 grad shards");
  for (auto& w : w_slots_) w = dalloc<unsigned char>(max_chunks_ * C, "gathered layer");
  x_slot_bytes_ = round_up(static_cast<std::size_t>(max_slice_) * C, 4096);
  grad_slot_bytes_ = round_up(static_cast<std::size_t>(max_chunks_) * C, 4096);
  arena_bytes_ = x_slot_bytes_ * cfg_.x_slots + 2 * grad_slot_bytes_;
  // ZeRO++ keeps this GPU's intra slice of every gathered layer in HBM (the
  // node-level secondary partition, W/g per GPU; reference strategy.cpp:107-108)
  replica_off_ = arena_bytes_;
  if (zeropp_) arena_bytes_ += round_up(static_cast<std::size_t>(host_chunks_) * C, 4096);
  peer_arena_ = dalloc<unsigned char>(arena_bytes_, "peer arena");
  for (int i = 0; i < 2; ++i) {
    own32_[i] = dalloc<float>(static_cast<std::size_t>(max_shard_t_) * V_ * sizeof(float), "rs own");
    wire_[i] = dalloc<unsigned char>(max_slice_t_ * C, "rs wire");
    rx_[i] = dalloc<unsigned char>(static_cast<std::size_t>(N_) * max_shard_t_ * C, "rs rx");
  }
  shared_cache_ = N_ > 1 && (plan_.kind == shardsim::StrategyKind::Fcdp || plan_.kind == shardsim::StrategyKind::FcdpComm);
  if (shared_cache_) {
    hc_own_ = std::make_unique<ShmSegment>(shm_name_ + "_hc" + std::to_string(rank_), host_chunks_ * C, true,
                                           cfg_.timeout_s);
    host_cache_ = hc_own_->base();
  } else {
    host_cache_map_bytes_ = std::max<std::size_t>(host_chunks_ * C, 4096);
    void* p = mmap(nullptr, host_cache_map_bytes_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) {
      host_cache_map_bytes_ = 0;
      throw OomError("mmap(host cache, " + std::to_string(host_chunks_ * C) + " B) failed");
    }
    host_cache_ = static_cast<unsigned char*>(p);
  }
  const std::size_t hc_bytes = hc_own_ ? hc_own_->bytes() : host_cache_map_bytes_;
  if (numa_.cpus_bound && numa_prefer(host_cache_, hc_bytes, numa_.gpu_node)) numa_.bytes_bound += hc_bytes;
  std::memset(host_cache_, 0, host_chunks_ * C);  // first touch: pages land on the preferred node
  {
    const cudaError_t e = cudaHostRegister(host_cache_, hc_bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw OomError("cudaHostRegister(host cache, " + std::to_string(hc_bytes) + " B) failed");
    }
  }
  hc_base_[n_] = host_cache_;
  const std::size_t L = layers_.size();
  cache_stage_t_.assign(L, 0);
  cache_stage_f_.assign(L, 0);
  cache_last_id_t_.assign(L, 0);
  cache_last_id_f_.assign(L, 0);
  cache_staged_.assign(L, nullptr);
  for (auto& ev : cache_staged_) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  ag_staged_.assign(L, nullptr);
  for (auto& ev : ag_staged_) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  ag_staged_valid_.assign(L, 0);
  stepped_.assign(L, 0);
  prev_retained_.assign(L, 0);
  grad_segs_.assign(L, GradSegs{});
  grad_segs_set_.assign(L, 0);
  d2h_done_.assign(L, nullptr);
  for (auto& ev : d2h_done_) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  d2h_done_valid_.assign(L, 0);
  {
    const char* e = std::getenv("FCDP_DEFER_D2H");
    defer_d2h_ = !(e && std::strcmp(e, "0") == 0);
  }
}

void Engine::exchange_handles() {
  RankBlock& mine = shm_->rank_block(rank_);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, peer_arena_));
  static_assert(sizeof(h) <= sizeof(mine.ipc_handle), "ipc handle size");
  std::memcpy(mine.ipc_handle, &h, sizeof(h));
  mine.arena_bytes = arena_bytes_;
  mine.device = cfg_.device;
  shm_->barrier(cfg_.timeout_s);
  for (int jj = 0; jj < g_; ++jj) {
    if (jj == j_) {
      peer_base_[jj] = peer_arena_;
      continue;
    }
    const RankBlock& pb = shm_->rank_block(n_ * g_ + jj);
    if (pb.arena_bytes != arena_bytes_) throw shardsim::ConfigError("engine: ranks disagree on arena size");
    cudaIpcMemHandle_t ph;
    std::memcpy(&ph, pb.ipc_handle, sizeof(ph));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess));
    peer_base_[jj] = static_cast<unsigned char*>(p);
  }
  if (shared_cache_)
    for (int nn = 0; nn < N_; ++nn) {
      if (nn == n_) continue;
      hc_peer_[nn] = std::make_unique<ShmSegment>(shm_name_ + "_hc" + std::to_string(nn * g_ + j_),
                                                  host_chunks_ * kChunkBytes, false, cfg_.timeout_s);
      hc_base_[nn] = hc_peer_[nn]->base();
      CK(cudaHostRegister(hc_base_[nn], hc_peer_[nn]->bytes(), cudaHostRegisterPortable));
    }
}

void Engine::init_params(std::uint64_t seed, const fcdp_init_range* const* ranges, const int32_t* num_ranges) {
  const std::size_t C = kChunkBytes;
  cudaStream_t s = s_comp_;
  unsigned char* nat = dalloc<unsigned char>(max_chunks_ * C, "init natural");
  std::int64_t max_t = 0, max_f = 0;
  for (const LayerRt& l : layers_) {
    max_t = std::max(max_t, l.L.dev.shard_t * Ns_ * g_);
    max_f = std::max(max_f, l.L.dev.shard_f * Ns_ * g_);
  }
  unsigned char* tv = dalloc<unsigned char>(max_t * C, "init t");
  unsigned char* fv = dalloc<unsigned char>(max_f * C, "init f");
  InitRange* d_ranges = nullptr;
  int max_r = 1;
  for (std::size_t l = 0; l < layers_.size(); ++l) max_r = std::max(max_r, num_ranges ? num_ranges[l] : 0);
  d_ranges = dalloc<InitRange>(sizeof(InitRange) * max_r, "init ranges");
  const int r = j_ * Ns_ + ns_;
  try {
    for (std::size_t li = 0; li < layers_.size(); ++li) {
      LayerRt& l = layers_[li];
      const int nr = num_ranges ? num_ranges[li] : 0;
      if (nr > 0) CK(cudaMemcpy(d_ranges, ranges[li], sizeof(InitRange) * nr, cudaMemcpyHostToDevice));
      CK(launch_init_natural(l.elems, eb_, seed, static_cast<int>(li), d_ranges, nr, nat, s));
      CK(cudaMemsetAsync(tv, 0, l.L.dev.shard_t * Ns_ * g_ * C, s));
      CK(cudaMemsetAsync(fv, 0, l.L.dev.shard_f * Ns_ * g_ * C, s));
      CK(launch_partition(l.L, nat, tv, fv, s));
      if (l.has_t)
        CK(cudaMemcpyAsync(param_t_ + l.off_t * C, tv + r * l.L.dev.shard_t * C, l.L.dev.shard_t * C,
                           cudaMemcpyDeviceToDevice, s));
      if (l.has_f)
        CK(cudaMemcpyAsync(param_f_ + l.off_f * C, fv + r * l.L.dev.shard_f * C, l.L.dev.shard_f * C,
                           cudaMemcpyDeviceToDevice, s));
      l.shard_version_t = 0;
      l.host_version_t = l.host_version_f = -1;
      CK(cudaStreamSynchronize(s));
    }
    CK(launch_widen(arena_t_ * V_, param_t_, eb_, master_, s));
    CK(cudaMemsetAsync(adam_m_, 0, arena_t_ * V_ * sizeof(float), s));
    CK(cudaMemsetAsync(adam_v_, 0, arena_t_ * V_ * sizeof(float), s));
    CK(cudaMemsetAsync(grad32_, 0, arena_t_ * V_ * sizeof(float), s));
    CK(cudaStreamSynchronize(s));
  } catch (...) {
    cudaFree(nat);
    cudaFree(tv);
    cudaFree(fv);
    cudaFree(d_ranges);
    throw;
  }
  cudaFree(nat);
  cudaFree(tv);
  cudaFree(fv);
  cudaFree(d_ranges);
  opt_steps_ = 0;
}

// ----------------------------------------------------------------- helpers

unsigned char* Engine::x_slot(int jj, int slot) const { return peer_base_[jj] + slot * x_slot_bytes_; }

unsigned char* Engine::replica(int jj, int layer) const {
  return peer_base_[jj] + replica_off_ + layers_[layer].host_off * kChunkBytes;
}

unsigned char* Engine::grad_slot(int jj, int slot) const {
  return peer_base_[jj] + cfg_.x_slots * x_slot_bytes_ + slot * grad_slot_bytes_;
}

void Engine::wait_flag(cudaStream_t s, int rank, Flag f, std::uint32_t v) {
  shm_->await_posted(rank, f, v, cfg_.timeout_s);
  const auto off = reinterpret_cast<const volatile unsigned char*>(shm_->flag(rank, f)) -
                   static_cast<const volatile unsigned char*>(shm_->base());
  StreamOps::wait_geq(s, reinterpret_cast<const volatile std::uint32_t*>(
                             static_cast<const unsigned char*>(shm_dev_base_) + off), v);
}

void Engine::write_flag(cudaStream_t s, Flag f, std::uint32_t v) {
  const auto off = reinterpret_cast<unsigned char*>(const_cast<std::uint32_t*>(shm_->flag(rank_, f))) -
                   static_cast<unsigned char*>(shm_->base());
  StreamOps::write(s, reinterpret_cast<volatile std::uint32_t*>(static_cast<unsigned char*>(shm_dev_base_) + off), v);
  shm_->post(rank_, f, v);
}

cudaStream_t Engine::stream_for(EventKind k) const {
  switch (k) {
    case EventKind::AgInter:
    case EventKind::AgIntra:
    case EventKind::H2D:
      return s_gather_;
    case EventKind::D2H:
      return s_cache_;
    case EventKind::ReduceScatter:
      return rs_stream();
    default:
      return s_comp_;
  }
}

unsigned char* Engine::w_buffer(int layer) {
  if (w_of_layer_[layer] < 0) {
    if (prog_->layer_retained[layer]) {
      if (!retained_[layer]) {
        // stream-ordered allocation: no host synchronisation inside run()
        void* p = nullptr;
        const std::size_t bytes = static_cast<std::size_t>(layers_[layer].chunks) * kChunkBytes;
        const cudaError_t e = cudaMallocAsync(&p, bytes, s_gather_);
        if (e != cudaSuccess) {
          cudaGetLastError();
          throw OomError("cudaMallocAsync(retained layer) failed: " + std::string(cudaGetErrorString(e)));
        }
        retained_[layer] = static_cast<unsigned char*>(p);
      }
      w_of_layer_[layer] = 2;  // marker: retained buffer
    } else {
      w_of_layer_[layer] = static_cast<int>(w_instances_++ % 2);
    }
  }
  return w_of_layer_[layer] == 2 ? retained_[layer] : w_slots_[w_of_layer_[layer]];
}

int Engine::begin_slice_fill(int /*layer*/) {
  const std::uint32_t q = ++q_;
  const int slot = static_cast<int>(q % static_cast<std::uint32_t>(cfg_.x_slots));
  if (q > static_cast<std::uint32_t>(cfg_.x_slots))
    for (int jj = 0; jj < g_; ++jj)
      if (jj != j_) wait_flag(s_gather_, n_ * g_ + jj, kSliceFree, q - cfg_.x_slots);
  CK(cudaStreamWaitEvent(s_gather_, x_reader_[slot], 0));
  return slot;
}

void Engine::finish_slice_fill(int /*slot*/, std::uint32_t q) { write_flag(s_gather_, kSliceReady, q); }

void Engine::pull_expand(int layer, int slot, std::uint32_t q, bool want_t, bool want_f, cudaStream_t s) {
  LayerRt& l = layers_[layer];
  for (int jj = 0; jj < g_; ++jj)
    if (jj != j_) wait_flag(s, n_ * g_ + jj, kSliceReady, q);
  unsigned char* W = w_buffer(layer);
  SlicePtrs ts{}, fs{};
  for (int jj = 0; jj < g_; ++jj) {
    ts.p[jj] = x_slot(jj, slot);
    fs.p[jj] = x_slot(jj, slot) + l.L.dev.slice_t * kChunkBytes;
  }
  const int set = want_t && want_f ? kSetAll : (want_t ? kSetTrainable : kSetFrozen);
  std::uint64_t rx = 0;  // bytes this GPU pulls from its NVLink peers
  for (int jj = 0; jj < g_; ++jj) {
    if (jj == j_) continue;
    if (want_t) rx += l.L.real_slice_chunks(false, jj) * kChunkBytes;
    if (want_f) rx += l.L.real_slice_chunks(true, jj) * kChunkBytes;
  }
  const bool dense = l.L.dense_trainable() || l.L.dense_frozen();
  if (use_ce_ && dense) {
    const bool tr = l.L.dense_trainable();
    const std::int64_t per = tr ? l.L.dev.slice_t : l.L.dev.slice_f;
    for (int jj = 0; jj < g_; ++jj) {
      const std::int64_t lo = jj * per;
      if (lo >= l.chunks) break;
      const std::int64_t n = std::min(per, l.chunks - lo);
      CK(cudaMemcpyAsync(W + lo * kChunkBytes, tr ? ts.p[jj] : fs.p[jj], n * kChunkBytes,
                         cudaMemcpyDeviceToDevice, s));
    }
  } else {
    std::uint64_t out_bytes = 0;
    if (want_t) out_bytes += l.L.dev.pt * kChunkBytes;
    if (want_f) out_bytes += l.L.dev.pf * kChunkBytes;
    timed(0, s, 2 * out_bytes, [&] { return launch_expand(l.L, ts, fs, W, set, s); }, rx);
  }
  write_flag(s, kSliceFree, q);
  shm_->add(rank_, kNvlinkRx, rx);
}

std::int64_t Engine::pieces_of(std::size_t bytes) const {
  const std::size_t ch = static_cast<std::size_t>(chunk_bytes_);
  return bytes == 0 ? 0 : static_cast<std::int64_t>((bytes + ch - 1) / ch);
}

void Engine::stage_one(int cls, cudaStream_t s, const void* src, std::size_t n, std::uint64_t wire_mult,
                       Counter counter, unsigned char* host_dst) {
  // Pipelined host-staged wire: the piece is staged into the next slot of
  // this rank's ring, flagged, and handed to the NIC thread, which puts it on
  // the emulated wire as soon as it lands.  A ring slot is reused only once
  // every receiver has marked the piece it held as consumed.
  const std::uint32_t ring = static_cast<std::uint32_t>(cfg_.inter_slots);
  const Flag consumed = static_cast<Flag>((cls == 0 ? kAgConsumed0 : kRsConsumed0) + n_);
  const std::uint32_t id = ++sent_pieces_[cls];
  if (id > ring)
    for (int nn = 0; nn < N_; ++nn)
      if (nn != n_) wait_flag(s, nn * g_ + j_, consumed, id - ring);
  unsigned char* dst = host_dst ? host_dst : shm_->slot(rank_, cls, static_cast<int>(id % ring));
  timed(7, s, n, [&] { return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s); }, n);
  write_flag(s, cls == 0 ? kAgStaged : kRsStaged, id);
  nic_->submit({cls, id, n * wire_mult, counter});
  shm_->post(rank_, cls == 0 ? kAgTxReady : kRsTxReady, id);
  shm_->add(rank_, kStagingD2H, n);
}

void Engine::mark_consumed(int cls, cudaStream_t s, int src_node, std::uint32_t id) {
  std::uint32_t& last = consumed_[cls][src_node];
  if (static_cast<std::int32_t>(id - last) <= 0) return;  // monotone
  last = id;
  write_flag(s, static_cast<Flag>((cls == 0 ? kAgConsumed0 : kRsConsumed0) + src_node), id);
}

void Engine::exchange(int cls, cudaStream_t send_s, const std::vector<SendSeg>& mine, std::uint64_t wire_mult,
                      Counter counter, cudaStream_t recv_s, const std::vector<Inbound>& inbound) {
  // Host enqueue order interleaves my k-th outgoing piece with every sender's
  // k-th incoming piece.  A rank that must wait (host side) for a receiver to
  // post consumption of its piece k - ring therefore never waits on a peer
  // host that is itself stuck before enqueuing that receive: every rank posts
  // piece k's consumption before it stages piece k + ring.
  const std::size_t ch = static_cast<std::size_t>(chunk_bytes_);
  const std::uint32_t ring = static_cast<std::uint32_t>(cfg_.inter_slots);
  struct P {
    const unsigned char* src;
    std::size_t n;
    unsigned char* host_dst;
  };
  std::vector<P> out;
  for (const SendSeg& sg : mine)
    for (std::size_t off = 0; off < sg.bytes; off += ch)
      out.push_back({static_cast<const unsigned char*>(sg.src) + off, std::min(ch, sg.bytes - off),
                     sg.host_dst ? sg.host_dst + off : nullptr});
  struct RP {
    std::size_t n;
    unsigned char* dst;             // null: not ours
    const unsigned char* host_src;  // null: the sender's ring slot
  };
  struct R {
    int src_rank;
    std::uint32_t first;
    std::vector<RP> pieces;
  };
  std::vector<R> in;
  std::size_t kmax = out.size();
  for (const Inbound& ib : inbound) {
    R r{ib.src_rank, recv_base_[cls][ib.src_rank] + 1, {}};
    for (const InSeg& sg : ib.segs)
      for (std::size_t off = 0; off < sg.bytes; off += ch)
        r.pieces.push_back({std::min(ch, sg.bytes - off), sg.dst ? sg.dst + off : nullptr,
                            sg.host_src ? sg.host_src + off : nullptr});
    recv_base_[cls][ib.src_rank] += static_cast<std::uint32_t>(r.pieces.size());
    kmax = std::max(kmax, r.pieces.size());
    in.push_back(std::move(r));
  }
  std::uint64_t rx = 0;
  for (std::size_t k = 0; k < kmax; ++k) {
    if (k < out.size()) stage_one(cls, send_s, out[k].src, out[k].n, wire_mult, counter, out[k].host_dst);
    for (R& r : in) {
      if (k >= r.pieces.size()) continue;
      const std::uint32_t id = r.first + static_cast<std::uint32_t>(k);
      const RP& pc = r.pieces[k];
      const std::size_t n = pc.n;
      unsigned char* dst = pc.dst;
      if (dst) {
        wait_flag(recv_s, r.src_rank, cls == 0 ? kAgTxReady : kRsTxReady, id);
        const unsigned char* src = pc.host_src ? pc.host_src : shm_->slot(r.src_rank, cls, static_cast<int>(id % ring));
        timed(8, recv_s, n, [&] { return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, recv_s); }, n);
        rx += n;
      }
      mark_consumed(cls, recv_s, r.src_rank / g_, id);  // read it, or it was never ours to read
    }
  }
  shm_->add(rank_, kStagingH2D, rx);
}

// ------------------------------------------------------------------ events

bool Engine::alias_gather(const Event& e, bool wt, bool wf) {
  // One GPU holding the whole model (G = 1) and a single-portion layer (dense
  // trainable, or frozen-only): the shard IS the natural layer, so the gather
  // is the identity and compute reads the shard in place - no copy.
  static const char* env = std::getenv("FCDP_ALIAS");
  if (G_ != 1 || zeropp_ || (env && std::strcmp(env, "0") == 0)) return false;
  LayerRt& l = layers_[e.layer];
  if (!((wt && !l.has_f) || (wf && !l.has_t))) return false;
  w_of_layer_[e.layer] = kAliasW;
  if (wt) x_of_t_[e.layer] = kAliasX;
  if (wf) x_of_f_[e.layer] = kAliasX;
  alias_used_ = true;
  return true;
}

unsigned char* Engine::alias_ptr(int li) const {
  const LayerRt& l = layers_[li];
  return l.has_t ? param_t_ + l.off_t * kChunkBytes : param_f_ + l.off_f * kChunkBytes;
}

void Engine::fence_alias_reads(cudaStream_t s, int layer) {
  // FCDP-Cache D2H of an aliased layer reads the shard that AdamW rewrites
  if (!alias_used_) return;
  if (layer >= 0) {  // only that layer's store reads that layer's shard
    if (d2h_done_valid_[layer]) CK(cudaStreamWaitEvent(s, d2h_done_[layer], 0));
    return;
  }
  CK(cudaEventRecord(alias_fence_, s_cache_));
  CK(cudaStreamWaitEvent(s, alias_fence_, 0));
}

void Engine::ev_ag_inter(const Event& e, bool backward) {
  // FCDP's backward reconstructs from the host cache + intra-node gather and
  // issues no inter-node all-gather; ZeRO++
  // gathers from its GPU replicas.  An executed program that does is rejected.
  if (backward && !mics_ &&
      (plan_.kind == shardsim::StrategyKind::Fcdp || plan_.kind == shardsim::StrategyKind::FcdpComm || zeropp_))
    throw shardsim::ProtocolError("zero_bwd_ag_inter: backward AgInter of layer " + std::to_string(e.layer) + " in a " +
                                  shardsim::to_string(plan_.kind) + " program");
  LayerRt& l = layers_[e.layer];
  const bool wt = wants_t(e.param_set) && l.has_t, wf = wants_f(e.param_set) && l.has_f;
  if (alias_gather(e, wt, wf)) {
    if (!mics_) shm_->add(rank_, backward ? kAgEventsBwd : kAgEventsFwd, 1);
    return;
  }
  cudaStream_t s = s_gather_;
  const std::size_t C = kChunkBytes;
  const int slot = begin_slice_fill(e.layer);
  const std::uint32_t q = q_;
  unsigned char* X = x_slot(j_, slot);
  unsigned char* Xf = X + l.L.dev.slice_t * C;
  // own shard -> its position n in this GPU's slice (global shard j*N + n)
  // (an SM copy, not cudaMemcpy: the copy engines are busy with FCDP-Cache D2H
  //  and host-staged NIC traffic, and a D2D queued behind them stalls the gather)
  if (wt && l.my_real_t)
    timed(4, s, 2 * l.my_real_t * C, [&] {
      return launch_copy(param_t_ + l.off_t * C, X + ns_ * l.L.dev.shard_t * C, l.my_real_t * C, s);
    });
  if (wf && l.my_real_f)
    timed(4, s, 2 * l.my_real_f * C, [&] {
      return launch_copy(param_f_ + l.off_f * C, Xf + ns_ * l.L.dev.shard_f * C, l.my_real_f * C, s);
    });
  if (Ns_ > 1) {
    // Inter-node all-gather among {(n', j)} through the host-staged NIC path,
    // pipelined in pieces of chunk_bytes_.  Staging runs on s_agsend_ (which
    // already waited on this event's deps in run()), so the receive side below
    // overlaps with it.
    const std::size_t bt = wt ? l.my_real_t * C : 0, bf = wf ? l.my_real_f * C : 0;
    // Write-once staging: portions the forward FCDP-Cache will store are staged
    // straight into their host-cache position (slice j, shard n) and served to
    // the wire from there.
    const bool ct = !backward && wt && cache_stage_t_[e.layer], cf = !backward && wf && cache_stage_f_[e.layer];
    const std::size_t t_off = (l.host_off + n_ * l.L.dev.shard_t) * C;
    const std::size_t f_off = (l.host_off + l.L.dev.slice_t + n_ * l.L.dev.shard_f) * C;
    if (ct || cf) {
      // WAR: receivers must be done with last iteration's pieces from this region
      const std::uint32_t last = std::max(ct ? cache_last_id_t_[e.layer] : 0u, cf ? cache_last_id_f_[e.layer] : 0u);
      if (last)
        for (int nn = 0; nn < N_; ++nn)
          if (nn != n_) wait_flag(s_agsend_, nn * g_ + j_, static_cast<Flag>(kAgConsumed0 + n_), last);
    }
    std::vector<Inbound> inbound;
    std::uint64_t rx = 0;
    for (int nn = 0; nn < N_; ++nn) {
      if (nn == n_) continue;
      const int r = j_ * N_ + nn;
      const std::size_t rt = wt ? l.L.real_chunks(false, r) * C : 0, rf = wf ? l.L.real_chunks(true, r) * C : 0;
      const unsigned char* hb = hc_base_[nn];
      inbound.push_back({nn * g_ + j_,
                         {{rt, X + nn * l.L.dev.shard_t * C,
                           ct ? hb + (l.host_off + nn * l.L.dev.shard_t) * C : nullptr},
                          {rf, Xf + nn * l.L.dev.shard_f * C,
                           cf ? hb + (l.host_off + l.L.dev.slice_t + nn * l.L.dev.shard_f) * C : nullptr}}});
      rx += rt + rf;
    }
    const std::uint32_t first_id = sent_pieces_[0] + 1;
    exchange(0, s_agsend_,
             {{param_t_ + l.off_t * C, bt, ct ? host_cache_ + t_off : nullptr},
              {param_f_ + l.off_f * C, bf, cf ? host_cache_ + f_off : nullptr}},
             N_ - 1, backward ? kTxBwdAg : kTxFwdAg, s, inbound);
    CK(cudaEventRecord(ag_staged_[e.layer], s_agsend_));
    ag_staged_valid_[e.layer] = 1;
    if (ct || cf) {
      const std::uint32_t pt = static_cast<std::uint32_t>(pieces_of(bt));
      if (ct) cache_last_id_t_[e.layer] = first_id + pt - 1;
      if (cf) cache_last_id_f_[e.layer] = sent_pieces_[0];
      CK(cudaEventRecord(cache_staged_[e.layer], s_agsend_));
    }
    shm_->add(rank_, backward ? kRxBwdAg : kRxFwdAg, rx);
  }
  finish_slice_fill(slot, q);
  // Intra-node all-gather over NVLink, fused with the PEFT expansion.
  pull_expand(e.layer, slot, q, wt, wf, s);
  WContent& wc = w_of_layer_[e.layer] == 2 ? retained_content_[e.layer] : w_content_[w_of_layer_[e.layer]];
  if (wc.layer != e.layer) wc = WContent{e.layer, -1, -1};
  if (wt) wc.ver_t = static_cast<std::int64_t>(l.shard_version_t), x_of_t_[e.layer] = slot;
  if (wf) wc.ver_f = 0, x_of_f_[e.layer] = slot;
  if (!mics_) shm_->add(rank_, backward ? kAgEventsBwd : kAgEventsFwd, 1);
  if (zeropp_ && !backward) {
    // keep slice j on the GPU for the backward intra-node gather (ZeRO++ hpZ)
    if (l.last_replica_pull_q)
      for (int jj = 0; jj < g_; ++jj)
        if (jj != j_) wait_flag(s, n_ * g_ + jj, kSliceFree, l.last_replica_pull_q);
    const std::size_t bytes = (l.L.dev.slice_t + l.L.dev.slice_f) * C;
    timed(4, s, 2 * bytes, [&] { return launch_copy(X, replica(j_, e.layer), bytes, s); });
    l.replica_version_t = static_cast<std::int64_t>(l.shard_version_t);
  }
}

void Engine::ev_h2d(const Event& e) {
  LayerRt& l = layers_[e.layer];
  const bool wt = wants_t(e.param_set) && l.has_t, wf = wants_f(e.param_set) && l.has_f;
  // Freshness (Algorithm 1 line 10): only a clean host copy may be reloaded.
  if (wt && l.host_version_t != static_cast<std::int64_t>(l.shard_version_t))
    throw shardsim::ProtocolError("freshness: layer " + std::to_string(e.layer) +
                                  " trainable portion reloaded from a stale host cache");
  if (wf && l.host_version_f != 0)
    throw shardsim::ProtocolError("freshness: layer " + std::to_string(e.layer) +
                                  " frozen portion reloaded before it was cached");
  // Frozen residency: a tau-retained layer whose retained buffer already holds
  // the frozen portion (version 0 forever) needs no reload -
  // the event's postcondition already holds.  Trainable data always moves.
  // At G = 1 a frozen-only layer retained in this and the previous iteration is
  // resident as the shard itself (read in place, see alias_gather).
  static const char* alias_env = std::getenv("FCDP_ALIAS");
  const bool alias_resident = !wt && wf && !l.has_t && G_ == 1 && !zeropp_ &&
                              !(alias_env && std::strcmp(alias_env, "0") == 0) &&
                              prog_->layer_retained[e.layer] && prev_retained_[e.layer];
  if (alias_resident || (!wt && wf && prog_->layer_retained[e.layer] && retained_[e.layer] &&
                         retained_content_[e.layer].layer == e.layer && retained_content_[e.layer].ver_f == 0)) {
    PendingSlice& p = pending_h2d_[e.layer];
    p.slot = kElided;
    p.alias = alias_resident;
    p.t = false;
    p.f = true;
    p.ver_f = 0;
    shm_->add(rank_, kResidentHits, 1);
    return;
  }
  const std::size_t C = kChunkBytes;
  const int slot = begin_slice_fill(e.layer);
  const std::uint32_t q = q_;
  unsigned char* X = x_slot(j_, slot);
  const unsigned char* H = host_cache_ + l.host_off * C;
  std::uint64_t bytes = 0;
  if (wt && l.slice_real_t) {
    const std::size_t b = l.slice_real_t * C;
    timed(6, s_gather_, b, [&] { return cudaMemcpyAsync(X, H, b, cudaMemcpyHostToDevice, s_gather_); }, b);
    bytes += l.slice_real_t * C;
  }
  if (wf && l.slice_real_f) {
    const std::size_t b = l.slice_real_f * C;
    timed(6, s_gather_, b, [&] {
      return cudaMemcpyAsync(X + l.L.dev.slice_t * C, H + l.L.dev.slice_t * C, b, cudaMemcpyHostToDevice, s_gather_);
    }, b);
    bytes += l.slice_real_f * C;
  }
  shm_->add(rank_, kCacheH2D, bytes);
  finish_slice_fill(slot, q);
  PendingSlice& p = pending_h2d_[e.layer];
  p.slot = slot;
  p.q = q;
  p.t = wt;
  p.f = wf;
  p.ver_t = wt ? l.host_version_t : -1;
  p.ver_f = wf ? 0 : -1;
}

void Engine::ev_ag_intra(const Event& e, bool backward) {
  if (mics_) {  // MiCS within a node: gather the layer from the node's g shards over NVLink
    ev_ag_inter(e, backward);
    return;
  }
  if (zeropp_) {
    // backward reconstruction from the GPU replicas of the node (no PCIe, no NIC)
    LayerRt& l = layers_[e.layer];
    if (l.has_t && l.replica_version_t != static_cast<std::int64_t>(l.shard_version_t))
      throw shardsim::ProtocolError("freshness: stale GPU replica for layer " + std::to_string(e.layer));
    const std::uint32_t q = ++q_;
    write_flag(s_gather_, kSliceReady, q);
    for (int jj = 0; jj < g_; ++jj)
      if (jj != j_) wait_flag(s_gather_, n_ * g_ + jj, kSliceReady, q);
    unsigned char* W = w_buffer(e.layer);
    SlicePtrs ts{}, fs{};
    for (int jj = 0; jj < g_; ++jj) {
      ts.p[jj] = replica(jj, e.layer);
      fs.p[jj] = replica(jj, e.layer) + l.L.dev.slice_t * kChunkBytes;
    }
    std::uint64_t prx = 0;
    for (int jj = 0; jj < g_; ++jj)
      if (jj != j_) prx += (l.L.real_slice_chunks(false, jj) + l.L.real_slice_chunks(true, jj)) * kChunkBytes;
    timed(0, s_gather_, 2 * l.chunks * kChunkBytes,
          [&] { return launch_expand(l.L, ts, fs, W, kSetAll, s_gather_); }, prx);
    write_flag(s_gather_, kSliceFree, q);
    l.last_replica_pull_q = q;
    std::uint64_t rx = 0;
    for (int jj = 0; jj < g_; ++jj)
      if (jj != j_) rx += (l.L.real_slice_chunks(false, jj) + l.L.real_slice_chunks(true, jj)) * kChunkBytes;
    shm_->add(rank_, kNvlinkRx, rx);
    WContent& wc = w_content_[w_of_layer_[e.layer]];
    wc = WContent{e.layer, l.has_t ? l.replica_version_t : -1, l.has_f ? 0 : -1};
    return;
  }
  PendingSlice p = pending_h2d_[e.layer];
  if (p.slot == kElided) {  // frozen portion already resident in the retained buffer
    if (p.alias) {
      w_of_layer_[e.layer] = kAliasW;
      x_of_f_[e.layer] = kAliasX;
    } else {
      w_buffer(e.layer);
    }
    pending_h2d_[e.layer] = {};
    return;
  }
  if (p.slot < 0) throw shardsim::ProtocolError("ag_intra without a preceding h2d for layer " + std::to_string(e.layer));
  pull_expand(e.layer, p.slot, p.q, p.t, p.f, s_gather_);
  WContent& wc = w_of_layer_[e.layer] == 2 ? retained_content_[e.layer] : w_content_[w_of_layer_[e.layer]];
  if (wc.layer != e.layer) wc = WContent{e.layer, -1, -1};
  if (p.t) wc.ver_t = p.ver_t;
  if (p.f) wc.ver_f = p.ver_f;
  pending_h2d_[e.layer] = {};
}

void Engine::store_d2h(int layer, bool wt, bool wf, int slot_t, int slot_f) {
  LayerRt& l = layers_[layer];
  const std::size_t C = kChunkBytes;
  unsigned char* H = host_cache_ + l.host_off * C;
  // Copy slice j of a portion from X to the host cache; when this GPU's own
  // shard was staged there already (write-once staging), only the peers' shards.
  auto store = [&](bool frozen, int slot) {
    const std::int64_t shard = frozen ? l.L.dev.shard_f : l.L.dev.shard_t;
    const std::size_t base = frozen ? l.L.dev.slice_t * C : 0;
    const unsigned char* Xs = slot == kAliasX ? (frozen ? param_f_ + l.off_f * C : param_t_ + l.off_t * C)
                                              : x_slot(j_, slot) + base;
    const bool own_staged = frozen ? cache_stage_f_[layer] : cache_stage_t_[layer];
    if (!own_staged || N_ == 1) {
      const std::int64_t real = frozen ? l.slice_real_f : l.slice_real_t;
      const std::size_t b = static_cast<std::size_t>(real) * C;
      if (real) timed(5, s_cache_, b, [&] { return cudaMemcpyAsync(H + base, Xs, b, cudaMemcpyDeviceToHost, s_cache_); }, b);
      return;
    }
    for (int m = 0; m < N_; ++m) {
      if (m == n_) continue;
      const std::int64_t real = l.L.real_chunks(frozen, j_ * N_ + m);
      if (real)
        timed(5, s_cache_, static_cast<std::uint64_t>(real) * C, [&] {
          return cudaMemcpyAsync(H + base + m * shard * C, Xs + m * shard * C, real * C, cudaMemcpyDeviceToHost,
                                 s_cache_);
        }, static_cast<std::uint64_t>(real) * C);
    }
  };
  const bool staged_any = (wt && cache_stage_t_[layer]) || (wf && cache_stage_f_[layer]);
  if (staged_any && N_ > 1) CK(cudaStreamWaitEvent(s_cache_, cache_staged_[layer], 0));
  if (wt) store(false, slot_t);
  if (wf) store(true, slot_f);
  for (int sl : {slot_t, slot_f})
    if (sl >= 0) CK(cudaEventRecord(x_reader_[sl], s_cache_));
  CK(cudaEventRecord(d2h_done_[layer], s_cache_));
  d2h_done_valid_[layer] = 1;
}

void Engine::ev_d2h(const Event& e) {
  LayerRt& l = layers_[e.layer];
  const bool wt = wants_t(e.param_set) && l.has_t, wf = wants_f(e.param_set) && l.has_f;
  const std::size_t C = kChunkBytes;
  int slot_t = -1, slot_f = -1;
  std::uint64_t bytes = 0;
  if (wt) {
    slot_t = x_of_t_[e.layer];
    if (slot_t < 0 && slot_t != kAliasX)
      throw shardsim::ProtocolError("d2h of a trainable portion that was not gathered");
    bytes += l.slice_real_t * C;
    l.host_version_t = static_cast<std::int64_t>(l.shard_version_t);
  }
  if (wf) {
    slot_f = x_of_f_[e.layer];
    if (slot_f < 0 && slot_f != kAliasX)
      throw shardsim::ProtocolError("d2h of a frozen portion that was not gathered");
    bytes += l.slice_real_f * C;
    l.host_version_f = 0;
  }
  shm_->add(rank_, kCacheD2H, bytes);
  // One GPU, layer read in place (alias): the store's source is the shard,
  // which only this layer's own update rewrites, after its backward reload.
  // The backward needs the stores last-layer-first, while the program emits
  // them in forward order behind each ComputeFwd (schedule.cpp:209-223); on
  // one copy stream that puts the last layer's store - the first the backward
  // reloads - behind every other (about 50 ms of PCIe for GPT-2 1.3B).  So the
  // stores are queued and issued in reverse at the forward->backward turn (or
  // as soon as anything depends on one): same bytes, same deps, LIFO order.
  const bool alias_src = (!wt || slot_t == kAliasX) && (!wf || slot_f == kAliasX);
  if (defer_d2h_ && G_ == 1 && alias_src) {
    deferred_d2h_.push_back({e.id, e.layer, wt, wf});
    d2h_deferred_id_[e.id] = 1;
    return;
  }
  store_d2h(e.layer, wt, wf, slot_t, slot_f);
}

void Engine::flush_deferred_d2h() {
  for (auto it = deferred_d2h_.rbegin(); it != deferred_d2h_.rend(); ++it) {
    if (trace_) CK(cudaEventRecord(trace_begin_[it->id], s_cache_));
    store_d2h(it->layer, it->t, it->f, it->t ? kAliasX : -1, it->f ? kAliasX : -1);
    CK(cudaEventRecord(ev_done_[it->id], s_cache_));  // dependents enqueued from now on wait for the copy
    if (trace_) CK(cudaEventRecord(trace_end_[it->id], s_cache_));
    d2h_deferred_id_[it->id] = 0;
  }
  deferred_d2h_.clear();
}

void Engine::ev_compute(const Event& e, bool backward) {
  const int li = e.layer;
  LayerRt& l = layers_[li];
  if (w_of_layer_[li] < 0) throw shardsim::ProtocolError("freshness: layer " + std::to_string(li) + " computed without a gather");
  const WContent alias_wc{li, l.has_t ? static_cast<std::int64_t>(l.shard_version_t) : -1, l.has_f ? 0 : -1};
  const WContent& wc = w_of_layer_[li] == kAliasW ? alias_wc
                       : w_of_layer_[li] == 2    ? retained_content_[li]
                                                 : w_content_[w_of_layer_[li]];
  if (wc.layer != li || (l.has_t && wc.ver_t != static_cast<std::int64_t>(l.shard_version_t)) ||
      (l.has_f && wc.ver_f != 0))
    throw shardsim::ProtocolError("freshness: layer " + std::to_string(li) +
                                  " would compute on parameters that are not at their current version");
  unsigned char* W = w_of_layer_[li] == kAliasW ? alias_ptr(li)
                     : w_of_layer_[li] == 2    ? retained_[li]
                                               : w_slots_[w_of_layer_[li]];
  void* grad = nullptr;
  if (backward && l.has_t) {
    const std::uint32_t u = ++u_;
    const int gs = static_cast<int>(u % 2);
    u_of_layer_[li] = u;
    grad_slot_of_layer_[li] = gs;
    if (u > 2) {
      for (int jj = 0; jj < g_; ++jj)
        if (jj != j_) wait_flag(s_comp_, n_ * g_ + jj, kGradFree, u - 2);
      CK(cudaStreamWaitEvent(s_comp_, rs_done_[gs], 0));
    }
    grad = grad_slot(j_, gs);
  }
  if (grad) grad_segs_set_[li] = 0;
  if (compute_fn_) {
    bwd_callback_layer_ = grad ? li : -1;
    const int rc = compute_fn_(compute_user_, backward ? FCDP_EV_COMPUTE_BWD : FCDP_EV_COMPUTE_FWD, li, W, grad,
                               s_comp_);
    bwd_callback_layer_ = -1;
    if (rc != 0) throw std::runtime_error("compute callback failed for layer " + std::to_string(li));
  } else if (grad) {
    CK(cudaMemsetAsync(grad, 0, l.chunks * kChunkBytes, s_comp_));  // data-plane-only mode
  }
  if (grad && !grad_segs_set_[li]) {  // the gradient is in the natural slot
    GradSegs& sg = grad_segs_[li];
    sg.n = 1;
    sg.dst_chunk[0] = 0;
    sg.nchunks[0] = l.chunks;
    sg.src[0] = grad;
  }
  if (!backward && w_of_layer_[li] != 2 && !(w_of_layer_[li] == kAliasW && prog_->layer_retained[li]))
    w_of_layer_[li] = -1;  // the slot is free for the backward re-gather
}

void Engine::ev_reduce_scatter(const Event& e) {
  const int li = e.layer;
  LayerRt& l = layers_[li];
  if (!l.has_t) return;
  const std::uint32_t u = u_of_layer_[li];
  const int gs = grad_slot_of_layer_[li];
  if (gs < 0) throw shardsim::ProtocolError("reduce_scatter before compute_bwd of layer " + std::to_string(li));
  cudaStream_t s = rs_stream();
  const std::size_t C = kChunkBytes;
  write_flag(s, kGradReady, u);
  for (int jj = 0; jj < g_; ++jj)
    if (jj != j_) wait_flag(s, n_ * g_ + jj, kGradReady, u);
  if (N_ > 1) {
    CK(cudaStreamWaitEvent(s, rs_staged_[gs], 0));  // wire/rx [gs] staged out (use u-2)
    CK(cudaStreamWaitEvent(s, fin_done_[gs], 0));   // own32/rx [gs] consumed by epilogue u-2
  }
  GradPtrs gp{};
  for (int jj = 0; jj < g_; ++jj) gp.p[jj] = grad_slot(jj, gs);
  const float scale = 1.0f / static_cast<float>(G_);
  float* final_out = grad32_ + l.off_t * V_;
  if (fused_grad_ok(li)) {
    // G = 1: the RS is the identity up to widen + scale; fused into AdamW,
    // reading the gradient where backward left it (the slot or the segments)
    if (opt_low_ || opt_on_compute_) {
      CK(cudaEventRecord(opt_fork_, s));
      s = opt_on_compute_ ? s_comp_ : s_opt_;
      CK(cudaStreamWaitEvent(s, opt_fork_, 0));
      done_s_ = s;
    }
    fence_alias_reads(s, li);
    const std::int64_t n = l.L.dev.shard_t * V_;
    const std::size_t o = static_cast<std::size_t>(l.off_t) * V_;
    const AdamParams p = adam_params(opt_steps_ + 1);
    const std::uint64_t bytes = static_cast<std::uint64_t>(n) * (6 * sizeof(float) + 2 * eb_ + (keep_grad_ ? 4 : 0));
    timed(3, s, bytes, [&] {
      return launch_adam_grad(l.chunks, grad_segs_[li], p, scale, master_ + o, adam_m_ + o, adam_v_ + o,
                              param_t_ + l.off_t * kChunkBytes, eb_, keep_grad_ ? grad32_ + o : nullptr, s,
                              opt_ctas_per_sm_ * sm_count());
    });
    stepped_[li] = 1;
    write_flag(s, kGradFree, u);
    CK(cudaEventRecord(rs_done_[gs], s));
    grad_slot_of_layer_[li] = -1;
    return;
  }
  // FCDP_RS_CTAS_PER_SM=k caps the RS grid at k CTAs per SM (default 0: the
  // full grid).  Unlike the G = 1 fused update, capping measured no gain at
  // N > 1 (2x1 / 2x2: same step time, lower per-launch rate;
  // profiles/r02_ab_rs_cap.json): the step there is NIC-bound.
  const int rs_blocks = rs_ctas_per_sm_ * sm_count();
  // algorithmic bytes: g gradient slices read + fp32 own shard + dtype wire for the rest
  const std::uint64_t rs_bytes = static_cast<std::uint64_t>(g_) * l.slice_real_t * C +
                                 static_cast<std::uint64_t>(l.my_real_t) * V_ * sizeof(float) +
                                 static_cast<std::uint64_t>(l.slice_real_t - l.my_real_t) * C;
  if (mics_ && N_ > 1) {
    // every contribution (this node's included) in the wire dtype, so all
    // replicas sum identical values in the same order
    timed(1, s, static_cast<std::uint64_t>(g_ + 1) * l.slice_real_t * C, [&] {
      return launch_rs_slice(l.L, gp, j_, -1, scale, false, nullptr, rx_[gs] + n_ * l.L.dev.shard_t * C, s, rs_blocks);
    }, static_cast<std::uint64_t>(g_ - 1) * l.slice_real_t * C);
  } else if (N_ == 1) {
    timed(1, s, rs_bytes, [&] { return launch_rs_slice(l.L, gp, j_, 0, scale, true, final_out, wire_[gs], s, rs_blocks); },
          static_cast<std::uint64_t>(g_ - 1) * l.slice_real_t * C);
  } else {
    timed(1, s, rs_bytes, [&] { return launch_rs_slice(l.L, gp, j_, n_, scale, false, own32_[gs], wire_[gs], s,
                                                       rs_blocks); },
          static_cast<std::uint64_t>(g_ - 1) * l.slice_real_t * C);
  }
  write_flag(s, kGradFree, u);
  CK(cudaEventRecord(rs_done_[gs], s));
  shm_->add(rank_, kNvlinkRx, static_cast<std::uint64_t>(g_ - 1) * l.slice_real_t * C);
  grad_slot_of_layer_[li] = -1;
  if (N_ == 1) {
    if (early_opt_) adam_layer(li, s);
    return;
  }
  if (mics_) {
    mics_grad_sync(l, gs, scale, final_out);
    if (early_opt_) adam_layer(li, s_rsrecv_);
    return;
  }

  // Inter-node reduce-scatter among {(n', j)}: partial sums of the other
  // nodes' shards cross the NIC in the parameter dtype (costmodel.cpp:86-88).
  // staging side (s_rssend_): after this slice's kernel
  CK(cudaEventRecord(rs_kernel_done_[gs], s));
  CK(cudaStreamWaitEvent(s_rssend_, rs_kernel_done_[gs], 0));
  // region m (partials of shard j*N+m) goes to node m only; regions in ascending m
  std::vector<SendSeg> mine;
  for (int nn = 0; nn < N_; ++nn)
    if (nn != n_)
      mine.push_back({wire_[gs] + nn * l.L.dev.shard_t * C, l.L.real_chunks(false, j_ * N_ + nn) * C});
  std::vector<Inbound> inbound;
  std::uint64_t rx = 0;
  for (int nn = 0; nn < N_; ++nn) {
    if (nn == n_) continue;
    Inbound ib{nn * g_ + j_, {}};
    for (int m = 0; m < N_; ++m) {  // sender (nn, j)'s regions; only region n_ is ours
      if (m == nn) continue;
      const std::size_t b = l.L.real_chunks(false, j_ * N_ + m) * C;
      ib.segs.push_back({b, m == n_ ? rx_[gs] + nn * l.L.dev.shard_t * C : nullptr});
      if (m == n_) rx += b;
    }
    inbound.push_back(std::move(ib));
  }
  cudaStream_t r = s_rsrecv_;
  CK(cudaStreamWaitEvent(r, rs_kernel_done_[gs], 0));
  exchange(1, s_rssend_, mine, 1, kTxRs, r, inbound);
  CK(cudaEventRecord(rs_staged_[gs], s_rssend_));  // wire_[gs] may be rewritten after this
  shm_->add(rank_, kRxRs, rx);
  const std::uint64_t fin_elems = static_cast<std::uint64_t>(l.L.dev.shard_t) * V_;
  timed(2, r, fin_elems * (2 * sizeof(float) + static_cast<std::uint64_t>(N_ - 1) * eb_), [&] {
    return launch_rs_finalize(l.L.dev.shard_t * V_, N_, n_, eb_, own32_[gs], rx_[gs], l.L.dev.shard_t * V_, scale,
                              final_out, r);
  });
  CK(cudaEventRecord(fin_done_[gs], r));
  done_s_ = r;
  if (early_opt_) adam_layer(li, r);
}

void Engine::mics_grad_sync(LayerRt& l, int gs, float scale, float* final_out) {
  // MiCS replicas: all-reduce slice j over the N nodes' GPUs j through the
  // NIC path (each sends its whole node-reduced slice to every other node),
  // then one fixed-order sum of the N contributions.  The reference's cost
  // model books no bytes for this sync (costmodel.cpp:39-43, scope = 1 node),
  // so it has its own counter.
  const std::size_t C = kChunkBytes;
  const std::size_t stride = static_cast<std::size_t>(l.L.dev.shard_t) * C;
  CK(cudaEventRecord(rs_kernel_done_[gs], rs_stream()));
  CK(cudaStreamWaitEvent(s_rssend_, rs_kernel_done_[gs], 0));
  cudaStream_t s = s_rsrecv_;
  CK(cudaStreamWaitEvent(s, rs_kernel_done_[gs], 0));
  const std::size_t b = static_cast<std::size_t>(l.slice_real_t) * C;
  std::vector<Inbound> inbound;
  for (int nn = 0; nn < N_; ++nn)
    if (nn != n_) inbound.push_back({nn * g_ + j_, {{b, rx_[gs] + nn * stride}}});
  exchange(1, s_rssend_, {{rx_[gs] + n_ * stride, b}}, N_ - 1, kTxGradSync, s, inbound);
  CK(cudaEventRecord(rs_staged_[gs], s_rssend_));
  shm_->add(rank_, kRxGradSync, static_cast<std::uint64_t>(N_ - 1) * b);
  const std::uint64_t fin_elems = static_cast<std::uint64_t>(l.L.dev.shard_t) * V_;
  timed(2, s, fin_elems * (sizeof(float) + static_cast<std::uint64_t>(N_) * eb_), [&] {
    return launch_rs_finalize(l.L.dev.shard_t * V_, N_, -1, eb_, nullptr, rx_[gs], l.L.dev.shard_t * V_, scale,
                              final_out, s);
  });
  CK(cudaEventRecord(fin_done_[gs], s));
  done_s_ = s;
}

AdamParams Engine::adam_params(int step) const {
  return AdamParams{adam_.lr, adam_.beta1, adam_.beta2, adam_.eps, adam_.weight_decay,
                    static_cast<float>(1.0 - std::pow(static_cast<double>(adam_.beta1), step)),
                    static_cast<float>(1.0 - std::pow(static_cast<double>(adam_.beta2), step))};
}

bool Engine::fused_grad_ok(int li) const {
  static const char* env = std::getenv("FCDP_FUSED_ADAM");
  if (env && std::strcmp(env, "0") == 0) return false;
  const LayerRt& l = layers_.at(li);
  return G_ == 1 && !zeropp_ && !mics_ && l.has_t && !l.has_f && l.L.dense_trainable() &&
         prog_ != nullptr && has_opt_;
}

void Engine::grad_segments(int li, int n, const std::int64_t* offs, const void* const* ptrs,
                           const std::int64_t* counts) {
  if (li != bwd_callback_layer_)
    throw shardsim::ConfigError("grad_segments: only inside the backward compute callback of that layer");
  if (!fused_grad_ok(li))
    throw shardsim::ConfigError("grad_segments: layer " + std::to_string(li) +
                                " needs its gradient in grad_out (segments are taken at G = 1 for dense layers)");
  if (n < 0 || n > kMaxGradSegs) throw shardsim::ConfigError("grad_segments: at most 24 segments");
  const LayerRt& l = layers_[li];
  GradSegs sg;
  sg.n = n;
  std::int64_t prev_end = 0;
  for (int i = 0; i < n; ++i) {
    if (offs[i] % V_ || counts[i] % V_ || reinterpret_cast<std::uintptr_t>(ptrs[i]) % kChunkBytes || counts[i] < 0 ||
        offs[i] < prev_end || offs[i] + counts[i] > l.elems)
      throw shardsim::ConfigError("grad_segments: segment " + std::to_string(i) +
                                  " must be 16-byte aligned, sorted, disjoint and inside the layer");
    sg.dst_chunk[i] = offs[i] / V_;
    sg.nchunks[i] = counts[i] / V_;
    sg.src[i] = ptrs[i];
    prev_end = offs[i] + counts[i];
  }
  grad_segs_[li] = sg;
  grad_segs_set_[li] = 1;
}

void Engine::adam_layer(int li, cudaStream_t s) {
  LayerRt& l = layers_[li];
  const AdamParams p = adam_params(opt_steps_ + 1);  // the step the program's OptimizerStep will complete
  // the own shard must have left for the NIC before it is overwritten
  if (ag_staged_valid_[li]) CK(cudaStreamWaitEvent(s, ag_staged_[li], 0));
  fence_alias_reads(s, li);
  const std::int64_t n = l.L.dev.shard_t * V_;
  const std::size_t o = static_cast<std::size_t>(l.off_t) * V_;
  timed(3, s, static_cast<std::uint64_t>(n) * (7 * sizeof(float) + eb_), [&] {
    return launch_adam(n, p, master_ + o, adam_m_ + o, adam_v_ + o, grad32_ + o, param_t_ + l.off_t * kChunkBytes,
                       eb_, s);
  });
  stepped_[li] = 1;
}

void Engine::ev_optimizer(const Event&) {
  fence_alias_reads(s_comp_);
  bool any_stepped = false;
  for (char c : stepped_) any_stepped |= c != 0;
  if (early_opt_ || any_stepped) {
    for (std::size_t li = 0; li < layers_.size(); ++li)
      if (layers_[li].has_t && !stepped_[li]) adam_layer(static_cast<int>(li), s_comp_);
    ++opt_steps_;
    for (LayerRt& l : layers_)
      if (l.has_t) ++l.shard_version_t;
    return;
  }
  ++opt_steps_;
  AdamParams p{adam_.lr, adam_.beta1, adam_.beta2, adam_.eps, adam_.weight_decay,
               static_cast<float>(1.0 - std::pow(static_cast<double>(adam_.beta1), opt_steps_)),
               static_cast<float>(1.0 - std::pow(static_cast<double>(adam_.beta2), opt_steps_))};
  const std::uint64_t n = static_cast<std::uint64_t>(arena_t_) * V_;
  timed(3, s_comp_, n * (7 * sizeof(float) + eb_),
        [&] { return launch_adam(arena_t_ * V_, p, master_, adam_m_, adam_v_, grad32_, param_t_, eb_, s_comp_); });
  for (LayerRt& l : layers_)
    if (l.has_t) ++l.shard_version_t;
}

// --------------------------------------------------------------------- run

void Engine::run(const shardsim::EventProgram& prog, std::vector<shardsim::ParamState>& states) {
  begin(prog);
  try {
    for (const Event& e : prog.events) exec(e.id);
  } catch (...) {
    prog_ = nullptr;  // the enqueued prefix still drains; the program is abandoned
    throw;
  }
  end(states);
}

void Engine::fail_job() {
  // An error part-way through a program leaves this rank's sequence counters
  // (q_, u_, piece ids) out of step with its peers, so no later program may run
  // on this engine (peers could be satisfied early by stale flag values): latch
  // the failure and raise the job's abort flag so peers blocked on this rank's
  // posts fail fast instead of timing out.
  failed_ = true;
  if (shm_) shm_->header()->abort_flag.store(1);
}

std::uint64_t Engine::program_hash(const shardsim::EventProgram& prog) {
  // FNV-1a over everything that decides the cross-rank sequence numbers: the
  // iteration, the strategy, every event's kind / layer / portion set / deps
  // and the per-layer retention flags.
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&](std::uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  mix(prog.iteration_index);
  mix(static_cast<std::uint64_t>(prog.strategy));
  mix(prog.events.size());
  for (const Event& e : prog.events) {
    mix(static_cast<std::uint64_t>(e.kind) | (static_cast<std::uint64_t>(static_cast<std::uint32_t>(e.layer)) << 8) |
        (static_cast<std::uint64_t>(e.param_set) << 40));
    mix(e.deps.size());
    for (shardsim::EventId d : e.deps) mix(d);
  }
  for (char c : prog.layer_retained) mix(static_cast<std::uint64_t>(c != 0));
  return h;
}

void Engine::check_same_program(const shardsim::EventProgram& prog) {
  // Every rank must walk the same program (sequence numbers agree only then):
  // publish this program's hash, wait for every peer's hash of the same program
  // index and compare (e.g. per-rank gpu_capacity_bytes could make
  // tau retention differ between ranks, which would otherwise read wrong data).
  const std::uint32_t k = ++programs_;
  const std::uint64_t h = program_hash(prog);
  RankBlock& me = shm_->rank_block(rank_);
  me.prog_hash[k % kProgRing].store(h, std::memory_order_relaxed);
  me.prog_seq[k % kProgRing].store(k, std::memory_order_release);
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(cfg_.timeout_s);
  for (int r = 0; r < G_; ++r) {
    if (r == rank_) continue;
    RankBlock& pb = shm_->rank_block(r);
    for (int spin = 0;; ++spin) {
      const std::uint32_t seq = pb.prog_seq[k % kProgRing].load(std::memory_order_acquire);
      if (seq == k) {
        const std::uint64_t ph = pb.prog_hash[k % kProgRing].load(std::memory_order_relaxed);
        if (pb.prog_seq[k % kProgRing].load(std::memory_order_acquire) != k) continue;  // overwritten meanwhile
        if (ph != h)
          throw shardsim::ConfigError("engine: rank " + std::to_string(rank_) + " and rank " + std::to_string(r) +
                                      " were given different programs for program #" + std::to_string(k) +
                                      " (iteration " + std::to_string(prog.iteration_index) +
                                      "); every rank must execute the same program");
        break;
      }
      if (static_cast<std::int32_t>(seq - k) > 0) break;  // the peer is already kProgRing programs ahead
      if (shm_->header()->abort_flag.load(std::memory_order_relaxed))
        throw TimeoutError("engine: job aborted by a peer");
      if (spin > 2000) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        if (std::chrono::steady_clock::now() > deadline)
          throw TimeoutError("engine: rank " + std::to_string(r) + " never started program #" + std::to_string(k));
      }
    }
  }
}

void Engine::begin(const shardsim::EventProgram& prog) {
  if (failed_)
    throw shardsim::ProtocolError("engine: an earlier program failed on this rank; the engine cannot run further "
                                  "programs (destroy and recreate it)");
  if (prog_) throw shardsim::ProtocolError("engine: a program is already in progress (missing end)");
  if (prog.strategy != plan_.kind) throw shardsim::ConfigError("engine: program strategy differs from the engine plan");
  if (prog.layer_retained.size() != layers_.size()) throw shardsim::ConfigError("engine: program is for another model");
  CK(cudaSetDevice(cfg_.device));
  for (std::size_t i = 0; i < prog.events.size(); ++i)
    if (prog.events[i].id != i) throw shardsim::ConfigError("engine: event ids must be 0..n-1 in order");
  if (G_ > 1) {
    try {
      check_same_program(prog);
    } catch (...) {
      fail_job();
      throw;
    }
  }
  prog_ = &prog;
  const std::size_t n_ev = prog.events.size();
  while (ev_done_.size() < n_ev) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev_done_.push_back(e);
  }
  stream_of_.assign(n_ev, nullptr);
  last_fwd_ = 0;
  for (const Event& e : prog.events) {
    stream_of_[e.id] = stream_for(e.kind);
    if (e.kind == EventKind::ComputeFwd) last_fwd_ = e.id;
  }
  next_event_ = 0;
  for (cudaStream_t s : {s_gather_, s_cache_, s_rs_, s_agsend_, s_rssend_, s_rsrecv_, s_opt_})
    CK(cudaStreamWaitEvent(s, iter_done_, 0));
  if (trace_) {
    auto grow = [&](std::vector<cudaEvent_t>& v) {
      while (v.size() < n_ev) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        v.push_back(e);
      }
    };
    grow(trace_begin_);
    grow(trace_end_);
    if (!trace_start_) CK(cudaEventCreate(&trace_start_));
    CK(cudaEventRecord(trace_start_, s_comp_));
    for (cudaStream_t s : {s_gather_, s_cache_, s_rs_, s_agsend_, s_rssend_, s_rsrecv_, s_opt_})
      CK(cudaStreamWaitEvent(s, trace_start_, 0));
    traced_events_ = static_cast<std::uint32_t>(n_ev);
  } else {
    traced_events_ = 0;
  }
  std::fill(x_of_t_.begin(), x_of_t_.end(), -1);
  std::fill(x_of_f_.begin(), x_of_f_.end(), -1);
  std::fill(cache_stage_t_.begin(), cache_stage_t_.end(), 0);
  std::fill(stepped_.begin(), stepped_.end(), 0);
  alias_used_ = false;
  std::fill(ag_staged_valid_.begin(), ag_staged_valid_.end(), 0);
  {
    static const char* eo = std::getenv("FCDP_EARLY_OPT");
    bool has_opt = false;
    for (const Event& e : prog.events) has_opt |= e.kind == EventKind::OptimizerStep;
    // Worth it only where an inter-node RS tail follows the last backward
    // compute (N > 1); at N = 1 the update would just contend with the
    // backward GEMMs for HBM (measured: no gain).  FCDP_EARLY_OPT=0/1 forces.
    early_opt_ = has_opt && (eo ? std::strcmp(eo, "0") != 0 : N_ > 1);
    has_opt_ = has_opt;
  }
  std::fill(cache_stage_f_.begin(), cache_stage_f_.end(), 0);
  deferred_d2h_.clear();
  d2h_deferred_id_.assign(n_ev, 0);
  std::fill(d2h_done_valid_.begin(), d2h_done_valid_.end(), 0);
  if (shared_cache_)
    for (const Event& e : prog.events)
      if (e.kind == EventKind::D2H) {  // every D2H stores a forward-gathered layer
        if (wants_t(e.param_set) && layers_[e.layer].has_t) cache_stage_t_[e.layer] = 1;
        if (wants_f(e.param_set) && layers_[e.layer].has_f) cache_stage_f_[e.layer] = 1;
      }
  std::fill(w_of_layer_.begin(), w_of_layer_.end(), -1);
}

void Engine::exec(std::uint32_t event_id) {
  if (!prog_) throw shardsim::ProtocolError("engine: exec outside begin/end");
  const shardsim::EventProgram& prog = *prog_;
  if (event_id != next_event_ || event_id >= prog.events.size())
    throw shardsim::ProtocolError("engine: events must be executed once each, in id order (expected " +
                                  std::to_string(next_event_) + ", got " + std::to_string(event_id) + ")");
  std::vector<cudaStream_t>& stream_of = stream_of_;
  const std::uint32_t last_fwd = last_fwd_;
  static const bool debug = std::getenv("FCDP_DEBUG") != nullptr;
  {
    const Event& e = prog.events[event_id];
    const NvtxRange nvtx_range(e);
    cudaStream_t s = stream_of[e.id];
    if (debug)
      std::fprintf(stderr, "[fcdp r%d] it=%llu enqueue ev %u %s layer %d\n", rank_,
                   static_cast<unsigned long long>(prog.iteration_index), e.id, shardsim::to_string(e.kind), e.layer);
    if (!deferred_d2h_.empty()) {
      // the forward->backward turn: the first backward event that is not itself
      // one of the forward's cache stores (the last layer's D2H follows the last
      // ComputeFwd and must be the first store issued)
      bool flush = e.id > last_fwd && e.kind != EventKind::D2H;
      for (shardsim::EventId d : e.deps) flush |= d2h_deferred_id_[d] != 0;
      if (flush) flush_deferred_d2h();
    }
    // With tracing on, a dependent waits on the dependency's trace-end event
    // itself (recorded right after its done event on the same stream): the two
    // records are separate front-end commands, and waiting on the done event let
    // a dependent's begin timestamp precede the dependency's end timestamp when
    // the producer's channel was descheduled between them (seen once with two
    // ranks time-sharing one GPU), which the trace check reads as a violation.
    for (shardsim::EventId d : e.deps)
      if (stream_of[d] != s)
        CK(cudaStreamWaitEvent(s, trace_ && d < traced_events_ ? trace_end_[d] : ev_done_[d], 0));
    // (the staging side s_agsend_ needs none of the program's deps: its source,
    //  the own shard, is final since the previous iteration joined, and buffer
    //  reuse on it is guarded by the receivers' consumed markers - so the NIC
    //  keeps streaming the next layers while this one is expanded)
    const bool bwd = e.id > last_fwd;
    if (trace_) CK(cudaEventRecord(trace_begin_[e.id], s));
    try {
    switch (e.kind) {
      case EventKind::AgInter: ev_ag_inter(e, bwd); break;
      case EventKind::H2D: ev_h2d(e); break;
      case EventKind::AgIntra: ev_ag_intra(e, bwd); break;
      case EventKind::D2H: ev_d2h(e); break;
      case EventKind::ComputeFwd: ev_compute(e, false); break;
      case EventKind::ComputeBwd: ev_compute(e, true); break;
      case EventKind::ReduceScatter: ev_reduce_scatter(e); break;
      case EventKind::OptimizerStep: ev_optimizer(e); break;
      case EventKind::MaskDirty: break;  // bookkeeping only (step_state)
      case EventKind::Broadcast:
        throw shardsim::ConfigError("engine: broadcast events (zero2) are not part of this data plane");
    }
    } catch (...) {
      fail_job();
      throw;
    }
    const cudaStream_t ds = done_s_ ? done_s_ : s;
    done_s_ = nullptr;
    stream_of[e.id] = ds;
    if (!d2h_deferred_id_[e.id]) {  // a deferred store records these when it is issued
      CK(cudaEventRecord(ev_done_[e.id], ds));
      if (trace_) CK(cudaEventRecord(trace_end_[e.id], ds));
    }
  }
  ++next_event_;
}

void Engine::end(std::vector<shardsim::ParamState>& states) {
  if (!prog_) throw shardsim::ProtocolError("engine: end without begin");
  const shardsim::EventProgram& prog = *prog_;
  if (next_event_ != prog.events.size())
    throw shardsim::ProtocolError("engine: end after " + std::to_string(next_event_) + " of " +
                                  std::to_string(prog.events.size()) + " events");
  if (!deferred_d2h_.empty()) flush_deferred_d2h();
  // join: the next iteration starts after everything of this one
  const cudaStream_t side[7] = {s_gather_, s_cache_, s_rs_, s_agsend_, s_rssend_, s_rsrecv_, s_opt_};
  for (int i = 0; i < 7; ++i) {
    CK(cudaEventRecord(join_[i], side[i]));
    CK(cudaStreamWaitEvent(s_comp_, join_[i], 0));
  }
  CK(cudaEventRecord(iter_done_, s_comp_));
  for (std::size_t li = 0; li < layers_.size(); ++li) {
    if (!prog.layer_retained[li] && retained_[li]) {
      // retention is per iteration; the buffer stays allocated for reuse
      retained_content_[li] = {};
    }
    prev_retained_[li] = prog.layer_retained[li] ? 1 : 0;
  }
  states = shardsim::step_state(std::move(states), prog);
  prog_ = nullptr;
}

std::uint32_t Engine::trace(float* begin_ms, float* end_ms, std::uint32_t capacity) {
  sync();
  const std::uint32_t n = std::min(capacity, traced_events_);
  for (std::uint32_t i = 0; i < n; ++i) {
    CK(cudaEventElapsedTime(&begin_ms[i], trace_start_, trace_begin_[i]));
    CK(cudaEventElapsedTime(&end_ms[i], trace_start_, trace_end_[i]));
  }
  return traced_events_;
}

void Engine::sync() {
  // Poll instead of blocking so a cross-rank wait that can never be satisfied
  // (a peer died, a protocol bug) ends in a diagnosable TimeoutError.
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::duration<double>(cfg_.timeout_s);
  for (cudaStream_t s : {s_comp_, s_gather_, s_cache_, s_rs_, s_agsend_, s_rssend_, s_rsrecv_, s_opt_}) {
    if (!s) continue;
    for (int spin = 0;; ++spin) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) CK(q);
      if (std::chrono::steady_clock::now() > deadline) {
        std::string msg = "engine: rank " + std::to_string(rank_) + " stream did not drain within timeout; " +
                          "seq q=" + std::to_string(q_) + " ag_pieces=" + std::to_string(sent_pieces_[0]) + " rs_pieces=" +
                          std::to_string(sent_pieces_[1]) + " u=" + std::to_string(u_) + "; flags:";
        for (int r = 0; r < G_; ++r) {
          msg += " [r" + std::to_string(r);
          for (int f = 0; f < kNumFlags; ++f) msg += " " + std::to_string(*shm_->flag(r, static_cast<Flag>(f)));
          msg += "]";
        }
        std::fprintf(stderr, "%s\n", msg.c_str());
        shm_->header()->abort_flag.store(1);
        throw TimeoutError(msg);
      }
      if (spin > 100) std::this_thread::sleep_for(std::chrono::microseconds(spin > 10000 ? 1000 : 50));
    }
  }
}

void Engine::barrier() { shm_->barrier(cfg_.timeout_s); }

void Engine::counters(int rank, fcdp_counters* o) const {
  if (rank < 0 || rank >= G_) throw shardsim::ConfigError("counters: rank out of range");
  o->nic_tx_fwd_ag = shm_->counter(rank, kTxFwdAg);
  o->nic_tx_bwd_ag = shm_->counter(rank, kTxBwdAg);
  o->nic_tx_rs = shm_->counter(rank, kTxRs);
  o->nic_rx_fwd_ag = shm_->counter(rank, kRxFwdAg);
  o->nic_rx_bwd_ag = shm_->counter(rank, kRxBwdAg);
  o->nic_rx_rs = shm_->counter(rank, kRxRs);
  o->nvlink_rx = shm_->counter(rank, kNvlinkRx);
  o->cache_h2d = shm_->counter(rank, kCacheH2D);
  o->cache_d2h = shm_->counter(rank, kCacheD2H);
  o->staging_h2d = shm_->counter(rank, kStagingH2D);
  o->staging_d2h = shm_->counter(rank, kStagingD2H);
  o->ag_inter_events_fwd = shm_->counter(rank, kAgEventsFwd);
  o->ag_inter_events_bwd = shm_->counter(rank, kAgEventsBwd);
  o->nic_busy_ns = shm_->counter(rank, kNicBusyNs);
  o->resident_hits = shm_->counter(rank, kResidentHits);
  o->nic_tx_grad_sync = shm_->counter(rank, kTxGradSync);
  o->nic_rx_grad_sync = shm_->counter(rank, kRxGradSync);
}

void Engine::reset_counters() { shm_->reset_counters(rank_); }

void Engine::read_shard(int layer, bool frozen, void* host, std::size_t bytes) {
  const LayerRt& l = layers_.at(layer);
  const std::size_t have = (frozen ? l.L.dev.shard_f : l.L.dev.shard_t) * kChunkBytes;
  sync();
  CK(cudaMemcpy(host, (frozen ? param_f_ + l.off_f * kChunkBytes : param_t_ + l.off_t * kChunkBytes),
                std::min(bytes, have), cudaMemcpyDeviceToHost));
}

void Engine::read_master(int layer, float* host, std::size_t count) {
  const LayerRt& l = layers_.at(layer);
  sync();
  CK(cudaMemcpy(host, master_ + l.off_t * V_, std::min<std::size_t>(count, l.L.dev.shard_t * V_) * sizeof(float),
                cudaMemcpyDeviceToHost));
}

void Engine::read_grad(int layer, float* host, std::size_t count) {
  const LayerRt& l = layers_.at(layer);
  sync();
  CK(cudaMemcpy(host, grad32_ + l.off_t * V_, std::min<std::size_t>(count, l.L.dev.shard_t * V_) * sizeof(float),
                cudaMemcpyDeviceToHost));
}

void Engine::read_host_cache(int layer, bool frozen, void* host, std::size_t bytes) {
  const LayerRt& l = layers_.at(layer);
  sync();
  const unsigned char* H = host_cache_ + l.host_off * kChunkBytes + (frozen ? l.L.dev.slice_t * kChunkBytes : 0);
  const std::size_t have = (frozen ? l.slice_real_f : l.slice_real_t) * kChunkBytes;
  std::memcpy(host, H, std::min(bytes, have));
}

}  // namespace fcdp
