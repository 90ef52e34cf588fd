// Per-rank FCDP engine: shard store + executor of shardsim event programs.
//
// One process per GPU.  The engine owns
//   * the shard store: this GPU's trainable / frozen parameter shards (param
//     dtype), fp32 master / Adam moments / gradient shards for the trainable
//     portion, and the pinned host-cache tier holding this GPU's intra slice
//     of every layer (FCDP-Cache);
//   * peer-visible HBM (slice slots, natural gradient slots) that the other
//     GPUs of its emulated node read over NVLink;
//   * the executor that walks an EventProgram (reference schedule.hpp:53-61)
//     in id order and maps each event onto streams:
//        AgInter        -> host-staged NIC emulator + NVLink gather/expand
//        H2D / AgIntra  -> PCIe reload from the host cache + NVLink gather
//        D2H            -> FCDP-Cache store on a side stream
//        ComputeFwd/Bwd -> the user's compute callback on the compute stream
//        ReduceScatter  -> NVLink pull-reduce (fp32) + NIC hop + cast/scale
//        OptimizerStep  -> AdamW over the fp32 trainable arena
//     Event deps become cudaStreamWaitEvent edges; cross-rank edges are
//     stream waits on flags in the shared control block.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "common/layout.hpp"
#include "fcdp.h"
#include "kernels/kernels.hpp"
#include "runtime/nic.hpp"
#include "runtime/numa.hpp"
#include "runtime/shm.hpp"
#include "shardsim/schedule.hpp"

namespace fcdp {

struct LayerRt {
  Layout L;
  std::uint32_t* d_bits = nullptr;
  std::uint32_t* d_tpre = nullptr;
  std::int64_t elems = 0, chunks = 0;
  bool has_t = false, has_f = false;
  std::int64_t off_t = 0, off_f = 0;          // this rank's shards in the param arenas (chunks)
  std::int64_t host_off = 0;                  // this rank's slice in the host cache (chunks)
  std::int64_t my_real_t = 0, my_real_f = 0;  // real chunks of this rank's shards
  std::int64_t slice_real_t = 0, slice_real_f = 0;
  std::uint64_t shard_version_t = 0;          // version of this rank's trainable shard
  std::int64_t host_version_t = -1, host_version_f = -1;  // versions in the host cache (-1 none)
  std::int64_t replica_version_t = -1;   // ZeRO++: version in this GPU's HBM replica slice
  std::uint32_t last_replica_pull_q = 0; // ZeRO++: gather seq of the last backward pull
};

struct WContent {
  int layer = -1;
  std::int64_t ver_t = -1, ver_f = -1;  // -1: portion not present
};

class Engine {
 public:
  const NumaPlacement& numa() const { return numa_; }
  Engine(const fcdp_engine_config& cfg, const shardsim::ModelSpec& model,
         const shardsim::ClusterTopology& topo, const shardsim::StrategyPlan& plan,
         const std::uint8_t* const* chunk_masks);
  ~Engine();

  void init_params(std::uint64_t seed, const fcdp_init_range* const* ranges, const int32_t* num_ranges);
  void set_adam(const fcdp_adam_config& c) { adam_ = c; }
  void set_compute(fcdp_compute_fn fn, void* user) {
    compute_fn_ = fn;
    compute_user_ = user;
  }
  void run(const shardsim::EventProgram& prog, std::vector<shardsim::ParamState>& states);
  // The same, one event at a time: an external executor walking the program
  // in id order (begin, exec(0..n-1), end).  `prog` must outlive end().
  void begin(const shardsim::EventProgram& prog);
  void exec(std::uint32_t event_id);
  void end(std::vector<shardsim::ParamState>& states);
  void sync();
  void barrier();
  cudaStream_t compute_stream() const { return s_comp_; }
  void counters(int rank, fcdp_counters* out) const;
  void reset_counters();

  // G = 1 fused gradient -> AdamW (see kernels.cu adam_grad_kernel)
  bool fused_grad_ok(int layer) const;
  // Inside the backward compute callback of `layer`: its gradient lives in
  // these caller buffers (param dtype, 16-byte aligned) instead of grad_out.
  void grad_segments(int layer, int n, const std::int64_t* elem_offsets, const void* const* ptrs,
                     const std::int64_t* counts);
  void set_keep_grad(bool on) { keep_grad_ = on; }
  void set_timing(bool on) { timing_ = on; }
  void kernel_stats(fcdp_kernel_stats* out, bool reset);
  void set_trace(bool on) { trace_ = on; }
  void set_nic_log(bool on) { nic_->set_log(on); }
  std::size_t nic_log(WireRecord* out, std::size_t capacity) { return nic_->take_log(out, capacity); }
  std::uint32_t trace(float* begin_ms, float* end_ms, std::uint32_t capacity);

  void read_shard(int layer, bool frozen, void* host, std::size_t bytes);
  void read_master(int layer, float* host, std::size_t count);
  void read_grad(int layer, float* host, std::size_t count);
  void read_host_cache(int layer, bool frozen, void* host, std::size_t bytes);
  bool failed() const { return failed_; }

 private:
  // ---- failure / cross-rank program agreement
  void fail_job();
  static std::uint64_t program_hash(const shardsim::EventProgram& prog);
  void check_same_program(const shardsim::EventProgram& prog);
  bool failed_ = false;
  std::uint32_t programs_ = 0;  // programs begun on this engine (same count on every rank)
  // ---- setup
  void build_layouts(const std::uint8_t* const* masks);
  void allocate();
  void exchange_handles();
  // ---- events
  void ev_ag_inter(const shardsim::Event& e, bool backward);
  void ev_h2d(const shardsim::Event& e);
  void ev_ag_intra(const shardsim::Event& e, bool backward);
  void mics_grad_sync(LayerRt& l, int gs, float scale, float* final_out);
  void ev_d2h(const shardsim::Event& e);
  void ev_compute(const shardsim::Event& e, bool backward);
  void ev_reduce_scatter(const shardsim::Event& e);
  void ev_optimizer(const shardsim::Event& e);
  // ---- helpers
  cudaStream_t stream_for(shardsim::EventKind k) const;
  int begin_slice_fill(int layer);                       // returns X slot, waits WAR
  void finish_slice_fill(int slot, std::uint32_t q);
  void pull_expand(int layer, int slot, std::uint32_t q, bool want_t, bool want_f, cudaStream_t s);
  unsigned char* w_buffer(int layer);                    // W slot / retained buffer for layer
  unsigned char* x_slot(int rank_local, int slot) const; // local or peer pointer
  unsigned char* grad_slot(int rank_local, int slot) const;
  unsigned char* replica(int rank_local, int layer) const;
  void wait_flag(cudaStream_t s, int rank, Flag f, std::uint32_t v);
  void write_flag(cudaStream_t s, Flag f, std::uint32_t v);
  std::int64_t pieces_of(std::size_t bytes) const;
  struct SendSeg {
    const void* src;
    std::size_t bytes;
    unsigned char* host_dst = nullptr;  // stage into this host address (the host cache) instead of the ring
  };
  struct InSeg {
    std::size_t bytes;
    unsigned char* dst;  // null: part of the sender's message that is not for this rank
    const unsigned char* host_src = nullptr;  // the sender staged this segment here (its host cache)
  };
  struct Inbound {
    int src_rank;
    std::vector<InSeg> segs;  // the sender's whole message, in its staging order
  };
  void stage_one(int cls, cudaStream_t s, const void* src, std::size_t n, std::uint64_t wire_mult, Counter counter,
                 unsigned char* host_dst);
  void mark_consumed(int cls, cudaStream_t s, int src_node, std::uint32_t id);
  void exchange(int cls, cudaStream_t send_s, const std::vector<SendSeg>& mine, std::uint64_t wire_mult,
                Counter counter, cudaStream_t recv_s, const std::vector<Inbound>& inbound);

  fcdp_engine_config cfg_;
  std::string shm_name_;
  shardsim::ModelSpec model_;
  shardsim::ClusterTopology topo_;
  shardsim::StrategyPlan plan_;
  int N_, g_, G_, n_, j_, rank_, eb_, V_;
  // Sharding scope: the nodes one parameter shard set spans.  Every strategy
  // but MiCS shards over the whole job (Ns_ = N_, ns_ = n_); MiCS with
  // subgroup = gpus_per_node shards inside each node (Ns_ = 1) and keeps a
  // replica per node, whose gradients are summed over the NIC after the RS.
  int Ns_ = 1, ns_ = 0;
  bool mics_ = false;
  std::vector<LayerRt> layers_;
  std::int64_t max_chunks_ = 0, max_slice_ = 0, max_shard_t_ = 0, max_slice_t_ = 0;
  std::int64_t arena_t_ = 0, arena_f_ = 0, host_chunks_ = 0;

  std::unique_ptr<SharedBlock> shm_;
  void* shm_dev_base_ = nullptr;
  std::unique_ptr<NicEmulator> nic_;

  // device memory
  unsigned char* param_t_ = nullptr;
  unsigned char* param_f_ = nullptr;
  float *master_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr, *grad32_ = nullptr;
  unsigned char* w_slots_[2] = {nullptr, nullptr};
  std::vector<unsigned char*> retained_;
  unsigned char* peer_arena_ = nullptr;  // [X slots | grad slots]
  std::size_t x_slot_bytes_ = 0, grad_slot_bytes_ = 0, arena_bytes_ = 0;
  unsigned char* peer_base_[kMaxLocal] = {};  // local index -> arena base (own = peer_arena_)
  float* own32_[2] = {nullptr, nullptr};
  unsigned char* wire_[2] = {nullptr, nullptr};
  unsigned char* rx_[2] = {nullptr, nullptr};
  unsigned char* host_cache_ = nullptr;
  std::size_t host_cache_map_bytes_ = 0;  // anonymous mapping (non-shared cache)
  NumaPlacement numa_;
  // Shared host cache (N > 1, FCDP family): a forward AgInter stages this GPU's
  // own shard straight into its host-cache position and the wire serves it from
  // there, so FCDP-Cache's D2H only copies the peers' shards (write once).
  bool shared_cache_ = false;
  std::unique_ptr<ShmSegment> hc_own_;
  std::unique_ptr<ShmSegment> hc_peer_[kMaxNodes];
  unsigned char* hc_base_[kMaxNodes] = {};   // node -> host cache of (node, j_) in this process
  std::vector<char> cache_stage_t_, cache_stage_f_;  // per layer, this iteration
  std::vector<cudaEvent_t> cache_staged_;           // per layer: own shard landed in the host cache
  std::vector<std::uint32_t> cache_last_id_t_, cache_last_id_f_;  // last piece id staged into each region

  cudaStream_t s_comp_ = nullptr, s_gather_ = nullptr, s_cache_ = nullptr, s_rs_ = nullptr;
  // staging (send) side of the NIC path, so a message's pieces are staged
  // while the same layer's incoming pieces are already being received
  cudaStream_t s_agsend_ = nullptr, s_rssend_ = nullptr;
  // inter-node RS receive + epilogue: off s_rs_, so the next layer's intra RS
  // kernel and staging start while this layer's pieces are still on the wire
  cudaStream_t s_rsrecv_ = nullptr;
  cudaStream_t done_s_ = nullptr;      // set by a handler whose event completes on another stream
  cudaEvent_t fin_done_[2] = {nullptr, nullptr};  // RS epilogue of grad slot gs finished
  cudaEvent_t rs_kernel_done_[2] = {nullptr, nullptr};
  cudaEvent_t rs_staged_[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_done_;
  std::vector<cudaEvent_t> x_reader_;  // last local reader of each X slot
  cudaEvent_t rs_done_[2] = {nullptr, nullptr};
  cudaEvent_t iter_done_ = nullptr;
  cudaEvent_t join_[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaStream_t s_opt_ = nullptr;   // G = 1 fused RS + AdamW when FCDP_OPT_PRIO=low (else compute stream)
  cudaEvent_t opt_fork_ = nullptr;
  bool opt_low_ = false;
  // FCDP_RS_STREAM=compute: the reduce-scatter (G > 1) serialised on the compute stream
  bool rs_on_compute_ = false;
  cudaStream_t rs_stream() const { return rs_on_compute_ ? s_comp_ : s_rs_; }
  int rs_ctas_per_sm_ = 0;       // FCDP_RS_CTAS_PER_SM: grid cap of the RS kernel (0 = full grid)
  int opt_ctas_per_sm_ = 0;      // grid cap of the G = 1 fused update, CTAs per SM (0 = full grid)
  bool opt_on_compute_ = true;  // the G = 1 fused update on the compute stream (FCDP_OPT_STREAM=rs: beside the GEMMs)

  // sequence counters (identical on every rank)
  std::uint32_t q_ = 0, u_ = 0;
  std::int64_t chunk_bytes_ = 4ll << 20;          // inter-node wire piece size
  std::uint32_t sent_pieces_[2] = {0, 0};         // my cumulative staged pieces per class
  std::uint32_t recv_base_[2][64] = {};           // replica of every sender's piece counter
  std::uint32_t consumed_[2][8] = {};             // last consumed marker written, per sender node
  std::uint64_t w_instances_ = 0;
  int opt_steps_ = 0;
  // Early optimizer: AdamW of a layer's shard runs as soon as its gradient is
  // final (after its RS), overlapping later layers' backward instead of one
  // launch after the last RS.  Elementwise, so results are identical.  On
  // by default when N > 1.
  bool early_opt_ = false;
  bool has_opt_ = false;       // the current program has an OptimizerStep
  std::vector<char> stepped_;                 // per layer: updated early this iteration
  std::vector<cudaEvent_t> ag_staged_;        // per layer: own shard staged for the NIC (s_agsend_)
  std::vector<char> ag_staged_valid_;
  void adam_layer(int li, cudaStream_t s);
  AdamParams adam_params(int step) const;
  bool keep_grad_ = false;        // fused path also writes the fp32 gradient shard (readback)
  int bwd_callback_layer_ = -1;   // layer whose backward callback is running
  std::vector<GradSegs> grad_segs_;  // per layer: where its gradient is (fused path)
  std::vector<char> grad_segs_set_;
  // G = 1: gathers of single-portion layers alias the shard (no copy)
  bool alias_used_ = false;
  std::vector<char> prev_retained_;  // per layer: retained in the previous executed program
  cudaEvent_t alias_fence_ = nullptr;
  bool alias_gather(const shardsim::Event& e, bool wt, bool wf);
  unsigned char* alias_ptr(int li) const;
  void fence_alias_reads(cudaStream_t s, int layer = -1);
  // G = 1: FCDP-Cache stores read the shard itself, which nothing overwrites
  // before that layer's update in the backward; they are queued and issued
  // last-layer-first at the forward->backward turn (see ev_d2h).
  struct DeferredD2H {
    std::uint32_t id;
    int layer;
    bool t, f;
  };
  std::vector<DeferredD2H> deferred_d2h_;
  std::vector<char> d2h_deferred_id_;       // per event id of the current program
  std::vector<cudaEvent_t> d2h_done_;       // per layer: its FCDP-Cache store finished (this iteration)
  std::vector<char> d2h_done_valid_;
  bool defer_d2h_ = true;
  void store_d2h(int layer, bool wt, bool wf, int slot_t, int slot_f);
  void flush_deferred_d2h();

  // per-iteration bookkeeping
  struct PendingSlice {
    int slot = -1;
    std::uint32_t q = 0;
    bool t = false, f = false;
    std::int64_t ver_t = -1, ver_f = -1;
    bool alias = false;  // elided reload served by the shard itself (G = 1)
  };
  std::vector<PendingSlice> pending_h2d_;             // per layer (H2D -> AgIntra)
  std::vector<int> x_of_t_, x_of_f_;                  // per layer: X slot holding fresh gather
  std::vector<int> w_of_layer_;                       // per layer: W slot index or -1
  WContent w_content_[2];
  std::vector<WContent> retained_content_;
  std::vector<int> grad_slot_of_layer_;
  std::vector<std::uint32_t> u_of_layer_;
  const shardsim::EventProgram* prog_ = nullptr;
  std::vector<cudaStream_t> stream_of_;  // per event: stream its completion is recorded on
  std::uint32_t last_fwd_ = 0, next_event_ = 0;

  fcdp_adam_config adam_{1e-4f, 0.9f, 0.95f, 1e-8f, 0.0f, 0};
  fcdp_compute_fn compute_fn_ = nullptr;
  void* compute_user_ = nullptr;
  bool use_ce_ = false;
  bool zeropp_ = false;
  std::size_t replica_off_ = 0;

  // kernel accounting (launch counts always, event timing when enabled)
  template <typename F>
  void timed(int cls, cudaStream_t s, std::uint64_t alg_bytes, F&& launch, std::uint64_t link_bytes = 0);
  struct TimedLaunch {
    int cls;
    cudaEvent_t a, b;
    std::uint64_t bytes;
  };
  bool timing_ = false;
  std::vector<TimedLaunch> timed_pending_;
  std::vector<cudaEvent_t> timing_pool_;
  fcdp_kernel_stats kstats_{};
  bool trace_ = false;
  std::uint32_t traced_events_ = 0;
  cudaEvent_t trace_start_ = nullptr;
  std::vector<cudaEvent_t> trace_begin_, trace_end_;
};

}  // namespace fcdp
