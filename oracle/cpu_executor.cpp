// cpu_executor.cpp - C++ CPU executor of shardsim EventPrograms.
// TEST / BASELINE INFRASTRUCTURE ONLY (never linked into libfcdp.so).
//
// This is the "C++ CPU reference of the path" that bench.py's --impl reference
// arm times on the GPU box's host cores (BASELINE.md §3 "Timing 2", SURVEY
// §8(d) "CPU reference beside it" (2)):
//   * the programs come from the REFERENCE's own control plane
//     (/root/reference/proj/src/*.cpp compiled unchanged into
//     oracle/_ref/libshardsim_ref.a and linked here): build_iteration
//     (schedule.cpp:341-352) and step_state (schedule.cpp:354-387);
//   * the data plane the reference does not have is restated from the paper
//     with the oracle's arithmetic (oracle/fcdp_oracle.c): one std::thread per
//     simulated rank (node n, GPU j), all ranks walking the same program in id
//     order in lock step, buffers in host DRAM:
//       AgInter   (Alg. 1 l.11)  slice j <- the N shards {(n',j)}
//                 (memcpy; the inter-node bytes are counted), then the natural
//                 layer <- the g slices of the node (fo_expand)
//       H2D          slice j <- this rank's host cache
//       AgIntra                               natural layer <- the g slices
//       D2H  host cache <- slice j
//       Compute*                              a callback (the driving model), or a
//                                             synthetic gradient (1+rank)/8 * W
//       ReduceScatter          fo_rs_slice over the g natural
//                                             gradients, then fo_rs_finalize over
//                                             the N node partials (param-dtype wire)
//       OptimizerStep                         fo_adam over the fp32 master shard
//   * freshness: a reload of a stale host copy, or a compute on
//     parameters that are not at their current version, fails the step.
// Inside a rank the heavy loops are split over threads_per_rank OpenMP threads
// (the _part variants of the oracle give identical results for any split).
// Results are bit-identical to tests/engine_oracle.py (checked by
// tests/test_cpu_executor.py) and therefore to the B200 engine.
#include <algorithm>
#include <atomic>
#include <barrier>
#include <condition_variable>
#include <functional>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>


#include "fcdp_oracle.h"
#include "shardsim/error.hpp"
#include "shardsim/schedule.hpp"
#include "shardsim/strategy.hpp"
#include "shardsim/topology.hpp"
#include "shardsim/workload.hpp"

using shardsim::Event;
using shardsim::EventKind;
using shardsim::ParamSet;

extern "C" {
typedef int (*fce_compute_fn)(void* user, int32_t kind, int32_t rank, int32_t layer, const void* w, void* grad);

typedef struct fce_config {
  int32_t nodes, local;
  const char* strategy;     // shardsim spelling: zero3 | fcdp | fcdp-comm | zeropp | mics
  double tau;
  uint64_t gpu_capacity_bytes;
  int32_t elem_bytes;       // 2 (bf16) or 4 (fp32)
  int32_t num_layers;
  const int64_t* params;    // per layer
  const uint8_t* const* masks;  // per layer chunk mask (1 = trainable) or NULL = dense trainable
  const int64_t* act_bytes;     // per layer activation bytes per sample (tau admission), may be NULL
  int32_t batch_per_gpu;
  uint64_t seed;            // uniform(-0.05, 0.05) init of every element, as tests/engine_worker.py
  float init_scale;
  int32_t threads;          // total host threads (0 = all the process may use)
  float lr, beta1, beta2, eps, weight_decay;
  const fo_init_range* const* init_ranges;  // per layer (NULL: uniform(-init_scale, init_scale) everywhere)
  const int32_t* num_init_ranges;
} fce_config;

typedef struct fce_stats {
  double seconds;           // wall time of the step (program build + execution + step_state)
  double build_seconds;
  uint64_t events;
  // per-node sums over the step, same names as the engine counters
  uint64_t nic_tx_fwd_ag, nic_tx_bwd_ag, nic_tx_rs, nic_tx_grad_sync, cache_h2d, cache_d2h, nvlink_rx;
  uint64_t bytes_moved;     // memcpy + kernel-equivalent bytes touched (read + write), all ranks
} fce_stats;
}

namespace {

constexpr int64_t C = 16;
constexpr int64_t kBlock = 4096;  // chunks per work item inside a rank

struct Geo {
  fo_geom g{};
  std::vector<uint8_t> mask;        // empty: dense trainable
  std::vector<int64_t> kt_at;       // trainable chunks before block b
  bool has_t = false, has_f = false;
  const uint8_t* m() const { return mask.empty() ? nullptr : mask.data(); }
};

// A rank's worker team (persistent threads; the rank thread itself takes part).
class Team {
 public:
  explicit Team(int threads) {
    for (int i = 1; i < threads; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Team() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }

  template <typename F>
  void run(int64_t n_blocks, F&& fn) {
    if (workers_.empty() || n_blocks <= 1) {
      for (int64_t b = 0; b < n_blocks; ++b) fn(b);
      return;
    }
    std::function<void(int64_t)> job = fn;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      n_ = n_blocks;
      next_.store(0);
      active_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    drain(job);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return active_ == 0; });
    job_ = nullptr;
  }

 private:
  void drain(const std::function<void(int64_t)>& job) {
    for (int64_t b; (b = next_.fetch_add(1)) < n_;) job(b);
  }
  void loop() {
    std::uint64_t seen = 0;
    for (;;) {
      const std::function<void(int64_t)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        job = job_;
      }
      if (job) drain(*job);
      std::lock_guard<std::mutex> lk(mu_);
      if (--active_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::uint64_t gen_ = 0;
  bool stop_ = false;
  const std::function<void(int64_t)>* job_ = nullptr;
  int64_t n_ = 0;
  std::atomic<int64_t> next_{0};
  int active_ = 0;
};

struct Rank {
  int n = 0, j = 0, r = 0, rank = 0;
  std::vector<std::vector<uint8_t>> shard_t, shard_f, host_t, host_f, x_t, x_f;
  std::vector<std::vector<float>> master, m, v, grad;
  std::vector<std::vector<uint8_t>> retained;  // per layer, tau-retained natural layer
  std::vector<uint8_t> w_slot[2];
  std::vector<uint8_t> grad_nat;               // natural gradient of the layer in backward
  std::vector<float> own32;
  std::vector<uint8_t> wire;
  std::vector<uint64_t> shard_version;         // trainable portion version per layer
  std::vector<int64_t> host_ver_t, host_ver_f; // -1: not cached
  std::vector<int> w_of;                       // per layer: 0/1 slot, 2 retained, -1 none
  std::vector<int64_t> w_ver_t, w_ver_f;       // version held by the buffer of each layer
  uint64_t w_instances = 0;
  // counters
  uint64_t tx_fwd = 0, tx_bwd = 0, tx_rs = 0, tx_sync = 0, h2d = 0, d2h = 0, nvl = 0, moved = 0;
  std::unique_ptr<Team> team;
  int drop_d2h = -1;  // mutation hook: skip this layer's D2H in the next step
  template <typename F>
  void par(int64_t n_blocks, F&& fn) { team->run(n_blocks, std::forward<F>(fn)); }
  void pcopy(void* dst, const void* src, int64_t bytes) {
    const int64_t blk = 1 << 22;
    par((bytes + blk - 1) / blk, [&](int64_t b) {
      const int64_t off = b * blk;
      std::memcpy(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off,
                  std::min(blk, bytes - off));
    });
  }
};

struct Exec {
  fce_config cfg{};
  std::string strategy;
  shardsim::ModelSpec model;
  shardsim::ClusterTopology topo;
  shardsim::StrategyPlan plan;
  int N = 1, g = 1, G = 1, Ns = 1, L = 0, eb = 2, V = 8, tpr = 1;
  bool mics = false, zeropp = false;
  std::vector<Geo> geo;
  std::vector<Rank> ranks;
  std::vector<shardsim::ParamState> states;
  std::vector<char> prev_retained;
  uint64_t iteration = 0;
  int opt_steps = 0;
  fce_compute_fn compute = nullptr;
  void* user = nullptr;

  int64_t real(int l, bool frozen, int s) const {
    const fo_geom& q = geo[l].g;
    const int64_t per = frozen ? q.shard_f : q.shard_t, tot = frozen ? q.pf : q.pt;
    return std::max<int64_t>(0, std::min(per, tot - s * per));
  }
  int64_t real_slice(int l, bool frozen, int jj) const {
    int64_t s = 0;
    for (int nn = 0; nn < Ns; ++nn) s += real(l, frozen, jj * Ns + nn);
    return s;
  }
  int shard_index(int rank) const { return (rank % g) * Ns + (Ns > 1 ? rank / g : 0); }

  void setup(const fce_config& c) {
    cfg = c;
    strategy = c.strategy ? c.strategy : "fcdp";
    N = c.nodes;
    g = c.local;
    G = N * g;
    eb = c.elem_bytes;
    V = static_cast<int>(C / eb);
    L = c.num_layers;
    plan.kind = shardsim::strategy_kind_from_string(strategy);
    plan.tau = c.tau;
    mics = plan.kind == shardsim::StrategyKind::MiCS;
    zeropp = plan.kind == shardsim::StrategyKind::ZeroPP;
    if (plan.kind == shardsim::StrategyKind::Zero2)
      throw shardsim::ConfigError("cpu executor: zero2 has no data plane here");
    Ns = mics ? 1 : N;
    topo = shardsim::make_topology(N, g);
    plan.validate(topo);
    model.param_bytes_per_element = eb;
    model.batch_per_gpu = c.batch_per_gpu > 0 ? c.batch_per_gpu : 8;
    int threads = c.threads > 0 ? c.threads : static_cast<int>(std::thread::hardware_concurrency());
    tpr = std::max(1, threads / G);
    geo.resize(L);
    for (int l = 0; l < L; ++l) {
      const int64_t E = c.params[l];
      if ((E * eb) % C) throw shardsim::ConfigError("cpu executor: layer is not whole 16-byte chunks");
      const int64_t chunks = E * eb / C;
      Geo& q = geo[l];
      if (c.masks && c.masks[l]) q.mask.assign(c.masks[l], c.masks[l] + chunks);
      fo_geom_of(chunks, q.m(), Ns, g, &q.g);
      q.has_t = q.g.pt > 0;
      q.has_f = q.g.pf > 0;
      const int64_t nb = (chunks + kBlock - 1) / kBlock;
      q.kt_at.assign(nb + 1, 0);
      for (int64_t b = 0; b < nb; ++b) {
        int64_t t = 0;
        for (int64_t cc = b * kBlock; cc < std::min(chunks, (b + 1) * kBlock); ++cc) t += q.mask.empty() || q.mask[cc];
        q.kt_at[b + 1] = q.kt_at[b] + t;
      }
      shardsim::LayerSpec ls;
      ls.layer_id = l;
      ls.param_count = E;
      ls.trainable_fraction = static_cast<double>(q.g.pt * V) / static_cast<double>(E);
      ls.activation_bytes_per_sample = c.act_bytes ? c.act_bytes[l] : 0;
      model.layers.push_back(ls);
    }
    model.validate();
    int64_t max_chunks = 0, max_shard_t = 0, max_slice_t = 0;
    for (const Geo& q : geo) {
      max_chunks = std::max(max_chunks, q.g.chunks);
      max_shard_t = std::max(max_shard_t, q.g.shard_t);
      max_slice_t = std::max(max_slice_t, q.g.slice_t);
    }
    ranks.resize(G);
    for (int rk = 0; rk < G; ++rk) {
      Rank& R = ranks[rk];
      R.rank = rk;
      R.team = std::make_unique<Team>(tpr);
      R.n = rk / g;
      R.j = rk % g;
      R.r = shard_index(rk);
      for (auto* v : {&R.shard_t, &R.shard_f, &R.host_t, &R.host_f, &R.x_t, &R.x_f, &R.retained}) v->resize(L);
      for (auto* v : {&R.master, &R.m, &R.v, &R.grad}) v->resize(L);
      R.shard_version.assign(L, 0);
      R.host_ver_t.assign(L, -1);
      R.host_ver_f.assign(L, -1);
      R.w_of.assign(L, -1);
      R.w_ver_t.assign(L, -1);
      R.w_ver_f.assign(L, -1);
      for (auto& w : R.w_slot) w.assign(max_chunks * C, 0);
      R.grad_nat.assign(max_chunks * C, 0);
      R.own32.assign(std::max<int64_t>(max_shard_t * V, 1), 0.0f);
      R.wire.assign(std::max<int64_t>(max_slice_t * C, 16), 0);
    }
    // deterministic init: natural layer -> portions (mask order) -> padded shards;
    // layers in parallel (first touch of every buffer happens here, not in step 1)
    auto init_layer = [&](int l, std::vector<uint8_t>& nat, std::vector<uint8_t>& tv, std::vector<uint8_t>& fv) {
      const fo_geom& q = geo[l].g;
      nat.assign(q.chunks * C, 0);
      const fo_init_range rg{0, c.params[l], 0, c.init_scale};
      if (c.init_ranges && c.init_ranges[l])
        fo_init_natural(c.params[l], eb, c.seed, l, c.init_ranges[l], c.num_init_ranges[l], nat.data());
      else
        fo_init_natural(c.params[l], eb, c.seed, l, &rg, 1, nat.data());
      const int Gs = Ns * g;
      tv.assign(std::max<int64_t>(q.shard_t * Gs * C, 16), 0);
      fv.assign(std::max<int64_t>(q.shard_f * Gs * C, 16), 0);
      fo_partition(q.chunks, geo[l].m(), nat.data(), tv.data(), fv.data());
      for (Rank& R : ranks) {
        R.shard_t[l].assign(tv.begin() + R.r * q.shard_t * C, tv.begin() + (R.r + 1) * q.shard_t * C);
        R.shard_f[l].assign(fv.begin() + R.r * q.shard_f * C, fv.begin() + (R.r + 1) * q.shard_f * C);
        const int64_t n = q.shard_t * V;
        R.master[l].resize(n);
        for (int64_t i = 0; i < n; ++i)
          R.master[l][i] = eb == 2 ? fo_bf16_to_f32(reinterpret_cast<const uint16_t*>(R.shard_t[l].data())[i])
                                   : reinterpret_cast<const float*>(R.shard_t[l].data())[i];
        R.m[l].assign(n, 0.0f);
        R.v[l].assign(n, 0.0f);
        R.grad[l].assign(n, 0.0f);
        R.host_t[l].assign(q.slice_t * C, 0);
        R.host_f[l].assign(q.slice_f * C, 0);
        R.x_t[l].assign(q.slice_t * C, 0);
        R.x_f[l].assign(q.slice_f * C, 0);
      }
    };
    {
      std::atomic<int> next{0};
      std::vector<std::thread> pool;
      std::exception_ptr init_err;
      std::mutex mu;
      for (int t = 0; t < std::min(threads, L); ++t)
        pool.emplace_back([&] {
          std::vector<uint8_t> nat, tv, fv;
          for (int l; (l = next.fetch_add(1)) < L;) {
            try {
              init_layer(l, nat, tv, fv);
            } catch (...) {
              std::lock_guard<std::mutex> lk(mu);
              init_err = std::current_exception();
            }
          }
        });
      for (auto& t : pool) t.join();
      if (init_err) std::rethrow_exception(init_err);
    }
    states = shardsim::init_param_states(model);
    prev_retained.assign(L, 0);
  }

  // ---------------------------------------------------------------- events
  static bool wt_of(ParamSet s) { return s != ParamSet::FrozenOnly; }
  static bool wf_of(ParamSet s) { return s != ParamSet::TrainableOnly; }

  uint8_t* w_buffer(Rank& R, int l, const shardsim::EventProgram& p) {
    if (R.w_of[l] < 0) {
      if (p.layer_retained[l]) {
        if (R.retained[l].empty()) R.retained[l].assign(geo[l].g.chunks * C, 0);
        R.w_of[l] = 2;
      } else {
        R.w_of[l] = static_cast<int>(R.w_instances++ % 2);
      }
    }
    return R.w_of[l] == 2 ? R.retained[l].data() : R.w_slot[R.w_of[l]].data();
  }

  // phase 1 of a gather: slice j of this rank (x_t/x_f) from the scope's shards
  void fill_from_shards(Rank& R, int l, bool wt, bool wf, bool bwd) {
    const fo_geom& q = geo[l].g;
    uint64_t tx = 0;
    for (int nn = 0; nn < Ns; ++nn) {
      const Rank& P = ranks[nn * g + R.j];  // (n', j): the shard j*Ns + n' (MiCS: the own node)
      const Rank& S = Ns > 1 ? P : R;
      const int s = R.j * Ns + nn;
      if (wt && real(l, false, s)) {
        R.pcopy(R.x_t[l].data() + nn * q.shard_t * C, S.shard_t[l].data(), real(l, false, s) * C);
        R.moved += 2 * real(l, false, s) * C;
      }
      if (wf && real(l, true, s)) {
        R.pcopy(R.x_f[l].data() + nn * q.shard_f * C, S.shard_f[l].data(), real(l, true, s) * C);
        R.moved += 2 * real(l, true, s) * C;
      }
    }
    const int s = R.r;
    if (wt) tx += real(l, false, s);
    if (wf) tx += real(l, true, s);
    if (!mics) (bwd ? R.tx_bwd : R.tx_fwd) += tx * C * (N - 1);
  }

  // phase 2 of a gather: natural layer <- the node's g slices
  void pull(Rank& R, int l, bool wt, bool wf, const shardsim::EventProgram& p, int64_t ver_t) {
    const Geo& q = geo[l];
    uint8_t* W = w_buffer(R, l, p);
    std::vector<const void*> ts(g), fs(g);
    for (int jj = 0; jj < g; ++jj) {
      const Rank& P = ranks[R.n * g + jj];
      ts[jj] = P.x_t[l].data();
      fs[jj] = P.x_f[l].data();
    }
    const int set = wt && wf ? 0 : (wt ? 1 : 2);
    const int64_t nb = (q.g.chunks + kBlock - 1) / kBlock;
    R.par(nb, [&](int64_t b) {
      fo_expand_part(&q.g, q.m(), ts.data(), fs.data(), W, set, b * kBlock, std::min(q.g.chunks, (b + 1) * kBlock),
                     q.kt_at[b]);
    });
    uint64_t out = 0, rx = 0;
    if (wt) out += q.g.pt * C;
    if (wf) out += q.g.pf * C;
    for (int jj = 0; jj < g; ++jj)
      if (jj != R.j) rx += ((wt ? real_slice(l, false, jj) : 0) + (wf ? real_slice(l, true, jj) : 0)) * C;
    R.nvl += rx;
    R.moved += 2 * out;
    if (wt) R.w_ver_t[l] = ver_t;
    if (wf) R.w_ver_f[l] = 0;
  }

  bool resident(const Event& e, const shardsim::EventProgram& p) const {
    const Geo& q = geo[e.layer];
    const bool frozen_only = e.param_set == ParamSet::FrozenOnly || (e.param_set == ParamSet::All && q.g.pt == 0);
    return frozen_only && p.layer_retained[e.layer] && prev_retained[e.layer];
  }

  void synthetic_grad(Rank& R, int l, const uint8_t* W) {
    const float c = static_cast<float>(1 + R.rank) / 8.0f;
    const int64_t n = geo[l].g.chunks * V;
    const int64_t blk = kBlock * V;
    R.par((n + blk - 1) / blk, [&](int64_t b) {
      const int64_t lo = b * blk, hi = std::min(n, lo + blk);
      if (eb == 2) {
        const uint16_t* w = reinterpret_cast<const uint16_t*>(W);
        uint16_t* o = reinterpret_cast<uint16_t*>(R.grad_nat.data());
        for (int64_t i = lo; i < hi; ++i) o[i] = fo_f32_to_bf16(fo_bf16_to_f32(w[i]) * c);
      } else {
        const float* w = reinterpret_cast<const float*>(W);
        float* o = reinterpret_cast<float*>(R.grad_nat.data());
        for (int64_t i = lo; i < hi; ++i) o[i] = w[i] * c;
      }
    });
    R.moved += 2 * geo[l].g.chunks * C;
  }

  void adam(Rank& R, int l, int step) {
    const int64_t n = geo[l].g.shard_t * V;
    const float bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(cfg.beta1), step));
    const float bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(cfg.beta2), step));
    const int64_t blk = kBlock * V;
    R.par((n + blk - 1) / blk, [&](int64_t b) {
      const int64_t lo = b * blk, cnt = std::min(n, lo + blk) - lo;
      fo_adam(cnt, cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.weight_decay, bc1, bc2, R.master[l].data() + lo,
              R.m[l].data() + lo, R.v[l].data() + lo, R.grad[l].data() + lo, R.shard_t[l].data() + lo * eb, eb);
    });
    R.moved += static_cast<uint64_t>(n) * (7 * 4 + eb);
  }

  // ------------------------------------------------------------------ step
  std::exception_ptr err;
  std::mutex err_mu;
  std::atomic<bool> failed{false};

  void fail(std::exception_ptr e) {
    std::lock_guard<std::mutex> lk(err_mu);
    if (!err) err = e;
    failed.store(true);
  }

  void rank_main(int rk, const shardsim::EventProgram& p, std::barrier<>& bar) {
    Rank& R = ranks[rk];
    std::fill(R.w_of.begin(), R.w_of.end(), -1);
    R.w_instances = 0;
    shardsim::EventId last_fwd = 0;
    for (const Event& e : p.events)
      if (e.kind == EventKind::ComputeFwd) last_fwd = e.id;
    std::vector<char> pending(L, 0);   // H2D done, AgIntra pending (or elided: 2)
    std::vector<int64_t> pending_ver(L, -1);
    for (const Event& e : p.events) {
      const int l = e.layer;
      const bool bwd = e.id > last_fwd;
      // barriers inside an event (phase boundaries); a rank that fails part-way
      // still arrives at the rest, so its peers are never left waiting
      const int need = e.kind == EventKind::ReduceScatter ? 2
                       : (e.kind == EventKind::AgInter || e.kind == EventKind::H2D || e.kind == EventKind::AgIntra) ? 1
                                                                                                                 : 0;
      int done = 0;
      auto sync = [&] {
        bar.arrive_and_wait();
        ++done;
      };
      try {
        if (failed.load()) throw std::runtime_error("peer failed");
        const Geo* q = l >= 0 ? &geo[l] : nullptr;
        const bool wt = q && wt_of(e.param_set) && q->has_t, wf = q && wf_of(e.param_set) && q->has_f;
        switch (e.kind) {
          case EventKind::AgInter:
            fill_from_shards(R, l, wt, wf, bwd);
            sync();
            pull(R, l, wt, wf, p, static_cast<int64_t>(R.shard_version[l]));
            break;
          case EventKind::H2D:
            if (resident(e, p)) {
              pending[l] = 2;
              sync();
              break;
            }
            if (wt && R.host_ver_t[l] != static_cast<int64_t>(R.shard_version[l]))
              throw shardsim::ProtocolError("freshness: layer " + std::to_string(l) +
                                            " trainable portion reloaded from a stale host cache");
            if (wf && R.host_ver_f[l] != 0)
              throw shardsim::ProtocolError("freshness: layer " + std::to_string(l) +
                                            " frozen portion reloaded before it was cached");
            if (wt) {
              R.pcopy(R.x_t[l].data(), R.host_t[l].data(), real_slice(l, false, R.j) * C);
              R.h2d += real_slice(l, false, R.j) * C;
            }
            if (wf) {
              R.pcopy(R.x_f[l].data(), R.host_f[l].data(), real_slice(l, true, R.j) * C);
              R.h2d += real_slice(l, true, R.j) * C;
            }
            R.moved += 2 * (wt ? real_slice(l, false, R.j) * C : 0) + 2 * (wf ? real_slice(l, true, R.j) * C : 0);
            pending[l] = 1;
            pending_ver[l] = wt ? R.host_ver_t[l] : -1;
            sync();
            break;
          case EventKind::AgIntra:
            if (mics) {
              fill_from_shards(R, l, wt, wf, bwd);
              sync();
              pull(R, l, wt, wf, p, static_cast<int64_t>(R.shard_version[l]));
            } else if (zeropp) {  // backward from the node's GPU replicas (x_* kept since the forward)
              sync();
              pull(R, l, q->has_t, q->has_f, p, static_cast<int64_t>(R.shard_version[l]));
            } else if (pending[l] == 2) {
              w_buffer(R, l, p);  // the retained buffer already holds the frozen portion
              sync();
            } else {
              if (pending[l] != 1) throw shardsim::ProtocolError("ag_intra without a preceding h2d");
              sync();
              pull(R, l, wt, wf, p, pending_ver[l]);
            }
            pending[l] = 0;
            break;
          case EventKind::D2H:
            if (l == R.drop_d2h) break;
            if (wt) {
              R.pcopy(R.host_t[l].data(), R.x_t[l].data(), real_slice(l, false, R.j) * C);
              R.d2h += real_slice(l, false, R.j) * C;
              R.host_ver_t[l] = static_cast<int64_t>(R.shard_version[l]);
            }
            if (wf) {
              R.pcopy(R.host_f[l].data(), R.x_f[l].data(), real_slice(l, true, R.j) * C);
              R.d2h += real_slice(l, true, R.j) * C;
              R.host_ver_f[l] = 0;
            }
            R.moved += 2 * (wt ? real_slice(l, false, R.j) * C : 0) + 2 * (wf ? real_slice(l, true, R.j) * C : 0);
            break;
          case EventKind::ComputeFwd:
          case EventKind::ComputeBwd: {
            if (R.w_of[l] < 0) throw shardsim::ProtocolError("freshness: layer computed without a gather");
            if ((q->has_t && R.w_ver_t[l] != static_cast<int64_t>(R.shard_version[l])) || (q->has_f && R.w_ver_f[l] != 0))
              throw shardsim::ProtocolError("freshness: layer " + std::to_string(l) +
                                            " would compute on parameters that are not at their current version");
            const uint8_t* W = R.w_of[l] == 2 ? R.retained[l].data() : R.w_slot[R.w_of[l]].data();
            const bool b = e.kind == EventKind::ComputeBwd;
            void* gp = b && q->has_t ? R.grad_nat.data() : nullptr;
            if (compute) {
              if (compute(user, b ? 5 : 4, rk, l, W, gp) != 0) throw std::runtime_error("compute callback failed");
            } else if (gp) {
              synthetic_grad(R, l, W);
            }
            if (!b && R.w_of[l] != 2) R.w_of[l] = -1;
            break;
          }
          case EventKind::ReduceScatter: {
            if (!q->has_t) {
              sync();
              sync();
              break;
            }
            sync();  // every rank's natural gradient is written
            std::vector<const void*> gs(g);
            for (int jj = 0; jj < g; ++jj) gs[jj] = ranks[R.n * g + jj].grad_nat.data();
            const float scale = 1.0f / static_cast<float>(G);
            const int own_idx = N > 1 ? (mics ? -1 : R.n) : 0;
            const int64_t nb = (q->g.chunks + kBlock - 1) / kBlock;
            R.par(nb, [&](int64_t b) {
              fo_rs_slice_part(&q->g, q->m(), eb, gs.data(), R.j, own_idx, scale, N == 1 ? 1 : 0,
                               N == 1 ? R.grad[l].data() : R.own32.data(), R.wire.data(), b * kBlock,
                               std::min(q->g.chunks, (b + 1) * kBlock), q->kt_at[b]);
            });
            R.nvl += static_cast<uint64_t>(g - 1) * real_slice(l, false, R.j) * C;
            R.moved += static_cast<uint64_t>(g) * real_slice(l, false, R.j) * C + q->g.shard_t * V * 4 +
                       (q->g.slice_t - q->g.shard_t) * C;
            sync();  // every rank's partials (own32 / wire) are final
            if (N > 1) {
              const int64_t sh = q->g.shard_t * V;
              std::vector<uint8_t> rx(static_cast<size_t>(N) * sh * eb, 0);
              for (int nn = 0; nn < N; ++nn) {
                const Rank& P = ranks[nn * g + R.j];
                if (mics) {
                  std::memcpy(rx.data() + nn * sh * eb, P.wire.data(), sh * eb);
                } else if (nn != R.n) {
                  std::memcpy(rx.data() + nn * sh * eb, P.wire.data() + R.n * sh * eb, sh * eb);
                  R.tx_rs += real(l, false, R.j * N + nn) * C;
                }
              }
              if (mics) R.tx_sync += static_cast<uint64_t>(N - 1) * real_slice(l, false, R.j) * C;
              const int64_t blk = kBlock * V;
              R.par((sh + blk - 1) / blk, [&](int64_t b) {
                const int64_t lo = b * blk, cnt = std::min(sh, lo + blk) - lo;
                fo_rs_finalize(cnt, N, mics ? -1 : R.n, eb, R.own32.data() + lo, rx.data() + lo * eb, sh, scale,
                               R.grad[l].data() + lo);
              });
              R.moved += static_cast<uint64_t>(sh) * (2 * 4 + (N - 1) * eb);
            }
            break;
          }
          case EventKind::OptimizerStep:
            for (int ll = 0; ll < L; ++ll)
              if (geo[ll].has_t) {
                adam(R, ll, opt_steps + 1);
                ++R.shard_version[ll];
              }
            break;
          case EventKind::MaskDirty:
            break;
          case EventKind::Broadcast:
            throw shardsim::ConfigError("cpu executor: broadcast (zero2) events are not executed");
        }
      } catch (...) {
        fail(std::current_exception());
      }
      while (done < need) sync();
      bar.arrive_and_wait();  // lock step: event e is complete on every rank
    }
  }

  void step(fce_stats* st) {
    const auto t0 = std::chrono::steady_clock::now();
    ++iteration;
    shardsim::BuildOptions opts;
    opts.gpu_capacity_bytes = cfg.gpu_capacity_bytes;
    const shardsim::EventProgram p = shardsim::build_iteration(plan, model, topo, states, iteration, opts);
    const auto t1 = std::chrono::steady_clock::now();
    for (Rank& R : ranks) R.tx_fwd = R.tx_bwd = R.tx_rs = R.tx_sync = R.h2d = R.d2h = R.nvl = R.moved = 0;
    err = nullptr;
    failed.store(false);
    std::barrier<> bar(G);
    std::vector<std::thread> th;
    for (int rk = 0; rk < G; ++rk) th.emplace_back([&, rk] { rank_main(rk, p, bar); });
    for (auto& t : th) t.join();
    for (Rank& R : ranks) R.drop_d2h = -1;
    if (err) std::rethrow_exception(err);
    ++opt_steps;
    for (int l = 0; l < L; ++l) prev_retained[l] = p.layer_retained[l];
    states = shardsim::step_state(std::move(states), p);
    const auto t2 = std::chrono::steady_clock::now();
    if (st) {
      *st = fce_stats{};
      st->seconds = std::chrono::duration<double>(t2 - t0).count();
      st->build_seconds = std::chrono::duration<double>(t1 - t0).count();
      st->events = p.events.size();
      for (const Rank& R : ranks) {
        st->nic_tx_fwd_ag += R.tx_fwd;
        st->nic_tx_bwd_ag += R.tx_bwd;
        st->nic_tx_rs += R.tx_rs;
        st->nic_tx_grad_sync += R.tx_sync;
        st->cache_h2d += R.h2d;
        st->cache_d2h += R.d2h;
        st->nvlink_rx += R.nvl;
        st->bytes_moved += R.moved;
      }
      for (uint64_t* v : {&st->nic_tx_fwd_ag, &st->nic_tx_bwd_ag, &st->nic_tx_rs, &st->nic_tx_grad_sync,
                          &st->cache_h2d, &st->cache_d2h, &st->nvlink_rx})
        *v /= static_cast<uint64_t>(N);  // per node
    }
  }
};

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const shardsim::ConfigError& e) {
    g_err = e.what();
    return -1;
  } catch (const shardsim::ProtocolError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -5;
  }
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* fce_last_error() { return g_err.c_str(); }

__attribute__((visibility("default"))) int fce_create(const fce_config* cfg, void** out) {
  return guard([&] {
    auto* x = new Exec();
    try {
      x->setup(*cfg);
    } catch (...) {
      delete x;
      throw;
    }
    *out = x;
  });
}

__attribute__((visibility("default"))) int fce_set_compute(void* h, fce_compute_fn fn, void* user) {
  return guard([&] {
    static_cast<Exec*>(h)->compute = fn;
    static_cast<Exec*>(h)->user = user;
  });
}

__attribute__((visibility("default"))) int fce_step(void* h, fce_stats* st) {
  return guard([&] { static_cast<Exec*>(h)->step(st); });
}

__attribute__((visibility("default"))) int fce_threads_per_rank(void* h) { return static_cast<Exec*>(h)->tpr; }

// Readback (tests): what the GPU engine's fcdp_engine_read_* return.
__attribute__((visibility("default"))) int fce_read(void* h, int32_t rank, int32_t layer, int32_t what, void* out,
                                                    uint64_t bytes) {
  return guard([&] {
    Exec& x = *static_cast<Exec*>(h);
    if (rank < 0 || rank >= x.G || layer < 0 || layer >= x.L) throw shardsim::ConfigError("fce_read: out of range");
    const Rank& R = x.ranks[rank];
    const void* src = nullptr;
    uint64_t have = 0;
    switch (what) {
      case 0: src = R.shard_t[layer].data(); have = R.shard_t[layer].size(); break;
      case 1: src = R.shard_f[layer].data(); have = R.shard_f[layer].size(); break;
      case 2: src = R.host_t[layer].data(); have = R.host_t[layer].size(); break;
      case 3: src = R.host_f[layer].data(); have = R.host_f[layer].size(); break;
      case 4: src = R.master[layer].data(); have = R.master[layer].size() * 4; break;
      case 5: src = R.grad[layer].data(); have = R.grad[layer].size() * 4; break;
      default: throw shardsim::ConfigError("fce_read: unknown field");
    }
    std::memcpy(out, src, std::min(bytes, have));
  });
}

// Mutation hook: in the next step, rank `rank` loses the
// FCDP-Cache store (D2H) of `layer` - its host copy keeps the previous version -
// so that layer's backward reload must fail with a ProtocolError.
__attribute__((visibility("default"))) int fce_drop_d2h(void* h, int32_t rank, int32_t layer) {
  return guard([&] {
    Exec& x = *static_cast<Exec*>(h);
    x.ranks.at(rank).drop_d2h = layer;
  });
}

__attribute__((visibility("default"))) void fce_destroy(void* h) { delete static_cast<Exec*>(h); }

}  // extern "C"
