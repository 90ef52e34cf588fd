// C ABI over the shardsim control plane (include/fcdp.h, "control plane").
//
// Each entry point is a thin, exception-free wrapper of the corresponding
// reference function; the reference signature it stands in for is cited at
// the declaration in include/fcdp.h.
#include <cstring>
#include <new>
#include <string>

#include "capi_util.hpp"
#include "fcdp.h"
#include "shardsim/collective.hpp"
#include "shardsim/costmodel.hpp"
#include "shardsim/schedule.hpp"

struct fcdp_model {
  shardsim::ModelSpec spec;
};
struct fcdp_states {
  std::vector<shardsim::ParamState> v;
};
struct fcdp_program {
  shardsim::EventProgram prog;
};

using fcdp::guarded;

namespace {

shardsim::ClusterTopology to_topo(const fcdp_topology* t) {
  shardsim::ClusterTopology o;
  o.num_nodes = t->num_nodes;
  o.gpus_per_node = t->gpus_per_node;
  shardsim::LinkClass* links[3] = {&o.intra_gpu, &o.host_gpu, &o.inter_node};
  for (int k = 0; k < 3; ++k) {
    links[k]->kind = static_cast<shardsim::LinkKind>(k);
    links[k]->bandwidth_bytes_per_s = t->bandwidth_bytes_per_s[k];
    links[k]->latency_s = t->latency_s[k];
    links[k]->duplex = t->duplex[k] ? shardsim::Duplex::HalfDuplex : shardsim::Duplex::FullDuplex;
  }
  return o;
}

void from_topo(const shardsim::ClusterTopology& t, fcdp_topology* o) {
  o->num_nodes = t.num_nodes;
  o->gpus_per_node = t.gpus_per_node;
  const shardsim::LinkClass* links[3] = {&t.intra_gpu, &t.host_gpu, &t.inter_node};
  for (int k = 0; k < 3; ++k) {
    o->bandwidth_bytes_per_s[k] = links[k]->bandwidth_bytes_per_s;
    o->latency_s[k] = links[k]->latency_s;
    o->duplex[k] = links[k]->duplex == shardsim::Duplex::HalfDuplex ? 1 : 0;
  }
}

shardsim::StrategyPlan to_plan(const fcdp_plan* p) {
  if (p->kind < 0 || p->kind > 5) throw shardsim::ConfigError("strategy.kind: out of range");
  shardsim::StrategyPlan o;
  o.kind = static_cast<shardsim::StrategyKind>(p->kind);
  o.subgroup_size = p->subgroup_size;
  o.tau = p->tau;
  o.host_cache_enabled = p->host_cache_enabled != 0;
  return o;
}

}  // namespace

namespace fcdp {
shardsim::ClusterTopology topo_from_c(const fcdp_topology* t) { return to_topo(t); }
shardsim::StrategyPlan plan_from_c(const fcdp_plan* p) { return to_plan(p); }
const shardsim::ModelSpec& model_from_c(const fcdp_model* m) { return m->spec; }
const shardsim::EventProgram& program_from_c(const fcdp_program* p) { return p->prog; }
std::vector<shardsim::ParamState>& states_from_c(fcdp_states* s) { return s->v; }
}  // namespace fcdp

extern "C" {

const char* fcdp_version(void) { return "fcdp-b200 0.1 (sm_100a)"; }

uint64_t fcdp_ag_inter_bytes(uint64_t payload, int32_t scope_nodes) {
  return scope_nodes < 1 ? 0 : shardsim::ag_inter_bytes(payload, scope_nodes);
}
uint64_t fcdp_ring_intra_bytes(uint64_t payload, int32_t ring_gpus) {
  return ring_gpus < 1 ? 0 : shardsim::ring_intra_bytes(payload, ring_gpus);
}

int fcdp_link_preset(const char* name, int32_t* kind, double* bw) {
  return guarded([&] {
    const shardsim::LinkClass c = shardsim::link_preset(name ? name : "");
    if (kind) *kind = static_cast<int32_t>(c.kind);
    if (bw) *bw = c.bandwidth_bytes_per_s;
  });
}

int fcdp_make_topology(int32_t n, int32_t g, const char* intra, const char* host, const char* inter,
                       fcdp_topology* out) {
  return guarded([&] {
    from_topo(shardsim::make_topology(n, g, intra ? intra : "nvlink3-theoretical",
                                      host ? host : "pcie4-measured",
                                      inter ? inter : "ib100-rdma-measured"),
              out);
  });
}

int fcdp_transfer_time(uint64_t size, int32_t kind, const fcdp_topology* topo, double* out) {
  return guarded([&] {
    if (kind < 0 || kind > 2) throw shardsim::ConfigError("topology: unknown link class");
    *out = shardsim::transfer_time(size, static_cast<shardsim::LinkKind>(kind), to_topo(topo));
  });
}

int fcdp_model_create(int32_t L, const int64_t* counts, const double* frac, int32_t dtype,
                      double opt_mult, int32_t batch, const double* fwd, const double* bwd,
                      const int64_t* act, fcdp_model** out) {
  return guarded([&] {
    auto* m = new fcdp_model;
    m->spec.param_bytes_per_element = dtype;
    m->spec.optimizer_state_multiplier = opt_mult;
    m->spec.batch_per_gpu = batch;
    for (int32_t i = 0; i < L; ++i) {
      shardsim::LayerSpec l;
      l.layer_id = i;
      l.param_count = counts[i];
      l.trainable_fraction = frac ? frac[i] : 1.0;
      l.fwd_compute_s_per_sample = fwd ? fwd[i] : 0.0;
      l.bwd_compute_s_per_sample = bwd ? bwd[i] : 0.0;
      l.activation_bytes_per_sample = act ? act[i] : 0;
      m->spec.layers.push_back(l);
    }
    *out = m;
  });
}

int fcdp_model_preset(const char* name, fcdp_model** out) {
  return guarded([&] { *out = new fcdp_model{shardsim::model_preset(name ? name : "")}; });
}

int fcdp_model_apply_lora_mask(const fcdp_model* model, double f, fcdp_model** out) {
  return guarded([&] { *out = new fcdp_model{shardsim::apply_lora_mask(model->spec, f)}; });
}

int fcdp_model_info(const fcdp_model* m, int32_t* L, int64_t* total, int64_t* trainable, int32_t* dtype) {
  return guarded([&] {
    if (L) *L = m->spec.num_layers();
    if (total) *total = m->spec.total_params();
    if (trainable) *trainable = m->spec.trainable_params();
    if (dtype) *dtype = m->spec.param_bytes_per_element;
  });
}

int fcdp_model_layer_bytes(const fcdp_model* m, int32_t l, uint64_t* all, uint64_t* t, uint64_t* f) {
  return guarded([&] {
    if (l < 0 || l >= m->spec.num_layers()) throw shardsim::ConfigError("layer: out of range");
    if (all) *all = shardsim::layer_bytes(m->spec, l);
    if (t) *t = shardsim::layer_trainable_bytes(m->spec, l);
    if (f) *f = shardsim::layer_frozen_bytes(m->spec, l);
  });
}

void fcdp_model_destroy(fcdp_model* m) { delete m; }

int fcdp_strategy_from_string(const char* s, int32_t* kind) {
  return guarded([&] { *kind = static_cast<int32_t>(shardsim::strategy_kind_from_string(s ? s : "")); });
}

int fcdp_memory_footprint_of(const fcdp_plan* p, const fcdp_model* m, const fcdp_topology* t,
                             fcdp_memory_footprint* out) {
  return guarded([&] {
    const auto fp = shardsim::memory_footprint(to_plan(p), m->spec, to_topo(t));
    out->gpu_param_shard_bytes = fp.gpu_param_shard_bytes;
    out->gpu_gradient_bytes = fp.gpu_gradient_bytes;
    out->gpu_optimizer_bytes = fp.gpu_optimizer_bytes;
    out->gpu_persistent_bytes = fp.gpu_persistent_bytes;
    out->gpu_cache_bytes = fp.gpu_cache_bytes;
    out->gpu_transient_peak_bytes = fp.gpu_transient_peak_bytes;
    out->host_cache_bytes_per_node = fp.host_cache_bytes_per_node;
  });
}

int fcdp_max_feasible_batch(const fcdp_plan* p, const fcdp_model* m, const fcdp_topology* t,
                            uint64_t cap, int32_t* max_batch, int32_t* oom) {
  return guarded([&] {
    const auto r = shardsim::max_feasible_batch(to_plan(p), m->spec, to_topo(t), cap);
    *max_batch = r.max_batch;
    *oom = r.oom_at_batch_1 ? 1 : 0;
  });
}

int fcdp_comm_volume_of(const fcdp_plan* p, const fcdp_model* m, const fcdp_topology* t, uint64_t it,
                        fcdp_comm_volume* out) {
  return guarded([&] {
    const auto v = shardsim::comm_volume(to_plan(p), m->spec, to_topo(t), it);
    out->fwd_ag_inter = v.fwd_ag_inter;
    out->bwd_ag_inter = v.bwd_ag_inter;
    out->reduce_scatter_inter = v.reduce_scatter_inter;
    out->param_sync_inter = v.param_sync_inter;
    out->intra_node_total = v.intra_node_total;
    out->h2d_total = v.h2d_total;
    out->d2h_total = v.d2h_total;
  });
}

int fcdp_iteration_time_estimate(const fcdp_plan* p, const fcdp_model* m, const fcdp_topology* t, double* out) {
  return guarded([&] { *out = shardsim::iteration_time_estimate(to_plan(p), m->spec, to_topo(t)); });
}

int fcdp_states_init(const fcdp_model* m, fcdp_states** out) {
  return guarded([&] { *out = new fcdp_states{shardsim::init_param_states(m->spec)}; });
}

int fcdp_states_create(int32_t n, fcdp_states** out) {
  return guarded([&] {
    if (n < 0) throw shardsim::ConfigError("states: negative count");
    *out = new fcdp_states{std::vector<shardsim::ParamState>(static_cast<std::size_t>(n))};
  });
}

int fcdp_states_count(const fcdp_states* s, int32_t* n) {
  return guarded([&] { *n = static_cast<int32_t>(s->v.size()); });
}

int fcdp_states_get(const fcdp_states* s, int32_t i, fcdp_param_state* out) {
  return guarded([&] {
    const shardsim::ParamState& p = s->v.at(static_cast<std::size_t>(i));
    out->layer = p.layer;
    out->frozen = p.frozen;
    out->version = p.version;
    out->dirty = p.dirty;
    out->host_cached_version = p.host_cached_version ? static_cast<int64_t>(*p.host_cached_version) : -1;
    out->gpu_cached = p.gpu_cached;
  });
}

int fcdp_states_set(fcdp_states* s, int32_t i, const fcdp_param_state* in) {
  return guarded([&] {
    shardsim::ParamState& p = s->v.at(static_cast<std::size_t>(i));
    p.layer = in->layer;
    p.frozen = in->frozen != 0;
    p.version = in->version;
    p.dirty = in->dirty != 0;
    if (in->host_cached_version >= 0)
      p.host_cached_version = static_cast<std::uint64_t>(in->host_cached_version);
    else
      p.host_cached_version.reset();
    p.gpu_cached = in->gpu_cached != 0;
  });
}

void fcdp_states_destroy(fcdp_states* s) { delete s; }

int fcdp_build_iteration(const fcdp_plan* p, const fcdp_model* m, const fcdp_topology* t,
                         const fcdp_states* s, uint64_t it, int32_t prefetch, uint64_t cap,
                         fcdp_program** out) {
  return guarded([&] {
    shardsim::BuildOptions o;
    o.prefetch = prefetch != 0;
    o.gpu_capacity_bytes = cap;
    *out = new fcdp_program{shardsim::build_iteration(to_plan(p), m->spec, to_topo(t), s->v, it, o)};
  });
}

int fcdp_step_state(fcdp_states* s, const fcdp_program* p) {
  return guarded([&] { s->v = shardsim::step_state(std::move(s->v), p->prog); });
}

int fcdp_program_num_events(const fcdp_program* p, uint32_t* n) {
  return guarded([&] { *n = static_cast<uint32_t>(p->prog.events.size()); });
}

int fcdp_program_event(const fcdp_program* p, uint32_t i, fcdp_event* out, uint32_t* deps, uint32_t cap) {
  return guarded([&] {
    const shardsim::Event& e = p->prog.events.at(i);
    out->id = e.id;
    out->kind = static_cast<int32_t>(e.kind);
    out->layer = e.layer;
    out->param_set = static_cast<int32_t>(e.param_set);
    out->bytes_total = e.bytes_total;
    out->num_deps = static_cast<uint32_t>(e.deps.size());
    for (uint32_t k = 0; deps && k < cap && k < e.deps.size(); ++k) deps[k] = e.deps[k];
  });
}

int fcdp_program_create(uint64_t it, int32_t strategy, uint32_t n, const fcdp_event* ev, const uint32_t* off,
                        const uint32_t* deps, int32_t num_layers, const uint8_t* flags, fcdp_program** out) {
  return guarded([&] {
    if (strategy < 0 || strategy > static_cast<int32_t>(shardsim::StrategyKind::FcdpComm) || num_layers < 0)
      throw shardsim::ConfigError("program_create: bad strategy or layer count");
    shardsim::EventProgram p;
    p.iteration_index = it;
    p.strategy = static_cast<shardsim::StrategyKind>(strategy);
    for (uint32_t i = 0; i < n; ++i) {
      if (ev[i].id != i) throw shardsim::ConfigError("program_create: event ids must be 0..n-1 in order");
      if (ev[i].kind < 0 || ev[i].kind > static_cast<int32_t>(shardsim::EventKind::Broadcast) ||
          ev[i].param_set < 0 || ev[i].param_set > static_cast<int32_t>(shardsim::ParamSet::FrozenOnly) ||
          ev[i].layer >= num_layers)
        throw shardsim::ConfigError("program_create: event " + std::to_string(i) + " is malformed");
      shardsim::Event e;
      e.id = i;
      e.kind = static_cast<shardsim::EventKind>(ev[i].kind);
      e.layer = ev[i].layer;
      e.param_set = static_cast<shardsim::ParamSet>(ev[i].param_set);
      e.bytes_total = ev[i].bytes_total;
      for (uint32_t k = off[i]; k < off[i + 1]; ++k) {
        if (deps[k] >= i) throw shardsim::ConfigError("program_create: deps must point to earlier events");
        e.deps.push_back(deps[k]);
      }
      p.events.push_back(std::move(e));
    }
    for (int32_t l = 0; l < num_layers; ++l) {
      const uint8_t f = flags ? flags[l] : 0;
      p.layer_retained.push_back((f & 1) ? 1 : 0);
      p.layer_clean_path.push_back((f & 2) ? 1 : 0);
      p.layer_dirty_path.push_back((f & 4) ? 1 : 0);
    }
    *out = new fcdp_program{std::move(p)};
  });
}

int fcdp_program_layer_flags(const fcdp_program* p, uint8_t* out, int32_t cap) {
  return guarded([&] {
    const auto& pr = p->prog;
    for (int32_t l = 0; l < cap && l < static_cast<int32_t>(pr.layer_retained.size()); ++l)
      out[l] = static_cast<uint8_t>((pr.layer_retained[l] ? 1 : 0) | (pr.layer_clean_path[l] ? 2 : 0) |
                                    (pr.layer_dirty_path[l] ? 4 : 0));
  });
}

int fcdp_program_serialize(const fcdp_program* p, char* buf, size_t cap, size_t* len) {
  return guarded([&] {
    const std::string s = shardsim::serialize_program(p->prog);
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

void fcdp_program_destroy(fcdp_program* p) { delete p; }

}  // extern "C"
