// Golden dump of the shardsim control plane through its PUBLIC API only.
//
// The same source is compiled twice:
//   * against /root/reference/proj (by oracle/Makefile -> oracle/_ref/golden_ref)
//     to produce the committed goldens tests/golden/control_plane.txt;
//   * against this repo's include/shardsim + libfcdp.so (tests/test_control_plane.py)
// and the two outputs must be byte-identical.  That is the drop-in proof for
// the step interface (schedule.hpp), the byte oracle (costmodel.hpp) and the
// memory model (strategy.hpp).
#include <cinttypes>
#include <cstdio>
#include <string>
#include <vector>

#include "shardsim/collective.hpp"
#include "shardsim/costmodel.hpp"
#include "shardsim/error.hpp"
#include "shardsim/schedule.hpp"
#include "shardsim/strategy.hpp"
#include "shardsim/topology.hpp"
#include "shardsim/workload.hpp"

using namespace shardsim;

namespace {

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

ModelSpec uniform(int layers, std::int64_t params, int dtype, double frac = 1.0) {
  ModelSpec m;
  m.param_bytes_per_element = dtype;
  for (int i = 0; i < layers; ++i) {
    LayerSpec l;
    l.layer_id = i;
    l.param_count = params;
    l.trainable_fraction = frac;
    m.layers.push_back(l);
  }
  return m;
}

ModelSpec explicit_list(const std::vector<std::int64_t>& counts, const std::vector<double>& fracs,
                        int dtype) {
  ModelSpec m;
  m.param_bytes_per_element = dtype;
  for (std::size_t i = 0; i < counts.size(); ++i) {
    LayerSpec l;
    l.layer_id = static_cast<int>(i);
    l.param_count = counts[i];
    l.trainable_fraction = fracs[i];
    m.layers.push_back(l);
  }
  return m;
}

struct NamedModel {
  std::string name;
  ModelSpec model;
  bool full_text;  // print whole programs (small models) or their hash
};

std::vector<NamedModel> models() {
  std::vector<NamedModel> out;
  // C1: tiny 2-layer transformer, hidden 256, fp32: 12h^2 + 13h params per block.
  out.push_back({"tiny-h256-fp32", uniform(2, 12 * 256 * 256 + 13 * 256, 4), true});
  // 3-layer toy with a LoRA split and activations (tau admission paths).
  {
    ModelSpec m = uniform(3, 1000, 2, 0.25);
    for (auto& l : m.layers) {
      l.activation_bytes_per_sample = 100;
      l.fwd_compute_s_per_sample = 1e-3;
      l.bwd_compute_s_per_sample = 2e-3;
    }
    m.batch_per_gpu = 4;
    out.push_back({"toy3-lora25", m, true});
  }
  // Frozen-only middle layer and a fully-trainable last layer.
  out.push_back({"toy3-mixed", explicit_list({4096, 8192, 4096}, {0.5, 0.0, 1.0}, 2), true});
  // C2: GPT-2 1.3B blocks (h=2048), bf16.
  out.push_back({"gpt2-1.3b-blocks", uniform(24, 50358272, 2), false});
  // C2 explicit list: wte+wpe | 24 blocks | final LN (tied head).
  {
    std::vector<std::int64_t> c{50257LL * 2048 + 1024LL * 2048};
    std::vector<double> f{1.0};
    for (int i = 0; i < 24; ++i) c.push_back(50358272), f.push_back(1.0);
    c.push_back(2 * 2048);
    f.push_back(1.0);
    out.push_back({"gpt2-1.3b-explicit", explicit_list(c, f, 2), false});
  }
  // C3: Llama-7B + LoRA r=16 on q,k,v,o (524,288 trainable of 202,907,648 per block).
  out.push_back({"llama7b-lora16-blocks", uniform(32, 202907648, 2, 524288.0 / 202907648.0), false});
  {
    std::vector<std::int64_t> c{32000LL * 4096};
    std::vector<double> f{0.0};
    for (int i = 0; i < 32; ++i) c.push_back(202907648), f.push_back(524288.0 / 202907648.0);
    c.push_back(4096 + 32000LL * 4096);
    f.push_back(0.0);
    out.push_back({"llama7b-lora16-explicit", explicit_list(c, f, 2), false});
  }
  // C4: Llama-13B blocks.
  out.push_back({"llama13b-blocks", uniform(40, 317204480, 2), false});
  for (const std::string& p : model_preset_names()) {
    out.push_back({p, model_preset(p), false});
    out.push_back({p + "+lora0.01", apply_lora_mask(model_preset(p), 0.01), false});
  }
  return out;
}

struct NamedPlan {
  std::string name;
  StrategyPlan plan;
};

std::vector<NamedPlan> plans() {
  std::vector<NamedPlan> out;
  for (StrategyKind k : {StrategyKind::Zero2, StrategyKind::Zero3, StrategyKind::ZeroPP,
                         StrategyKind::Fcdp, StrategyKind::FcdpComm}) {
    StrategyPlan p;
    p.kind = k;
    out.push_back({to_string(k), p});
  }
  StrategyPlan mics;
  mics.kind = StrategyKind::MiCS;
  out.push_back({"mics", mics});
  for (StrategyKind k : {StrategyKind::Fcdp, StrategyKind::FcdpComm})
    for (double tau : {0.5, 1.0}) {
      StrategyPlan p;
      p.kind = k;
      p.tau = tau;
      char nm[64];
      std::snprintf(nm, sizeof nm, "%s/tau=%.2f", to_string(k), tau);
      out.push_back({nm, p});
    }
  return out;
}

void print_volume(const char* tag, const CommVolume& v) {
  std::printf("%s fwd=%" PRIu64 " bwd=%" PRIu64 " rs=%" PRIu64 " sync=%" PRIu64 " intra=%" PRIu64
              " h2d=%" PRIu64 " d2h=%" PRIu64 " inter_total=%" PRIu64 "\n",
              tag, v.fwd_ag_inter, v.bwd_ag_inter, v.reduce_scatter_inter, v.param_sync_inter,
              v.intra_node_total, v.h2d_total, v.d2h_total, v.inter_total());
}

template <typename F>
void expect_error(const char* what, F&& f) {
  try {
    f();
    std::printf("error[%s]: none\n", what);
  } catch (const ConfigError& e) {
    std::printf("error[%s]: ConfigError: %s\n", what, e.what());
  } catch (const ProtocolError& e) {
    std::printf("error[%s]: ProtocolError: %s\n", what, e.what());
  }
}

}  // namespace

int main() {
  // Byte-split rules.
  for (std::uint64_t s : {0ull, 1ull, 7ull, 100716544ull, 18446744073709551615ull})
    for (int n : {1, 2, 3, 4, 8})
      std::printf("split S=%" PRIu64 " n=%d ag=%" PRIu64 " ring=%" PRIu64 "\n", s, n,
                  ag_inter_bytes(s, n), ring_intra_bytes(s, n));

  // Link presets and transfer times.
  for (const std::string& p : link_preset_names()) {
    const LinkClass c = link_preset(p);
    std::printf("preset %s kind=%s bw=%.17g duplex=%s t16GiB=%.17g\n", p.c_str(), to_string(c.kind),
                c.bandwidth_bytes_per_s, to_string(c.duplex), 16.0 * kGiB / c.bandwidth_bytes_per_s);
  }
  {
    const ClusterTopology t = make_topology(2, 4, "nvlink3-theoretical", "pcie4-measured", "eth10g-measured");
    for (LinkKind k : {LinkKind::IntraGpu, LinkKind::HostGpu, LinkKind::InterNode})
      std::printf("transfer %s 0=%.17g 16GiB=%.17g 32GiB=%.17g eff=%.17g\n", to_string(k),
                  transfer_time(0, k, t), transfer_time(16 * kGiB, k, t),
                  transfer_time(32 * kGiB, k, t), effective_bandwidth(t, k));
  }

  const std::vector<std::pair<int, int>> topos{{1, 1}, {2, 1}, {1, 2}, {2, 2}, {4, 1},
                                               {1, 4}, {1, 8}, {2, 4}, {4, 2}};
  const std::vector<std::string> nics{"ib100-rdma-measured", "ib100-ipoib-measured",
                                      "eth10g-measured", "eth1g-measured", "eth100g-theoretical"};

  for (const NamedModel& nm : models()) {
    const ModelSpec& m = nm.model;
    std::printf("model %s L=%d W=%" PRId64 " Wt=%" PRId64 " Wf=%" PRId64 " bytesW=%" PRIu64
                " bytesWt=%" PRIu64 " bytesWf=%" PRIu64 " act=%" PRIu64 "\n",
                nm.name.c_str(), m.num_layers(), m.total_params(), m.trainable_params(),
                m.frozen_params(), param_bytes(m), trainable_param_bytes(m), frozen_param_bytes(m),
                activation_bytes_per_sample_total(m));
    const std::vector<ParamState> init = init_param_states(m);
    std::printf("  portions=%zu\n", init.size());

    for (auto [N, g] : topos) {
      for (const NamedPlan& np : plans()) {
        const StrategyPlan& plan = np.plan;
        ClusterTopology topo = make_topology(N, g);
        try {
          plan.validate(topo);
        } catch (const ConfigError& e) {
          std::printf("  %dx%d %s invalid: %s\n", N, g, np.name.c_str(), e.what());
          continue;
        }
        const MemoryFootprint fp = memory_footprint(plan, m, topo);
        std::printf("  %dx%d %s shard=%" PRIu64 " grad=%" PRIu64 " opt=%" PRIu64 " pers=%" PRIu64
                    " cache=%" PRIu64 " trans=%" PRIu64 " host=%" PRIu64 " total=%" PRIu64 "\n",
                    N, g, np.name.c_str(), fp.gpu_param_shard_bytes, fp.gpu_gradient_bytes,
                    fp.gpu_optimizer_bytes, fp.gpu_persistent_bytes, fp.gpu_cache_bytes,
                    fp.gpu_transient_peak_bytes, fp.host_cache_bytes_per_node, fp.gpu_total_bytes());
        for (std::uint64_t cap : {0ull, 48ull * kGiB, 180ull * kGiB}) {
          const BatchSearchResult b = max_feasible_batch(plan, m, topo, cap);
          std::printf("    maxbatch cap=%" PRIu64 " b=%d oom=%d\n", cap, b.max_batch, b.oom_at_batch_1 ? 1 : 0);
        }
        for (const std::string& nic : nics) {
          const ClusterTopology t2 = make_topology(N, g, "nvlink3-theoretical", "pcie4-measured", nic);
          std::printf("    est %s %.17g\n", nic.c_str(), iteration_time_estimate(plan, m, t2));
        }
        for (bool prefetch : {true, false}) {
          for (std::uint64_t cap : {0ull, 2048ull, 12000ull, 24ull * kGiB}) {
            if (!prefetch && cap != 0) continue;
            BuildOptions opts;
            opts.prefetch = prefetch;
            opts.gpu_capacity_bytes = cap;
            std::vector<ParamState> st = init;
            for (std::uint64_t it = 1; it <= 3; ++it) {
              char tag[64];
              std::snprintf(tag, sizeof tag, "    it=%" PRIu64 " vol", it);
              print_volume(tag, comm_volume(plan, m, topo, it));
              const EventProgram prog = build_iteration(plan, m, topo, st, it, opts);
              const std::string text = serialize_program(prog);
              std::string ann;
              for (std::size_t l = 0; l < prog.layer_retained.size(); ++l)
                ann += char('0' + prog.layer_retained[l] + 2 * prog.layer_clean_path[l] +
                             4 * prog.layer_dirty_path[l]);
              std::printf("    prog prefetch=%d cap=%" PRIu64 " it=%" PRIu64 " events=%zu hash=%016" PRIx64
                          " ann=%s\n",
                          prefetch ? 1 : 0, cap, it, prog.events.size(), fnv1a(text), ann.c_str());
              if (nm.full_text && (N == 2 && g == 1)) std::fputs(text.c_str(), stdout);
              st = step_state(st, prog);
              std::string s;
              for (const ParamState& p : st) {
                char b[96];
                std::snprintf(b, sizeof b, "[%d%c v%" PRIu64 " d%d h%s g%d]", p.layer, p.frozen ? 'f' : 't',
                              p.version, p.dirty ? 1 : 0,
                              p.host_cached_version ? std::to_string(*p.host_cached_version).c_str() : "-",
                              p.gpu_cached ? 1 : 0);
                s += b;
              }
              if (s.size() > 400) s = "hash:" + std::to_string(fnv1a(s));
              std::printf("    state %s\n", s.c_str());
            }
          }
        }
      }
    }
  }

  // Error behaviour.
  expect_error("unknown link preset", [] { link_preset("nope"); });
  expect_error("wrong link class", [] { make_topology(2, 2, "pcie4-measured"); });
  expect_error("zero nodes", [] { make_topology(0, 2); });
  expect_error("zero gpus", [] { make_topology(1, 0); });
  expect_error("unknown link kind", [] { link_kind_from_string("x"); });
  expect_error("unknown duplex", [] { duplex_from_string("x"); });
  expect_error("unknown model", [] { model_preset("gpt99b"); });
  expect_error("lora 0", [] { apply_lora_mask(model_preset("gpt10b"), 0.0); });
  expect_error("lora >1", [] { apply_lora_mask(model_preset("gpt10b"), 1.5); });
  expect_error("empty model", [] { ModelSpec m; m.validate(); });
  expect_error("bad dtype", [] { ModelSpec m = uniform(1, 10, 3); m.validate(); });
  expect_error("bad count", [] { ModelSpec m = uniform(1, 0, 2); m.validate(); });
  expect_error("bad frac", [] { ModelSpec m = uniform(1, 10, 2, 1.5); m.validate(); });
  expect_error("bad batch", [] { ModelSpec m = uniform(1, 10, 2); m.batch_per_gpu = 0; m.validate(); });
  expect_error("bad opt mult", [] { ModelSpec m = uniform(1, 10, 2); m.optimizer_state_multiplier = -1; m.validate(); });
  expect_error("bad act", [] { ModelSpec m = uniform(1, 10, 2); m.layers[0].activation_bytes_per_sample = -1; m.validate(); });
  expect_error("bad compute", [] { ModelSpec m = uniform(1, 10, 2); m.layers[0].fwd_compute_s_per_sample = -1; m.validate(); });
  expect_error("unknown strategy", [] { strategy_kind_from_string("zero4"); });
  expect_error("tau range", [] { StrategyPlan p; p.kind = StrategyKind::Fcdp; p.tau = 2; p.validate(make_topology(1, 1)); });
  expect_error("tau kind", [] { StrategyPlan p; p.tau = 0.5; p.validate(make_topology(1, 1)); });
  expect_error("host cache kind", [] { StrategyPlan p; p.host_cache_enabled = true; p.validate(make_topology(1, 1)); });
  expect_error("subgroup kind", [] { StrategyPlan p; p.subgroup_size = 2; p.validate(make_topology(1, 2)); });
  expect_error("mics divide", [] { StrategyPlan p; p.kind = StrategyKind::MiCS; p.subgroup_size = 3; p.validate(make_topology(2, 4)); });
  expect_error("mics multiple", [] { StrategyPlan p; p.kind = StrategyKind::MiCS; p.subgroup_size = 6; p.validate(make_topology(3, 4)); });
  expect_error("iteration 0", [] {
    ModelSpec m = uniform(2, 10, 2);
    build_iteration(StrategyPlan{}, m, make_topology(1, 1), init_param_states(m), 0);
  });
  expect_error("state layout", [] {
    ModelSpec m = uniform(2, 10, 2);
    build_iteration(StrategyPlan{}, m, make_topology(1, 1), {}, 1);
  });
  expect_error("frozen version", [] {
    ModelSpec m = uniform(1, 10, 2, 0.5);
    auto st = init_param_states(m);
    st[1].version = 1;
    build_iteration(StrategyPlan{}, m, make_topology(1, 1), st, 1);
  });
  expect_error("clean empty cache", [] {
    ModelSpec m = uniform(1, 10, 2);
    auto st = init_param_states(m);
    st[0].dirty = false;
    StrategyPlan p;
    p.kind = StrategyKind::Fcdp;
    build_iteration(p, m, make_topology(1, 1), st, 1);
  });
  expect_error("dirty but fresh", [] {
    ModelSpec m = uniform(1, 10, 2);
    auto st = init_param_states(m);
    st[0].host_cached_version = 0;
    StrategyPlan p;
    p.kind = StrategyKind::FcdpComm;
    build_iteration(p, m, make_topology(1, 1), st, 1);
  });
  expect_error("zero3 ignores cache flags", [] {
    ModelSpec m = uniform(1, 10, 2);
    auto st = init_param_states(m);
    st[0].dirty = false;
    build_iteration(StrategyPlan{}, m, make_topology(1, 1), st, 1);
  });
  std::printf("param_state_index missing=%d\n", param_state_index(init_param_states(uniform(2, 10, 2)), 5, false));
  return 0;
}
