// Times the control-plane part of a training step - build_iteration +
// step_state + comm_volume - through the shardsim API only, so the same source
// links against the reference's compiled sources (oracle/_ref/time_ref, the
// "reference control plane timed on the host" of BASELINE.md §3) and against
// libfcdp.so (oracle/_ref/time_ours).
//
//   time_ref <strategy> <nodes> <gpus> <iterations> <elem_bytes> <params...>
// prints {"us_per_step": ..., "steps": ..., "events_per_step": ...}
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "shardsim/costmodel.hpp"
#include "shardsim/schedule.hpp"

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s strategy nodes gpus iterations elem_bytes params...\n", argv[0]);
    return 2;
  }
  using namespace shardsim;
  StrategyPlan plan;
  plan.kind = strategy_kind_from_string(argv[1]);
  const ClusterTopology topo = make_topology(std::atoi(argv[2]), std::atoi(argv[3]));
  const int iters = std::atoi(argv[4]);
  ModelSpec model;
  model.param_bytes_per_element = std::atoi(argv[5]);
  for (int i = 6; i < argc; ++i) {
    LayerSpec l;
    l.layer_id = i - 6;
    l.param_count = std::atoll(argv[i]);
    model.layers.push_back(l);
  }
  std::vector<ParamState> states = init_param_states(model);
  std::uint64_t events = 0, sink = 0;
  for (int it = 1; it <= 50; ++it) {  // warm-up: page in code, allocator
    std::vector<ParamState> scratch = init_param_states(model);
    sink += build_iteration(plan, model, topo, scratch, static_cast<std::uint64_t>(it)).events.size();
  }
  sink = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 1; it <= iters; ++it) {
    const EventProgram prog = build_iteration(plan, model, topo, states, static_cast<std::uint64_t>(it));
    states = step_state(std::move(states), prog);
    sink += comm_volume(plan, model, topo, static_cast<std::uint64_t>(it)).inter_total();
    events += prog.events.size();
  }
  const double us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
  std::printf("{\"us_per_step\": %.3f, \"steps\": %d, \"events_per_step\": %.1f, \"check\": %llu}\n", us, iters,
              static_cast<double>(events) / iters, static_cast<unsigned long long>(sink % 1000003));
  return 0;
}
