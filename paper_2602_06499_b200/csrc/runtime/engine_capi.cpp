// C ABI of the per-rank engine (include/fcdp.h, "engine").
#include "capi_util.hpp"
#include "fcdp.h"
#include "runtime/engine.hpp"

#include <sys/mman.h>

#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

struct fcdp_engine {
  fcdp::Engine* impl;
};

using fcdp::guarded;

namespace {
fcdp::Engine& E(fcdp_engine* e) {
  if (!e || !e->impl) throw shardsim::ConfigError("engine: null handle");
  return *e->impl;
}
}  // namespace

extern "C" {

int fcdp_engine_create(const fcdp_engine_config* cfg, const fcdp_model* model, const fcdp_topology* topo,
                       const fcdp_plan* plan, const uint8_t* const* masks, fcdp_engine** out) {
  return guarded([&] {
    auto* impl = new fcdp::Engine(*cfg, fcdp::model_from_c(model), fcdp::topo_from_c(topo),
                                  fcdp::plan_from_c(plan), masks);
    *out = new fcdp_engine{impl};
  });
}

int fcdp_engine_init_params(fcdp_engine* e, uint64_t seed, const fcdp_init_range* const* ranges,
                            const int32_t* num_ranges) {
  return guarded([&] { E(e).init_params(seed, ranges, num_ranges); });
}

int fcdp_engine_set_adam(fcdp_engine* e, const fcdp_adam_config* cfg) {
  return guarded([&] { E(e).set_adam(*cfg); });
}

int fcdp_engine_set_compute(fcdp_engine* e, fcdp_compute_fn fn, void* user) {
  return guarded([&] { E(e).set_compute(fn, user); });
}

int fcdp_engine_run(fcdp_engine* e, const fcdp_program* program, fcdp_states* states) {
  return guarded([&] { E(e).run(fcdp::program_from_c(program), fcdp::states_from_c(states)); });
}

int fcdp_engine_begin(fcdp_engine* e, const fcdp_program* program) {
  return guarded([&] { E(e).begin(fcdp::program_from_c(program)); });
}

int fcdp_engine_exec(fcdp_engine* e, uint32_t event_id) { return guarded([&] { E(e).exec(event_id); }); }

int fcdp_engine_end(fcdp_engine* e, fcdp_states* states) {
  return guarded([&] { E(e).end(fcdp::states_from_c(states)); });
}

int fcdp_engine_sync(fcdp_engine* e) { return guarded([&] { E(e).sync(); }); }
int fcdp_engine_barrier(fcdp_engine* e) { return guarded([&] { E(e).barrier(); }); }

int fcdp_engine_streams(fcdp_engine* e, void** compute_stream) {
  return guarded([&] { *compute_stream = E(e).compute_stream(); });
}

int fcdp_engine_counters(fcdp_engine* e, int32_t rank, fcdp_counters* out) {
  return guarded([&] { E(e).counters(rank, out); });
}

int fcdp_engine_numa(fcdp_engine* e, int32_t* gpu_node, int32_t* num_nodes, int32_t* cpus_bound,
                     uint64_t* bytes_bound) {
  return guarded([&] {
    const fcdp::NumaPlacement& p = E(e).numa();
    if (gpu_node) *gpu_node = p.gpu_node;
    if (num_nodes) *num_nodes = p.num_nodes;
    if (cpus_bound) *cpus_bound = p.cpus_bound ? 1 : 0;
    if (bytes_bound) *bytes_bound = p.bytes_bound;
  });
}

int fcdp_engine_reset_counters(fcdp_engine* e) { return guarded([&] { E(e).reset_counters(); }); }

int fcdp_engine_read_shard(fcdp_engine* e, int32_t layer, int32_t frozen, void* host, size_t bytes) {
  return guarded([&] { E(e).read_shard(layer, frozen != 0, host, bytes); });
}

int fcdp_engine_read_master(fcdp_engine* e, int32_t layer, float* host, size_t count) {
  return guarded([&] { E(e).read_master(layer, host, count); });
}

int fcdp_engine_read_grad(fcdp_engine* e, int32_t layer, float* host, size_t count) {
  return guarded([&] { E(e).read_grad(layer, host, count); });
}

int fcdp_engine_read_host_cache(fcdp_engine* e, int32_t layer, int32_t frozen, void* host, size_t bytes) {
  return guarded([&] { E(e).read_host_cache(layer, frozen != 0, host, bytes); });
}

int fcdp_engine_set_timing(fcdp_engine* e, int32_t on) { return guarded([&] { E(e).set_timing(on != 0); }); }

int fcdp_engine_grad_segments(fcdp_engine* e, int32_t layer, int32_t n, const int64_t* elem_offsets,
                              const void* const* ptrs, const int64_t* counts) {
  return guarded([&] { E(e).grad_segments(layer, n, elem_offsets, ptrs, counts); });
}

int fcdp_engine_takes_grad_segments(fcdp_engine* e, int32_t layer, int32_t* out) {
  return guarded([&] { *out = E(e).fused_grad_ok(layer) ? 1 : 0; });
}

int fcdp_engine_set_keep_grad(fcdp_engine* e, int32_t on) { return guarded([&] { E(e).set_keep_grad(on != 0); }); }

int fcdp_engine_kernel_stats(fcdp_engine* e, fcdp_kernel_stats* out, int32_t reset) {
  return guarded([&] { E(e).kernel_stats(out, reset != 0); });
}

int fcdp_engine_set_trace(fcdp_engine* e, int32_t on) { return guarded([&] { E(e).set_trace(on != 0); }); }

int fcdp_engine_trace(fcdp_engine* e, float* begin_ms, float* end_ms, uint32_t capacity, uint32_t* count) {
  return guarded([&] { *count = E(e).trace(begin_ms, end_ms, capacity); });
}

int fcdp_engine_set_nic_log(fcdp_engine* e, int32_t on) { return guarded([&] { E(e).set_nic_log(on != 0); }); }

int fcdp_engine_nic_log(fcdp_engine* e, uint64_t* start_ns, uint64_t* end_ns, uint64_t* bytes, int32_t* kind,
                        uint32_t capacity, uint32_t* count) {
  return guarded([&] {
    std::vector<fcdp::WireRecord> v(capacity);
    const std::size_t n = E(e).nic_log(v.data(), capacity);
    for (std::size_t i = 0; i < n; ++i) {
      start_ns[i] = v[i].start_ns;
      end_ns[i] = v[i].end_ns;
      bytes[i] = v[i].bytes;
      kind[i] = v[i].kind;
    }
    *count = static_cast<uint32_t>(n);
  });
}

int fcdp_numa_parse_cpulist(const char* list, int32_t* out, int32_t capacity, int32_t* count) {
  return guarded([&] {
    const std::vector<int> v = fcdp::parse_cpulist(list ? list : "");
    *count = static_cast<int32_t>(v.size());
    for (int32_t i = 0; i < capacity && i < static_cast<int32_t>(v.size()); ++i) out[i] = v[i];
  });
}

int fcdp_numa_selftest(int32_t node, uint64_t bytes, int32_t* num_nodes, int32_t* cpus_in_node,
                       int32_t* prefer_ok, int32_t* node_of_page, int32_t* affinity_restored) {
  return guarded([&] {
    *num_nodes = fcdp::numa_online_nodes();
    *cpus_in_node = static_cast<int32_t>(fcdp::numa_node_cpus(node).size());
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw fcdp::OomError("numa selftest: mmap failed");
    *prefer_ok = fcdp::numa_prefer(p, bytes, node) ? 1 : 0;
    std::memset(p, 1, bytes);  // first touch under the policy
    *node_of_page = fcdp::numa_node_of_page(p);
    munmap(p, bytes);
    const fcdp::SavedAffinity before = fcdp::numa_save_affinity();
    fcdp::numa_pin_thread(node);
    fcdp::numa_restore_affinity(before);
    const fcdp::SavedAffinity after = fcdp::numa_save_affinity();
    *affinity_restored = before.valid && after.valid && std::memcmp(before.set, after.set, sizeof(before.set)) == 0;
  });
}

int fcdp_nic_selftest(const char* name, int32_t rank, int32_t nodes, int32_t local, double bw, uint64_t payload,
                      int32_t rounds, double* elapsed) {
  return guarded([&] {
    fcdp::SharedBlock shm(name ? name : "", rank, nodes * local, nodes, local, 2, 4096, 60.0);
    shm.barrier(60.0);
    const std::uint64_t t0 = fcdp::SharedBlock::now_ns();
    const int node = rank / local;
    const auto ns = static_cast<std::uint64_t>(static_cast<double>(payload) / bw * 1e9);
    for (int i = 0; i < rounds; ++i) {
      const std::uint64_t finish = shm.reserve_nic(node, ns);
      while (fcdp::SharedBlock::now_ns() < finish) std::this_thread::sleep_for(std::chrono::microseconds(50));
      shm.add(rank, fcdp::kTxFwdAg, payload);
      shm.barrier(60.0);
    }
    *elapsed = static_cast<double>(fcdp::SharedBlock::now_ns() - t0) * 1e-9;
    std::uint64_t node_bytes = 0;
    for (int j = 0; j < local; ++j) node_bytes += shm.counter(node * local + j, fcdp::kTxFwdAg);
    if (node_bytes != payload * static_cast<std::uint64_t>(rounds) * static_cast<std::uint64_t>(local))
      throw std::runtime_error("nic selftest: node byte counter mismatch");
    shm.barrier(60.0);
  });
}

void fcdp_engine_destroy(fcdp_engine* e) {
  if (!e) return;
  delete e->impl;
  delete e;
}

}  // extern "C"
