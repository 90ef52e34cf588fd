// Temporary: engine entry points (filled in by engine.cpp).
#include "capi_util.hpp"
#include "fcdp.h"

using fcdp::guarded;

extern "C" {
#define NOT_YET return guarded([] { throw std::runtime_error("engine: not implemented yet"); })
int fcdp_engine_create(const fcdp_engine_config*, const fcdp_model*, const fcdp_topology*, const fcdp_plan*,
                       const uint8_t* const*, fcdp_engine**) { NOT_YET; }
int fcdp_engine_init_params(fcdp_engine*, uint64_t, const fcdp_init_range* const*, const int32_t*) { NOT_YET; }
int fcdp_engine_set_adam(fcdp_engine*, const fcdp_adam_config*) { NOT_YET; }
int fcdp_engine_set_compute(fcdp_engine*, fcdp_compute_fn, void*) { NOT_YET; }
int fcdp_engine_run(fcdp_engine*, const fcdp_program*, fcdp_states*) { NOT_YET; }
int fcdp_engine_sync(fcdp_engine*) { NOT_YET; }
int fcdp_engine_barrier(fcdp_engine*) { NOT_YET; }
int fcdp_engine_streams(fcdp_engine*, void**) { NOT_YET; }
int fcdp_engine_counters(fcdp_engine*, int32_t, fcdp_counters*) { NOT_YET; }
int fcdp_engine_reset_counters(fcdp_engine*) { NOT_YET; }
int fcdp_engine_read_shard(fcdp_engine*, int32_t, int32_t, void*, size_t) { NOT_YET; }
int fcdp_engine_read_master(fcdp_engine*, int32_t, float*, size_t) { NOT_YET; }
int fcdp_engine_read_grad(fcdp_engine*, int32_t, float*, size_t) { NOT_YET; }
int fcdp_engine_read_host_cache(fcdp_engine*, int32_t, int32_t, void*, size_t) { NOT_YET; }
int fcdp_engine_last_gathered(fcdp_engine*, int32_t, void*, size_t) { NOT_YET; }
void fcdp_engine_destroy(fcdp_engine*) {}
}
