/* A plain-C caller of the FCDP engine through include/fcdp.h only (no Python,
 * no torch): the reference-side host loop INTEGRATION.md §2 describes.
 *
 *   engine_driver <shm_name> <rank> <nodes> <gpus_per_node> <strategy>
 *
 * Builds a 3-layer bf16 model, runs 3 iterations of the reference-built
 * program on the engine with a compute callback that writes a constant
 * gradient (cudaMemsetAsync, byte 0x3C = bf16 0.011474609375 everywhere),
 * and checks, on this rank:
 *   - the NIC tx counters of the last iteration equal comm_volume (one GPU
 *     per node here, so a rank's counters are its node's);
 *   - AdamW with a constant gradient moves every fp32 master element by
 *     -lr per step (m_hat = g, v_hat = g^2), i.e. by -3 lr after 3 steps.
 * Prints "engine_driver ok ..." and exits 0, or prints the failure and exits 1.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "fcdp.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int rc_ = (x);                                                                \
    if (rc_ != FCDP_OK) {                                                         \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, fcdp_last_error());          \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

static int backward_calls = 0;

static int compute(void* user, int32_t kind, int32_t layer, const void* weights, void* grad_out, void* stream) {
  const int64_t* counts = (const int64_t*)user;
  (void)weights;
  if (kind == FCDP_EV_COMPUTE_BWD && grad_out) {
    ++backward_calls;
    return cudaMemsetAsync(grad_out, 0x3C, (size_t)counts[layer] * 2, (cudaStream_t)stream) == cudaSuccess ? 0 : -1;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 6) {
    fprintf(stderr, "usage: %s shm_name rank nodes gpus_per_node strategy\n", argv[0]);
    return 2;
  }
  const char* shm = argv[1];
  const int rank = atoi(argv[2]), nodes = atoi(argv[3]), g = atoi(argv[4]);
  const int world = nodes * g;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
    fprintf(stderr, "no CUDA device\n");
    return 1;
  }
  fcdp_topology topo;
  CHECK(fcdp_make_topology(nodes, g, NULL, NULL, "ib100-rdma-measured", &topo));
  int32_t kind = 0;
  CHECK(fcdp_strategy_from_string(argv[5], &kind));
  fcdp_plan plan = {kind, 0, 0.0, 0};
  enum { L = 3 };
  static int64_t counts[L] = {65536 * 8, 98304 * 8, 32768 * 8};  /* multiples of 8 * G elements */
  const double frac[L] = {1.0, 1.0, 1.0};
  fcdp_model* model = NULL;
  CHECK(fcdp_model_create(L, counts, frac, 2, 6.0, 1, NULL, NULL, NULL, &model));
  fcdp_engine_config cfg = {shm, rank, world, rank % ndev, 3, 16, 0, 0, 120.0, 0};
  fcdp_engine* eng = NULL;
  CHECK(fcdp_engine_create(&cfg, model, &topo, &plan, NULL, &eng));
  fcdp_init_range r0 = {0, counts[0], 0, 0.05f}, r1 = {0, counts[1], 0, 0.05f}, r2 = {0, counts[2], 0, 0.05f};
  const fcdp_init_range* ranges[L] = {&r0, &r1, &r2};
  const int32_t nranges[L] = {1, 1, 1};
  CHECK(fcdp_engine_init_params(eng, 0x5EED, ranges, nranges));
  const float lr = 1e-3f;
  fcdp_adam_config adam = {lr, 0.9f, 0.999f, 1e-8f, 0.0f, 1};
  CHECK(fcdp_engine_set_adam(eng, &adam));
  CHECK(fcdp_engine_set_compute(eng, compute, counts));

  /* this rank's fp32 master shard of layer 0 before training */
  const size_t shard0 = (size_t)(counts[0] / world);
  float* before = (float*)malloc(shard0 * sizeof(float));
  float* after = (float*)malloc(shard0 * sizeof(float));
  CHECK(fcdp_engine_read_master(eng, 0, before, shard0));

  fcdp_states* st = NULL;
  CHECK(fcdp_states_init(model, &st));
  const int K = 3;
  for (uint64_t it = 1; it <= (uint64_t)K; ++it) {
    fcdp_program* prog = NULL;
    CHECK(fcdp_build_iteration(&plan, model, &topo, st, it, 1, 0, &prog));
    if (it == (uint64_t)K) CHECK(fcdp_engine_reset_counters(eng));
    CHECK(fcdp_engine_run(eng, prog, st));
    CHECK(fcdp_engine_sync(eng));
    fcdp_program_destroy(prog);
  }
  fcdp_counters c;
  CHECK(fcdp_engine_counters(eng, rank, &c));
  fcdp_comm_volume vol;
  CHECK(fcdp_comm_volume_of(&plan, model, &topo, (uint64_t)K, &vol));
  int bad = 0;
  if (g == 1 && (c.nic_tx_fwd_ag != vol.fwd_ag_inter || c.nic_tx_bwd_ag != vol.bwd_ag_inter ||
                 c.nic_tx_rs != vol.reduce_scatter_inter)) {
    fprintf(stderr, "NIC counters %llu/%llu/%llu != comm_volume %llu/%llu/%llu\n",
            (unsigned long long)c.nic_tx_fwd_ag, (unsigned long long)c.nic_tx_bwd_ag, (unsigned long long)c.nic_tx_rs,
            (unsigned long long)vol.fwd_ag_inter, (unsigned long long)vol.bwd_ag_inter,
            (unsigned long long)vol.reduce_scatter_inter);
    bad = 1;
  }
  CHECK(fcdp_engine_read_master(eng, 0, after, shard0));
  double worst = 0.0;
  for (size_t i = 0; i < shard0; ++i) {
    const double d = fabs((double)after[i] - (double)before[i] + K * (double)lr);
    if (d > worst) worst = d;
  }
  if (worst > 1e-6) {
    fprintf(stderr, "AdamW step: worst |delta + %d lr| = %g\n", K, worst);
    bad = 1;
  }
  if (backward_calls != K * L) {
    fprintf(stderr, "backward callbacks %d != %d\n", backward_calls, K * L);
    bad = 1;
  }
  if (!bad)
    printf("engine_driver ok rank %d/%d %s: nic tx fwd %llu bwd %llu rs %llu, master delta err %.3g\n", rank, world,
           argv[5], (unsigned long long)c.nic_tx_fwd_ag, (unsigned long long)c.nic_tx_bwd_ag,
           (unsigned long long)c.nic_tx_rs, worst);
  fcdp_engine_barrier(eng);
  fcdp_engine_destroy(eng);
  fcdp_states_destroy(st);
  fcdp_model_destroy(model);
  free(before);
  free(after);
  return bad;
}
