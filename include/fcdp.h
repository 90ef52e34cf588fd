/*
 * fcdp.h - C ABI of the B200-native FCDP parameter-movement hot path.
 *
 * The reference (arxiv 2602.06499, `shardsim`, /root/reference/proj) is a
 * C++20 library with no FFI of its own: its public surface is the set of free
 * functions and value types in proj/include/shardsim/ (*.hpp).  This header is
 * the C boundary a maintainer binds (ctypes / cgo / JNI) to reach
 *
 *   (1) that control plane, re-implemented from scratch behind the same C++
 *       headers (include/shardsim/), flattened to plain C types, and
 *   (2) the data plane the reference only describes (PAPER.md:431-549,
 *       SPEC.md:315-376): an HBM shard store with a pinned host-cache tier,
 *       NVLink gathers fused with PEFT expansion, a throttled host-staged NIC
 *       emulator between emulated nodes, FCDP-Cache D2H/H2D, and a gradient
 *       reduce-scatter fused with fp32 accumulation, cast and 1/G scaling.
 *
 * Conventions
 *   - Every function returns int: FCDP_OK (0) or a negative FCDP_ERR_* code.
 *     fcdp_last_error() returns a thread-local message for the last failure.
 *     No C++ exception crosses this boundary.  Reference ConfigError maps to
 *     FCDP_ERR_CONFIG and ProtocolError to FCDP_ERR_PROTOCOL (error.hpp:10-20).
 *   - Device pointers are plain `void*`; streams are `void*` (a cudaStream_t).
 *   - Nothing here falls back to the CPU: data-plane entry points fail with
 *     FCDP_ERR_CUDA when no device is present.
 */
#ifndef FCDP_H_
#define FCDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

/* ------------------------------------------------------------------ status */
#define FCDP_OK 0
#define FCDP_ERR_CONFIG (-1)   /* shardsim::ConfigError */
#define FCDP_ERR_PROTOCOL (-2) /* shardsim::ProtocolError, freshness violations */
#define FCDP_ERR_CUDA (-3)     /* CUDA runtime / driver failure, no device */
#define FCDP_ERR_OOM (-4)      /* device or pinned-host allocation failed */
#define FCDP_ERR_INTERNAL (-5)
#define FCDP_ERR_TIMEOUT (-6)  /* a cross-rank wait exceeded its deadline */

const char* fcdp_last_error(void);
const char* fcdp_version(void);

/* ============================================================ control plane
 * Flattened shardsim API.  Enum integer values follow declaration order in
 * the reference headers.
 */

/* shardsim::StrategyKind (strategy.hpp:11) */
enum { FCDP_ZERO2 = 0, FCDP_ZERO3 = 1, FCDP_MICS = 2, FCDP_ZEROPP = 3, FCDP_FCDP = 4, FCDP_FCDP_COMM = 5 };
/* shardsim::EventKind (schedule.hpp:14-25) */
enum {
  FCDP_EV_AG_INTER = 0, FCDP_EV_AG_INTRA = 1, FCDP_EV_H2D = 2, FCDP_EV_D2H = 3,
  FCDP_EV_COMPUTE_FWD = 4, FCDP_EV_COMPUTE_BWD = 5, FCDP_EV_REDUCE_SCATTER = 6,
  FCDP_EV_OPTIMIZER_STEP = 7, FCDP_EV_MASK_DIRTY = 8, FCDP_EV_BROADCAST = 9
};
/* shardsim::ParamSet (schedule.hpp:27) */
enum { FCDP_SET_ALL = 0, FCDP_SET_TRAINABLE = 1, FCDP_SET_FROZEN = 2 };

/* shardsim::LinkClass / ClusterTopology (topology.hpp:16-36); index 0 = IntraGpu,
 * 1 = HostGpu, 2 = InterNode (LinkKind order). duplex: 0 full, 1 half. */
typedef struct fcdp_topology {
  int32_t num_nodes;
  int32_t gpus_per_node;
  double bandwidth_bytes_per_s[3];
  double latency_s[3];
  int32_t duplex[3];
} fcdp_topology;

/* shardsim::StrategyPlan (strategy.hpp:16-34) */
typedef struct fcdp_plan {
  int32_t kind;
  int32_t subgroup_size;
  double tau;
  int32_t host_cache_enabled;
} fcdp_plan;

/* shardsim::CommVolume (costmodel.hpp:14-26) */
typedef struct fcdp_comm_volume {
  uint64_t fwd_ag_inter, bwd_ag_inter, reduce_scatter_inter, param_sync_inter;
  uint64_t intra_node_total, h2d_total, d2h_total;
} fcdp_comm_volume;

/* shardsim::MemoryFootprint (strategy.hpp:37-49) */
typedef struct fcdp_memory_footprint {
  uint64_t gpu_param_shard_bytes, gpu_gradient_bytes, gpu_optimizer_bytes, gpu_persistent_bytes;
  uint64_t gpu_cache_bytes, gpu_transient_peak_bytes, host_cache_bytes_per_node;
} fcdp_memory_footprint;

/* shardsim::ParamState (schedule.hpp:43-50); host_cached_version < 0 = nullopt */
typedef struct fcdp_param_state {
  int32_t layer;
  int32_t frozen;
  uint64_t version;
  int32_t dirty;
  int64_t host_cached_version;
  int32_t gpu_cached;
} fcdp_param_state;

/* shardsim::Event (schedule.hpp:31-38) without its deps vector */
typedef struct fcdp_event {
  uint32_t id;
  int32_t kind;
  int32_t layer;
  int32_t param_set;
  uint64_t bytes_total;
  uint32_t num_deps;
} fcdp_event;

typedef struct fcdp_model fcdp_model;       /* shardsim::ModelSpec */
typedef struct fcdp_states fcdp_states;     /* std::vector<shardsim::ParamState> */
typedef struct fcdp_program fcdp_program;   /* shardsim::EventProgram */

/* collective.hpp:19-33 */
uint64_t fcdp_ag_inter_bytes(uint64_t payload, int32_t scope_nodes);
uint64_t fcdp_ring_intra_bytes(uint64_t payload, int32_t ring_gpus);

/* topology.hpp:44-58 -> link_preset / make_topology / transfer_time */
int fcdp_link_preset(const char* name, int32_t* kind, double* bandwidth_bytes_per_s);
int fcdp_make_topology(int32_t num_nodes, int32_t gpus_per_node, const char* intra_preset,
                       const char* host_preset, const char* inter_preset, fcdp_topology* out);
int fcdp_transfer_time(uint64_t size_bytes, int32_t link_kind, const fcdp_topology* topo, double* out);

/* workload.hpp:13-54 -> ModelSpec construction, model_preset, apply_lora_mask */
int fcdp_model_create(int32_t num_layers, const int64_t* param_counts, const double* trainable_fraction,
                      int32_t param_bytes_per_element, double optimizer_state_multiplier,
                      int32_t batch_per_gpu, const double* fwd_compute_s_per_sample,
                      const double* bwd_compute_s_per_sample,
                      const int64_t* activation_bytes_per_sample, fcdp_model** out);
int fcdp_model_preset(const char* name, fcdp_model** out);
int fcdp_model_apply_lora_mask(const fcdp_model* model, double trainable_fraction, fcdp_model** out);
int fcdp_model_info(const fcdp_model* model, int32_t* num_layers, int64_t* total_params,
                    int64_t* trainable_params, int32_t* param_bytes_per_element);
int fcdp_model_layer_bytes(const fcdp_model* model, int32_t layer, uint64_t* all, uint64_t* trainable,
                           uint64_t* frozen);
void fcdp_model_destroy(fcdp_model* model);

/* strategy.hpp:51-65 */
int fcdp_strategy_from_string(const char* s, int32_t* kind);
int fcdp_memory_footprint_of(const fcdp_plan* plan, const fcdp_model* model, const fcdp_topology* topo,
                             fcdp_memory_footprint* out);
int fcdp_max_feasible_batch(const fcdp_plan* plan, const fcdp_model* model, const fcdp_topology* topo,
                            uint64_t gpu_capacity_bytes, int32_t* max_batch, int32_t* oom_at_batch_1);

/* costmodel.hpp:31-38 */
int fcdp_comm_volume_of(const fcdp_plan* plan, const fcdp_model* model, const fcdp_topology* topo,
                        uint64_t iteration, fcdp_comm_volume* out);
int fcdp_iteration_time_estimate(const fcdp_plan* plan, const fcdp_model* model,
                                 const fcdp_topology* topo, double* out);

/* schedule.hpp:72-92 */
int fcdp_states_init(const fcdp_model* model, fcdp_states** out);
int fcdp_states_create(int32_t count, fcdp_states** out); /* default-initialised list */
int fcdp_states_count(const fcdp_states* states, int32_t* count);
int fcdp_states_get(const fcdp_states* states, int32_t index, fcdp_param_state* out);
int fcdp_states_set(fcdp_states* states, int32_t index, const fcdp_param_state* in);
void fcdp_states_destroy(fcdp_states* states);
int fcdp_build_iteration(const fcdp_plan* plan, const fcdp_model* model, const fcdp_topology* topo,
                         const fcdp_states* states, uint64_t iteration_index, int32_t prefetch,
                         uint64_t gpu_capacity_bytes, fcdp_program** out);
int fcdp_step_state(fcdp_states* states, const fcdp_program* program); /* in place */
int fcdp_program_num_events(const fcdp_program* program, uint32_t* count);
int fcdp_program_event(const fcdp_program* program, uint32_t index, fcdp_event* out, uint32_t* deps,
                       uint32_t deps_capacity);
/* per-layer flags: bit0 retained, bit1 clean path, bit2 dirty path */
int fcdp_program_layer_flags(const fcdp_program* program, uint8_t* out, int32_t capacity);
/* serialize_program (schedule.hpp:83-85); *len receives the full length (incl. when truncated) */
int fcdp_program_serialize(const fcdp_program* program, char* buf, size_t capacity, size_t* len);
void fcdp_program_destroy(fcdp_program* program);
/* A program from an explicit event list (an external scheduler's program, or a
 * mutated one for the SPEC.md:389-409 mutation harness).  Event i must have
 * id i; deps of event i are deps[dep_offsets[i] .. dep_offsets[i+1]); flags as
 * fcdp_program_layer_flags.  The engine checks what it executes (freshness,
 * zero backward AgInter for the FCDP family) and answers FCDP_ERR_PROTOCOL. */
int fcdp_program_create(uint64_t iteration_index, int32_t strategy, uint32_t num_events,
                        const fcdp_event* events, const uint32_t* dep_offsets, const uint32_t* deps,
                        int32_t num_layers, const uint8_t* layer_flags, fcdp_program** out);

/* ============================================================== data plane
 * Layer layout.  A layer is a flat natural-order buffer of E elements of
 * `elem_bytes` (2: bf16, 4: fp32), seen as C = E*elem/16 16-byte chunks.  The
 * PEFT trainable mask is chunk-granular (one flag per 16 B).  Trainable and
 * frozen chunks form two portion vectors (mask-order compaction), each padded
 * to a multiple of G chunks and split G ways: global shard r = j*N + n lives
 * on the GPU (node n, local j); intra slice j = shards j*N .. j*N+N-1 is
 * contiguous.  (shardsim ParamState portions, schedule.hpp:43-50.)
 */
typedef struct fcdp_layout fcdp_layout;

/* chunk_mask: host array of num_chunks bytes (non-zero = trainable). */
int fcdp_layout_create(int64_t num_chunks, const uint8_t* chunk_mask, int32_t elem_bytes,
                       int32_t num_nodes, int32_t gpus_per_node, fcdp_layout** out);
/* portion chunk counts and padded shard/slice sizes (in chunks) */
int fcdp_layout_info(const fcdp_layout* layout, int64_t* trainable_chunks, int64_t* frozen_chunks,
                     int64_t* shard_t, int64_t* shard_f, int64_t* slice_t, int64_t* slice_f);
void fcdp_layout_destroy(fcdp_layout* layout);

/* Stateless kernels (device pointers; `stream` is a cudaStream_t). ----------
 * fcdp_partition:  natural -> (trainable portion, frozen portion); warp-ballot
 *                  compaction by the chunk mask.  t / f hold >= padded sizes.
 * fcdp_expand:     (g slice pointers per portion, each possibly a peer GPU's
 *                  memory) -> natural layer; only portions in `param_set`
 *                  are written.  This is the intra-node all-gather fused with
 *                  the PEFT expansion (Alg. 1 lines 14-15).
 * fcdp_rs_slice:   intra-node reduce-scatter of the trainable gradient: reads
 *                  slice j's trainable chunks from g natural-layout gradient
 *                  buffers (peer pointers), fp32 sum in fixed order 0..g-1,
 *                  compacts.  Chunks of shard (j*N + n) go to own_out as fp32
 *                  (times `scale` when `final_scale` != 0); the other shards
 *                  go to wire_out in the parameter dtype (RNE) for the
 *                  inter-node hop.
 * fcdp_rs_finalize: out[i] = scale * sum_{m=0..N-1} part_m[i] in fixed order,
 *                  part_n = own (fp32), part_m = wire[m] (parameter dtype).
 * fcdp_adam_step:  AdamW on fp32 master/m/v with an fp32 grad; writes the
 *                  parameter shard in its dtype.  Bit-exact vs oracle.
 * fcdp_init_portion_shard: deterministic counter-based init of one shard.
 */
int fcdp_partition(const fcdp_layout* layout, const void* natural, void* trainable, void* frozen,
                   void* stream);
int fcdp_expand(const fcdp_layout* layout, const void* const* t_slices, const void* const* f_slices,
                void* natural, int32_t param_set, void* stream);
int fcdp_rs_slice(const fcdp_layout* layout, const void* const* grads, int32_t local_rank,
                  int32_t node, float scale, int32_t final_scale, float* own_out, void* wire_out,
                  void* stream);
int fcdp_rs_finalize(int64_t n_elems, int32_t num_nodes, int32_t node, int32_t elem_bytes,
                     const float* own, const void* wire, int64_t wire_stride_elems, float scale,
                     float* out, void* stream);

typedef struct fcdp_adam_config {
  float lr, beta1, beta2, eps, weight_decay;
  int32_t step; /* 1-based step for bias correction */
} fcdp_adam_config;
int fcdp_adam_step(int64_t n, const fcdp_adam_config* cfg, float* master, float* m, float* v,
                   const float* grad, void* param, int32_t param_elem_bytes, void* stream);
/* Driving-model LayerNorm (not the parameter-movement path; bf16 rows of h
 * elements, h a multiple of 256 and <= 2048, fp32 statistics): forward writes y
 * and per-row mean / rstd; backward writes dx and (if dw, db are non-NULL) the
 * gamma / beta gradients through a deterministic two-stage column reduction in
 * `scratch` (2 * splits * h floats). */
int fcdp_layernorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* w, const void* b, void* y,
                       float* mean, float* rstd, void* stream);
int fcdp_layernorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* mean,
                       const float* rstd, void* dx, void* dw, void* db, float* scratch, int32_t splits,
                       void* stream);

/* Residual add fused into the LayerNorm: s = x + r (bf16, written to s_out) and
 * y = LN(s) in one pass; backward with the residual's downstream gradient dres
 * added into dx (nullable: plain LayerNorm backward). */
int fcdp_add_layernorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* r, const void* w,
                           const void* b, void* s_out, void* y, float* mean, float* rstd, void* stream);
int fcdp_layernorm_bwd_res(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* mean,
                           const float* rstd, const void* dres, void* dx, void* dw, void* db, float* scratch,
                           int32_t splits, void* stream);
/* Driving-model Llama RMSNorm (bf16 rows, h a multiple of 1024 and <= 8192, fp32
 * statistics): y = x * rsqrt(mean(x^2) + eps) * w and per-row rstd; with r and
 * s_out the input is the residual sum s = x + r (bf16, written to s_out).
 * Backward: dx (+ dres, nullable) and, if dw != NULL, dgamma through `scratch`
 * (splits * h floats). */
int fcdp_rmsnorm_fwd(int64_t rows, int32_t h, float eps, const void* x, const void* r, const void* w, void* s_out,
                     void* y, float* rstd, void* stream);
int fcdp_rmsnorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w, const float* rstd,
                     const void* dres, void* dx, void* dw, float* scratch, int32_t splits, void* stream);
/* Driving-model bias gradient (bf16 [rows x cols], cols a multiple of 8 and
 * <= 16384): db[c] = sum_r dy[r, c] in fp32; row-split partials in `scratch`
 * (splits * cols floats; splits from fcdp_colsum_splits), summed in split order
 * by the last block of each column group (deterministic, one launch). */
int fcdp_colsum_splits(int64_t rows, int32_t cols);
int fcdp_bias_grad(int64_t rows, int32_t cols, const void* dy, void* db, float* scratch, int32_t splits,
                   void* stream);
/* Driving-model MLP activation: y = gelu_tanh(h + b) (bias add fused), and its
 * backward dh = dy * gelu'(h + b) fused with db = sum_r dh (scratch as above). */
int fcdp_bias_gelu_fwd(int64_t rows, int32_t cols, const void* h, const void* b, void* y, void* stream);
int fcdp_bias_gelu_bwd(int64_t rows, int32_t cols, const void* dy, const void* h, const void* b, void* dh, void* db,
                       float* scratch, int32_t splits, void* stream);
/* Driving-model LM head loss: cross-entropy of bf16 logit rows (vocab a
 * multiple of 8; label < 0 = ignored row).  Forward writes per-row loss and
 * log-sum-exp; backward writes dlogits = (softmax - onehot) * scale[0] (scale:
 * a device fp32 scalar, e.g. grad / valid rows) into a separate buffer. */
int fcdp_xent_fwd(int64_t rows, int32_t vocab, const void* logits, const int64_t* labels, float* loss, float* lse,
                  void* stream);
int fcdp_xent_bwd(int64_t rows, int32_t vocab, const void* logits, const int64_t* labels, const float* lse,
                  const float* scale, void* dlogits, void* stream);

/* Driving-model Llama blocks: rotary embedding of x [batch, seq, heads, dim]
 * (bf16; pairs (2i, 2i+1); fp32 cos / sin tables [seq, dim / 2]; inverse != 0
 * rotates back - the backward; x_stride / y_stride = elements between tokens,
 * 0 = heads * dim), and SwiGLU y = silu(g) * u over [rows x f]
 * with its backward (row strides in elements, multiples of 8, so g and u may
 * be the two halves of one [rows x 2f] GEMM output). */
int fcdp_rope(int64_t batch, int32_t seq, int32_t heads, int32_t dim, const void* x, int64_t x_stride,
              const float* cos_table, const float* sin_table, int32_t inverse, void* y, int64_t y_stride,
              void* stream);
int fcdp_swiglu_fwd(int64_t rows, int32_t f, const void* g, int64_t g_stride, const void* u, int64_t u_stride, void* y,
                    void* stream);
int fcdp_swiglu_bwd(int64_t rows, int32_t f, const void* dy, const void* g, int64_t g_stride, const void* u,
                    int64_t u_stride, void* dg, int64_t dg_stride, void* du, int64_t du_stride, void* stream);

/* rows x row_bytes strided device copy (pitches in bytes; pointers, row bytes and
 * pitches multiples of 16): e.g. the v third of a joint q|k|v projection. */
int fcdp_copy_rows(int64_t rows, int64_t row_bytes, const void* src, int64_t src_pitch, void* dst, int64_t dst_pitch,
                   void* stream);
/* n device copies (src[i] -> dst[i], bytes[i]; 16-byte aligned, sizes multiples
 * of 16) in ceil(n / 32) kernel launches: the gradient hand-off of a masked
 * (LoRA) layer into the engine's natural gradient slot. */
int fcdp_copy_segments(int32_t n, const void* const* src, void* const* dst, const int64_t* bytes, void* stream);

/* Driving-model GPT-2 MLP GEMMs with fused cuBLASLt epilogues (bf16, row-major):
 * forward act = gelu_tanh(x W^T + b) with aux = x W^T + b kept for the backward;
 * backward of the second linear's input gradient dpre = (dy W2) * gelu'(aux) with
 * db1 = sum over rows of dpre.  libcublasLt is resolved at run time;
 * fcdp_mlp_gemm_available() = 0 when it cannot be (the calls then answer
 * FCDP_ERR_CONFIG). */
int fcdp_mlp_gemm_available(void);
int fcdp_fc_gelu_fwd(int64_t rows, int64_t in, int64_t out, const void* x, const void* w, const void* b, void* act,
                     void* aux, void* stream);
int fcdp_fc2_dgrad_dgelu(int64_t rows, int64_t hidden, int64_t ffn, const void* dy, const void* w2, const void* aux,
                         void* dpre, void* db1, void* stream);

/* Kernels launched so far through the driving-model and copy entry points above
 * (the engine's own launches are in fcdp_engine_kernel_stats); reset != 0 zeroes it. */
uint64_t fcdp_model_kernel_launches(int32_t reset);

/* Let kernels launched on `device` dereference `peer`'s memory over NVLink
 * (single-process multi-GPU use of the stateless kernels; the engine itself
 * maps peers through CUDA IPC). */
int fcdp_enable_peer_access(int32_t device, int32_t peer);
/* G = 1 fused reduce-scatter + AdamW of a dense layer (the engine's path at one
 * GPU): the gradient in the parameter dtype from segments (element offset,
 * pointer, count; 16-byte aligned; uncovered elements have gradient 0),
 * g = (0 + x) * scale, then AdamW - bit-identical to fcdp_rs_slice (g = 1,
 * final scale) followed by fcdp_adam_step.  keep_grad (nullable) receives g. */
int fcdp_adam_grad_step(int64_t n, const fcdp_adam_config* cfg, float scale, int32_t num_segs,
                        const int64_t* elem_offsets, const void* const* grads, const int64_t* counts,
                        float* master, float* m, float* v, void* param, int32_t param_elem_bytes,
                        float* keep_grad, void* stream);

/* Init spec: element ranges of the natural layer with a rule each.
 * kind 0: uniform(-scale, scale) from splitmix64(seed, layer, element)
 * kind 1: constant `scale`.  Elements not covered are zero. */
typedef struct fcdp_init_range {
  int64_t begin, end;
  int32_t kind;
  float scale;
} fcdp_init_range;
int fcdp_init_natural(const fcdp_layout* layout, uint64_t seed, int32_t layer,
                      const fcdp_init_range* ranges, int32_t num_ranges, void* natural, void* stream);

/* ================================================================== engine
 * One engine per process, one process per GPU.  Ranks are numbered
 * node-major: rank = n * gpus_per_node + j.  Ranks of one job share a
 * POSIX shared-memory control block named `shm_name` that carries the
 * cross-rank signals, the NIC emulators' pacing state and byte counters, the
 * inter-node staging slots, and the CUDA IPC handles of every rank's
 * peer-visible buffers.
 */
typedef struct fcdp_engine fcdp_engine;

typedef struct fcdp_engine_config {
  const char* shm_name;     /* identical on every rank of the job */
  int32_t rank, world_size; /* world_size == num_nodes * gpus_per_node */
  int32_t device;           /* CUDA ordinal of this rank */
  int32_t x_slots;          /* slice buffer slots (>= 2; default 3) */
  int32_t inter_slots;      /* NIC staging ring depth in pieces (>= 4; default 16) */
  int32_t nic_pacing;       /* 1: pace inter-node traffic at topology inter bandwidth */
  int32_t use_copy_engine;  /* 1: dense intra gathers by cudaMemcpyAsync (CE) not SM kernels */
  double timeout_s;         /* deadline for host-side cross-rank waits */
  int64_t inter_chunk_bytes; /* NIC emulator wire piece size (0: 4 MiB); inter_slots = staging ring depth in pieces */
} fcdp_engine_config;

/* Counters of one rank (bytes).  Per node = sum over that node's ranks. */
typedef struct fcdp_counters {
  uint64_t nic_tx_fwd_ag, nic_tx_bwd_ag, nic_tx_rs;   /* bytes this rank put on its node's NIC */
  uint64_t nic_rx_fwd_ag, nic_rx_bwd_ag, nic_rx_rs;
  uint64_t nvlink_rx;                                  /* intra-node ingress (AG + RS) */
  uint64_t cache_h2d, cache_d2h;                       /* FCDP-Cache PCIe bytes */
  uint64_t staging_h2d, staging_d2h;                   /* NIC-emulator host staging bytes */
  uint64_t ag_inter_events_fwd, ag_inter_events_bwd;
  uint64_t nic_busy_ns;                                /* paced wire time charged by this rank */
  uint64_t resident_hits;  /* frozen reloads elided: portion already resident in a tau-retained buffer */
  uint64_t nic_tx_grad_sync, nic_rx_grad_sync;  /* MiCS: replica gradient all-reduce (not in comm_volume) */
} fcdp_counters;

/* Compute callback: `kind` FCDP_EV_COMPUTE_FWD/BWD.  `weights` is the natural
 * gathered layer (read-only), `grad_out` the natural gradient buffer to fill
 * in backward (NULL in forward).  Work must be enqueued on `stream`. */
typedef int (*fcdp_compute_fn)(void* user, int32_t kind, int32_t layer, const void* weights,
                               void* grad_out, void* stream);

int fcdp_engine_create(const fcdp_engine_config* cfg, const fcdp_model* model,
                       const fcdp_topology* topo, const fcdp_plan* plan,
                       const uint8_t* const* chunk_masks, fcdp_engine** out);
int fcdp_engine_init_params(fcdp_engine* e, uint64_t seed, const fcdp_init_range* const* ranges,
                            const int32_t* num_ranges);
int fcdp_engine_set_adam(fcdp_engine* e, const fcdp_adam_config* cfg);
int fcdp_engine_set_compute(fcdp_engine* e, fcdp_compute_fn fn, void* user);
/* Execute one program (built for this engine's plan/model/topology) and apply
 * step_state.  Asynchronous: returns once every event is enqueued.
 * The reference has no executor: it stops at build_iteration
 * (proj/src/schedule.cpp:341-352) and step_state (schedule.cpp:354-387).  The
 * event semantics executed here are Algorithm 1 and the
 * builder's event meanings (schedule.cpp:107-292). */
int fcdp_engine_run(fcdp_engine* e, const fcdp_program* program, fcdp_states* states);
/* Errors and engine state: an error while a program runs (a protocol violation,
 * a failed compute callback, an OOM, a cross-rank timeout) leaves this rank's
 * cross-rank sequence counters out of step with its peers.  The engine latches
 * the failure, raises the job's abort flag (peers waiting on this rank fail
 * fast with FCDP_ERR_TIMEOUT instead of reading stale data), and refuses every
 * later begin/run with FCDP_ERR_PROTOCOL: destroy and recreate it.  Every rank
 * must run the same program: begin compares a hash of the program with every
 * peer's and answers FCDP_ERR_CONFIG on a mismatch. */
/* The same, driven event by event by an external executor that walks
 * EventProgram.events in id order (SURVEY §8(b) caller): begin, then exec for
 * ids 0..n-1, then end (which applies step_state).  Each exec enqueues that
 * event's data movement - AgInter (pack + NIC + NVLink gather/unpack), AgIntra,
 * D2H (FCDP-Cache store), H2D (cache reload), ReduceScatter (fused cast/scale),
 * OptimizerStep (AdamW) - honouring its deps with stream waits.  Out-of-order
 * ids -> FCDP_ERR_PROTOCOL.  `program` must stay alive until end. */
int fcdp_engine_begin(fcdp_engine* e, const fcdp_program* program);
int fcdp_engine_exec(fcdp_engine* e, uint32_t event_id);
int fcdp_engine_end(fcdp_engine* e, fcdp_states* states);
int fcdp_engine_sync(fcdp_engine* e);
int fcdp_engine_barrier(fcdp_engine* e);
int fcdp_engine_streams(fcdp_engine* e, void** compute_stream);
int fcdp_engine_counters(fcdp_engine* e, int32_t rank, fcdp_counters* out);
int fcdp_engine_reset_counters(fcdp_engine* e);
/* NUMA placement of this rank's host side (multi-socket hosts): the GPU's
 * node (-1 unknown), online memory nodes, whether the host + NIC threads were
 * pinned to the GPU's node, and pinned host bytes given that node as preferred
 * (the FCDP-Cache tier).  FCDP_NUMA=0 disables placement. */
int fcdp_engine_numa(fcdp_engine* e, int32_t* gpu_node, int32_t* num_nodes, int32_t* cpus_bound,
                     uint64_t* bytes_bound);
/* Read back (device->host, synchronous) for tests: */
int fcdp_engine_read_shard(fcdp_engine* e, int32_t layer, int32_t frozen, void* host, size_t bytes);
int fcdp_engine_read_master(fcdp_engine* e, int32_t layer, float* host, size_t count);
int fcdp_engine_read_grad(fcdp_engine* e, int32_t layer, float* host, size_t count);
int fcdp_engine_read_host_cache(fcdp_engine* e, int32_t layer, int32_t frozen, void* host, size_t bytes);
void fcdp_engine_destroy(fcdp_engine* e);

/* Per-kernel-class launch counts, CUDA-event device time and algorithmic bytes
 * of the engine's own kernels.  Classes: 0 gather/expand (intra all-gather),
 * 1 reduce-scatter slice (pull-reduce), 2 reduce-scatter finalize, 3 AdamW,
 * 4 local shard copies (pack into the slice buffer, ZeRO++ replica); and the
 * host-link copies: 5 FCDP-Cache D2H, 6 FCDP-Cache H2D, 7 NIC staging D2H,
 * 8 NIC receive H2D (cudaMemcpyAsync, not kernels).
 * link_bytes: the part of the traffic that crossed NVLink (peer reads) for
 * classes 0-4, the PCIe bytes for classes 5-8. */
#define FCDP_KCLASSES 9
typedef struct fcdp_kernel_stats {
  uint64_t launches[FCDP_KCLASSES];
  double total_ms[FCDP_KCLASSES];  /* only while timing is on */
  uint64_t alg_bytes[FCDP_KCLASSES];
  uint64_t timed_launches[FCDP_KCLASSES];
  uint64_t link_bytes[FCDP_KCLASSES];
} fcdp_kernel_stats;
int fcdp_engine_set_timing(fcdp_engine* e, int32_t on);

/* One GPU (G = 1), dense trainable layer: the gradient reduce-scatter is the
 * identity up to its fp32 widen and 1/G scale, so the engine fuses it into
 * AdamW (cast/scale + update in one pass over the layer, per layer, right after
 * its backward).  The fused kernel can read the gradient straight from the
 * caller's own buffers: inside the backward compute callback of `layer`, call
 * fcdp_engine_grad_segments with up to 24 sorted, disjoint, 16-byte aligned
 * (offset, pointer, count) segments in the parameter dtype - elements no
 * segment covers have gradient 0 - instead of writing grad_out.  The buffers
 * must stay valid, and unwritten by work not ordered after the program's end
 * on the compute stream, until fcdp_engine_run / fcdp_engine_end returns.
 * takes_grad_segments answers whether `layer` qualifies (only inside a program;
 * otherwise FCDP_ERR_CONFIG from grad_segments: fill grad_out).
 * set_keep_grad(1): the fused path also writes the fp32 gradient shard (what
 * fcdp_engine_read_grad returns; tests), at 4 more bytes per parameter. */
int fcdp_engine_grad_segments(fcdp_engine* e, int32_t layer, int32_t n, const int64_t* elem_offsets,
                              const void* const* ptrs, const int64_t* counts);
int fcdp_engine_takes_grad_segments(fcdp_engine* e, int32_t layer, int32_t* out);
int fcdp_engine_set_keep_grad(fcdp_engine* e, int32_t on);
int fcdp_engine_kernel_stats(fcdp_engine* e, fcdp_kernel_stats* out, int32_t reset);

/* Executed-event trace of the last fcdp_engine_run (when tracing is on): for
 * every program event, the device time (ms, relative to the iteration start)
 * at which its stream reached it (begin) and finished it (end). */
int fcdp_engine_set_trace(fcdp_engine* e, int32_t on);
int fcdp_engine_trace(fcdp_engine* e, float* begin_ms, float* end_ms, uint32_t capacity, uint32_t* count);

/* NIC bandwidth profile (Fig. 10): when on, this rank's NIC emulator
 * records every payload it paces onto its node's emulated wire.  The drain call
 * returns up to `capacity` records made since the last call: the wire interval
 * [start_ns, end_ns) on steady_clock (the clock every rank's NIC shares), the
 * bytes, and the kind (0 = forward AgInter, 1 = backward AgInter, 2 =
 * inter-node reduce-scatter, 15 = MiCS/ZeRO++ gradient sync).  Payloads of one
 * node never overlap on its wire (one NIC per node, topology.hpp:23-25). */
int fcdp_engine_set_nic_log(fcdp_engine* e, int32_t on);
int fcdp_engine_nic_log(fcdp_engine* e, uint64_t* start_ns, uint64_t* end_ns, uint64_t* bytes, int32_t* kind,
                        uint32_t capacity, uint32_t* count);

/* Host-only NUMA placement checks (no GPU needed):
 * parse a sysfs cpulist ("0-3,8"); and for `node`: online memory nodes, its
 * CPU count, whether a preferred-node mbind of a fresh mapping succeeded, the
 * node its first page landed on after first touch, and whether a temporary
 * pin of the calling thread to the node was undone exactly (the engine pins
 * only during construction). */
int fcdp_numa_parse_cpulist(const char* list, int32_t* out, int32_t capacity, int32_t* count);
int fcdp_numa_selftest(int32_t node, uint64_t bytes, int32_t* num_nodes, int32_t* cpus_in_node,
                       int32_t* prefer_ok, int32_t* node_of_page, int32_t* affinity_restored);

/* Host-only protocol self-test (no GPU needed): attach the shared control
 * block, run `rounds` barrier-separated rounds in which every rank charges
 * `payload` bytes to its node's NIC emulator, return the wall time.  A node's
 * ranks serialise on its single NIC, nodes run in parallel. */
int fcdp_nic_selftest(const char* shm_name, int32_t rank, int32_t num_nodes, int32_t gpus_per_node,
                      double bytes_per_s, uint64_t payload, int32_t rounds, double* elapsed_s);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* FCDP_H_ */
