/*
 * fcdp_oracle.h - CPU restatement of the FCDP data plane.  TEST INFRASTRUCTURE.
 *
 * This library is the checker, never the product: only tests/, the smoke()
 * entry in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The shipped path (paper_2602_06499_b200/libfcdp.so) never
 * links or calls it.
 *
 * Parity status: the reference (arxiv 2602.06499, /root/reference/proj) has
 * NO data plane - "payloads are byte counts only" (proj/include/shardsim/
 * schedule.hpp:31-38).  What these functions restate is the behaviour the
 * reference specifies in prose:
 *   - Algorithm 1, PAPER.md:503-549 (inter AG when dirty + host refresh; host
 *     reload + intra AG when clean; backward reload + intra AG; RS of W_t),
 *   - FCDP-Sched / -Cache / -Comm, PAPER.md:431-500,
 *   - the event semantics of proj/src/schedule.cpp:107-292 and the byte
 *     split of proj/include/shardsim/collective.hpp:19-33,
 *   - SPEC.md:242 (D2H stores the intra-node shard), SPEC.md:324-327 (payload
 *     = param, shard index, version, bytes).
 * Gathered / cached parameter bytes are pure copies, so their parity is
 * bit-exact by construction.  Reduction and optimizer arithmetic are defined
 * here (fixed summation order, explicit fmaf, RNE casts) and the CUDA kernels
 * must match them bit for bit; the reference pins none of that arithmetic
 * ("parity unpinned" for values beyond copies - see DESIGN.md).
 */
#ifndef FCDP_ORACLE_H_
#define FCDP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Portion geometry of one layer (chunk = 16 bytes). */
typedef struct fo_geom {
  int64_t chunks, pt, pf;        /* natural chunks, trainable, frozen */
  int64_t shard_t, shard_f;      /* per global shard (portion padded to G) */
  int64_t slice_t, slice_f;      /* per intra slice = N shards */
  int32_t nodes, local;
} fo_geom;

void fo_geom_of(int64_t chunks, const uint8_t* mask, int32_t nodes, int32_t local, fo_geom* out);

/* natural -> (t, f): mask-order compaction (FCDP-Comm). */
void fo_partition(int64_t chunks, const uint8_t* mask, const void* natural, void* t, void* f);

/* Full portion vectors -> natural (the inverse). */
void fo_unpartition(int64_t chunks, const uint8_t* mask, const void* t, const void* f, void* natural,
                    int32_t param_set);

/* Gather + expand from g slice pointers, exactly what the fused intra-node
 * all-gather produces (Algorithm 1 lines 11, 14-15, 23-24). */
void fo_expand(const fo_geom* g, const uint8_t* mask, const void* const* t_slices,
               const void* const* f_slices, void* natural, int32_t param_set);

/* The same over natural chunks [c_lo, c_hi) only; kt_lo = trainable chunks
 * before c_lo (so a layer can be split across threads: results are identical). */
void fo_expand_part(const fo_geom* g, const uint8_t* mask, const void* const* t_slices,
                    const void* const* f_slices, void* natural, int32_t param_set, int64_t c_lo, int64_t c_hi,
                    int64_t kt_lo);

/* Hierarchical reduce-scatter, intra step, for slice j on node n:
 * sum over the g natural gradient buffers in order 0..g-1 in fp32.  Own shard
 * chunks -> own_out (fp32, times scale iff final_scale); other shards ->
 * wire_out (slice-relative, parameter dtype, RNE). */
void fo_rs_slice(const fo_geom* g, const uint8_t* mask, int32_t elem_bytes, const void* const* grads,
                 int32_t j, int32_t n, float scale, int32_t final_scale, float* own_out, void* wire_out);

void fo_rs_slice_part(const fo_geom* g, const uint8_t* mask, int32_t elem_bytes, const void* const* grads,
                      int32_t j, int32_t n, float scale, int32_t final_scale, float* own_out, void* wire_out,
                      int64_t c_lo, int64_t c_hi, int64_t kt_lo);

/* Inter step epilogue: out[i] = scale * sum_{m=0..N-1} part_m[i]. */
void fo_rs_finalize(int64_t n_elems, int32_t nodes, int32_t node, int32_t elem_bytes, const float* own,
                    const void* wire, int64_t wire_stride, float scale, float* out);

/* AdamW, arithmetic identical to the CUDA kernel (explicit fmaf, RNE). */
void fo_adam(int64_t n, float lr, float beta1, float beta2, float eps, float wd, float bias_c1,
             float bias_c2, float* master, float* m, float* v, const float* grad, void* param,
             int32_t param_elem_bytes);

/* Deterministic natural-layer init (kind 0 uniform(-s,s), 1 constant). */
typedef struct fo_init_range {
  int64_t begin, end;
  int32_t kind;
  float scale;
} fo_init_range;
void fo_init_natural(int64_t n_elems, int32_t elem_bytes, uint64_t seed, int32_t layer,
                     const fo_init_range* ranges, int32_t nr, void* out);

uint16_t fo_f32_to_bf16(float x);
float fo_bf16_to_f32(uint16_t h);

/* Multi-threaded memcpy / fp32 sum used by the CPU data-plane timing. */
void fo_parallel_copy(void* dst, const void* src, size_t bytes, int32_t threads);

#ifdef __cplusplus
}
#endif
#endif
