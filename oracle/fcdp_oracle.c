/*
 * CPU restatement of the FCDP data plane - TEST INFRASTRUCTURE ONLY.
 * See fcdp_oracle.h for the provenance of every rule restated here.
 * Compiled with -ffp-contract=off: the only fused multiply-adds are the
 * explicit fmaf() calls, mirrored by __fmaf_rn in the CUDA kernels.
 */
#include "fcdp_oracle.h"

#include <math.h>
#include <string.h>

#include <pthread.h>

enum { kChunk = 16 };

uint16_t fo_f32_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u); /* round to nearest even */
  return (uint16_t)(u >> 16);
}

float fo_bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float x;
  memcpy(&x, &u, 4);
  return x;
}

static float load_elem(const void* p, int64_t i, int32_t eb) {
  if (eb == 2) return fo_bf16_to_f32(((const uint16_t*)p)[i]);
  return ((const float*)p)[i];
}

static void store_elem(void* p, int64_t i, int32_t eb, float x) {
  if (eb == 2)
    ((uint16_t*)p)[i] = fo_f32_to_bf16(x);
  else
    ((float*)p)[i] = x;
}

/* Shard geometry: each portion is padded up to a multiple of G chunks and split
 * G ways; shard r = j*N + n sits on (node n, GPU j), so slice j (N shards) is
 * contiguous - the p^intra of PAPER.md:483. */
void fo_geom_of(int64_t chunks, const uint8_t* mask, int32_t nodes, int32_t local, fo_geom* out) {
  int64_t pt = 0;
  for (int64_t c = 0; c < chunks; ++c) pt += (mask == NULL || mask[c]) ? 1 : 0;
  const int64_t G = (int64_t)nodes * local;
  out->chunks = chunks;
  out->pt = pt;
  out->pf = chunks - pt;
  out->shard_t = (pt + G - 1) / G;
  out->shard_f = (out->pf + G - 1) / G;
  out->slice_t = out->shard_t * nodes;
  out->slice_f = out->shard_f * nodes;
  out->nodes = nodes;
  out->local = local;
}

void fo_partition(int64_t chunks, const uint8_t* mask, const void* natural, void* t, void* f) {
  const uint8_t* in = (const uint8_t*)natural;
  int64_t kt = 0, kf = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    if (mask == NULL || mask[c])
      memcpy((uint8_t*)t + kChunk * kt++, in + kChunk * c, kChunk);
    else
      memcpy((uint8_t*)f + kChunk * kf++, in + kChunk * c, kChunk);
  }
}

void fo_unpartition(int64_t chunks, const uint8_t* mask, const void* t, const void* f, void* natural,
                    int32_t param_set) {
  uint8_t* out = (uint8_t*)natural;
  int64_t kt = 0, kf = 0;
  for (int64_t c = 0; c < chunks; ++c) {
    const int tr = mask == NULL || mask[c];
    if (tr) {
      if (param_set != 2) memcpy(out + kChunk * c, (const uint8_t*)t + kChunk * kt, kChunk);
      ++kt;
    } else {
      if (param_set != 1) memcpy(out + kChunk * c, (const uint8_t*)f + kChunk * kf, kChunk);
      ++kf;
    }
  }
}

void fo_expand_part(const fo_geom* g, const uint8_t* mask, const void* const* t_slices,
                    const void* const* f_slices, void* natural, int32_t param_set, int64_t c_lo, int64_t c_hi,
                    int64_t kt_lo) {
  uint8_t* out = (uint8_t*)natural;
  int64_t kt = kt_lo, kf = c_lo - kt_lo;
  for (int64_t c = c_lo; c < c_hi; ++c) {
    const int tr = mask == NULL || mask[c];
    const int64_t k = tr ? kt++ : kf++;
    if (tr ? param_set == 2 : param_set == 1) continue;
    const int64_t per = tr ? g->slice_t : g->slice_f;
    const int64_t j = k / per;
    const uint8_t* src = (const uint8_t*)(tr ? t_slices[j] : f_slices[j]);
    memcpy(out + kChunk * c, src + kChunk * (k - j * per), kChunk);
  }
}

void fo_expand(const fo_geom* g, const uint8_t* mask, const void* const* t_slices,
               const void* const* f_slices, void* natural, int32_t param_set) {
  fo_expand_part(g, mask, t_slices, f_slices, natural, param_set, 0, g->chunks, 0);
}

void fo_rs_slice_part(const fo_geom* g, const uint8_t* mask, int32_t elem_bytes, const void* const* grads,
                      int32_t j, int32_t n, float scale, int32_t final_scale, float* own_out, void* wire_out,
                      int64_t c_lo, int64_t c_hi, int64_t kt_lo) {
  const int32_t V = kChunk / elem_bytes;
  const int64_t k0 = (int64_t)j * g->slice_t;
  int64_t k1 = k0 + g->slice_t;
  if (k1 > g->pt) k1 = g->pt;
  const int64_t own_lo = (int64_t)n * g->shard_t, own_hi = own_lo + g->shard_t;
  int64_t kt = kt_lo;
  for (int64_t c = c_lo; c < c_hi; ++c) {
    if (!(mask == NULL || mask[c])) continue;
    const int64_t k = kt++;
    if (k < k0 || k >= k1) continue;
    const int64_t rel = k - k0;
    for (int32_t e = 0; e < V; ++e) {
      float acc = 0.0f;
      for (int32_t i = 0; i < g->local; ++i) acc += load_elem(grads[i], c * V + e, elem_bytes);
      if (rel >= own_lo && rel < own_hi)
        own_out[(rel - own_lo) * V + e] = final_scale ? acc * scale : acc;
      else
        store_elem(wire_out, rel * V + e, elem_bytes, acc);
    }
  }
}

void fo_rs_slice(const fo_geom* g, const uint8_t* mask, int32_t elem_bytes, const void* const* grads,
                 int32_t j, int32_t n, float scale, int32_t final_scale, float* own_out, void* wire_out) {
  fo_rs_slice_part(g, mask, elem_bytes, grads, j, n, scale, final_scale, own_out, wire_out, 0, g->chunks, 0);
}

void fo_rs_finalize(int64_t n_elems, int32_t nodes, int32_t node, int32_t elem_bytes, const float* own,
                    const void* wire, int64_t wire_stride, float scale, float* out) {
  for (int64_t i = 0; i < n_elems; ++i) {
    float acc = 0.0f;
    for (int32_t m = 0; m < nodes; ++m)
      acc += m == node ? own[i] : load_elem(wire, (int64_t)m * wire_stride + i, elem_bytes);
    out[i] = acc * scale;
  }
}

void fo_adam(int64_t n, float lr, float beta1, float beta2, float eps, float wd, float bias_c1,
             float bias_c2, float* master, float* m, float* v, const float* grad, void* param,
             int32_t param_elem_bytes) {
  const float omb1 = 1.0f - beta1, omb2 = 1.0f - beta2;
  for (int64_t i = 0; i < n; ++i) {
    const float gr = grad[i];
    float w = master[i];
    const float mi = fmaf(beta1, m[i], omb1 * gr);
    const float vi = fmaf(beta2, v[i], (omb2 * gr) * gr);
    const float mhat = mi / bias_c1;
    const float vhat = vi / bias_c2;
    const float denom = sqrtf(vhat) + eps;
    const float upd = mhat / denom + wd * w;
    w = w - lr * upd;
    m[i] = mi;
    v[i] = vi;
    master[i] = w;
    store_elem(param, i, param_elem_bytes, w);
  }
}

static uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void fo_init_natural(int64_t n_elems, int32_t elem_bytes, uint64_t seed, int32_t layer,
                     const fo_init_range* ranges, int32_t nr, void* out) {
  for (int64_t e = 0; e < n_elems; ++e) {
    float x = 0.0f;
    for (int32_t r = 0; r < nr; ++r) {
      if (e < ranges[r].begin || e >= ranges[r].end) continue;
      if (ranges[r].kind == 1) {
        x = ranges[r].scale;
      } else {
        const uint64_t z = splitmix64(seed ^ ((uint64_t)layer << 40) ^ (uint64_t)e);
        const float u = (float)(z >> 40) * (1.0f / 16777216.0f);
        x = (2.0f * u - 1.0f) * ranges[r].scale;
      }
      break;
    }
    store_elem(out, e, elem_bytes, x);
  }
}

typedef struct copy_job {
  uint8_t* dst;
  const uint8_t* src;
  size_t bytes;
} copy_job;

static void* copy_worker(void* arg) {
  const copy_job* j = (const copy_job*)arg;
  memcpy(j->dst, j->src, j->bytes);
  return NULL;
}

void fo_parallel_copy(void* dst, const void* src, size_t bytes, int32_t threads) {
  enum { kMaxThreads = 64 };
  if (threads < 1) threads = 1;
  if (threads > kMaxThreads) threads = kMaxThreads;
  if (threads == 1 || bytes < ((size_t)1 << 20)) {
    memcpy(dst, src, bytes);
    return;
  }
  pthread_t tid[kMaxThreads];
  copy_job jobs[kMaxThreads];
  const size_t per = (bytes / (size_t)threads + 63) & ~(size_t)63;
  int32_t started = 0;
  for (int32_t t = 0; t < threads; ++t) {
    const size_t off = per * (size_t)t;
    if (off >= bytes) break;
    jobs[t].dst = (uint8_t*)dst + off;
    jobs[t].src = (const uint8_t*)src + off;
    jobs[t].bytes = bytes - off < per ? bytes - off : per;
    if (pthread_create(&tid[t], NULL, copy_worker, &jobs[t]) != 0) {
      copy_worker(&jobs[t]);
      tid[t] = 0;
    }
    started = t + 1;
  }
  for (int32_t t = 0; t < started; ++t)
    if (tid[t]) pthread_join(tid[t], NULL);
}
