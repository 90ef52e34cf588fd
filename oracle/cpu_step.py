"""CPU reference step of the FCDP path - TEST / BASELINE INFRASTRUCTURE ONLY.

Used by bench.py's cpu_baseline leg and `--impl reference` arm (and nowhere in
the product path).  The reference (`shardsim`) has no data plane, so the CPU
"reference implementation of the path" is the oracle restatement
(oracle/fcdp_oracle.c) executing the same per-layer FCDP data movement -
forward gather, FCDP-Cache store, backward reload + gather, gradient
reduce-scatter with cast/scale, AdamW - plus the driving model's forward and
backward on the host cores (torch CPU, same dtype as the GPU run).

A full 1-13B training step on CPU takes minutes, so the measured unit is a
bounded SAMPLE: one transformer block, one sequence, at the 1x1 geometry;
the step time is extrapolated as  L * (t_dataplane + batch * t_compute).
Embedding and LM-head layers are not in the sample (stated in the output).
"""
from __future__ import annotations

import os
import time

import numpy as np

from oracle import oracle as O


def cpu_step_sample(preset: str = "gpt2-1.3b", batch: int = 8, seq: int | None = None, threads: int | None = None,
                    repeats: int = 2, seed: int = 0x5EED) -> dict:
    import torch
    from paper_2602_06499_b200.driving_model import PRESETS, layer_forward

    threads = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    mc = PRESETS[preset]
    seq = seq or mc.seq
    defs = mc.layer_defs()
    block = defs[1]
    eb = mc.dtype_bytes
    V = 16 // eb
    chunks = block.numel // V
    mask = block.chunk_mask(eb)
    geo = O.geom(chunks, mask, 1, 1)
    nat = O.init_natural(block.numel, eb, seed, 1, block.init_ranges())
    t, f = O.partition(nat.view(np.uint8), mask)
    W = np.zeros(block.numel * eb, np.uint8)
    cache_t = np.zeros_like(t)
    cache_f = np.zeros_like(f)
    dtype = torch.bfloat16 if eb == 2 else torch.float32
    pt_elems = geo.pt * V
    master = (O.bf16_to_f32(t.view(np.uint16)) if eb == 2 else t.view(np.float32)).copy()
    m = np.zeros_like(master)
    v = np.zeros_like(master)
    param = t.view(np.uint16 if eb == 2 else np.float32).copy()
    g = torch.Generator().manual_seed(seed)
    x_in = (torch.randn(1, seq, mc.hidden, generator=g) * 0.1).to(dtype)

    def one():
        times = {}
        t0 = time.perf_counter()
        O.expand(geo, mask, [t], [f], W, 0)                 # forward AgInter (shard == slice at 1x1)
        O.parallel_copy(cache_t, t, threads)                # FCDP-Cache store
        if f.size:
            O.parallel_copy(cache_f, f, threads)
        O.parallel_copy(t, cache_t, threads)                # backward reload
        O.expand(geo, mask, [cache_t], [cache_f], W, 0)     # backward AgIntra
        times["gather_cache"] = time.perf_counter() - t0
        # driving-model compute for one sequence
        flat = torch.from_numpy(W.view(np.int16 if eb == 2 else np.float32).copy())
        flat = flat.view(dtype) if eb == 2 else flat
        p = {}
        for ts in block.tensors:
            p[ts.name] = flat[block.offsets[ts.name]:block.offsets[ts.name] + ts.numel].view(ts.shape).detach() \
                .requires_grad_(ts.trainable)
        x = x_in.clone().requires_grad_(True)
        t1 = time.perf_counter()
        y = layer_forward(mc, block, p, x)
        y.float().sum().backward()
        times["compute_per_seq"] = time.perf_counter() - t1
        grad_nat = np.zeros(block.numel, np.uint16 if eb == 2 else np.float32)
        gflat = torch.from_numpy(grad_nat.view(np.int16) if eb == 2 else grad_nat)
        for ts in block.tensors:
            if ts.trainable and p[ts.name].grad is not None:
                src = p[ts.name].grad.reshape(-1)
                gflat[block.offsets[ts.name]:block.offsets[ts.name] + ts.numel] = \
                    src.view(torch.int16) if eb == 2 else src
        t2 = time.perf_counter()
        own, _ = O.rs_slice(geo, mask, eb, [grad_nat], 0, 0, 1.0, True)   # RS + cast/scale (G = 1)
        O.adam(master, m, v, own[:pt_elems].copy(), param, 1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
        times["rs_adam"] = time.perf_counter() - t2
        return times

    one()  # warm-up
    samples = [one() for _ in range(repeats)]
    med = {k: float(np.median([s[k] for s in samples])) for k in samples[0]}
    t_dp = med["gather_cache"] + med["rs_adam"]
    t_layer = t_dp + batch * med["compute_per_seq"]
    L = mc.layers
    step_s = L * t_layer
    tokens = batch * seq
    return {"tokens_per_s_per_gpu": tokens / step_s, "step_s": step_s, "t_dataplane_layer_s": t_dp,
            "t_compute_seq_layer_s": med["compute_per_seq"], "threads": threads,
            "sample": f"1 of {L} {block.kind} layers x 1 of {batch} sequences (seq {seq}), {repeats} repeats; "
                      f"step = L*(dataplane + batch*compute); embedding/head excluded"}
