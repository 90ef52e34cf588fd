"""CPU reference steps of the FCDP path - TEST / BASELINE INFRASTRUCTURE ONLY.

Used by bench.py's cpu_baseline leg and `--impl reference` arm and by tests/
(never by the product path).  The reference (`shardsim`) has no data plane,
so the CPU "reference implementation of the path" is the C++ CPU executor
(oracle/cpu_executor.cpp): the reference's own compiled control plane builds
every program, and a host-memory data plane (one std::thread per simulated
rank, the oracle's arithmetic) executes all of it - forward all-gathers,
FCDP-Cache stores, backward reloads + intra gathers, the gradient
reduce-scatter with cast/scale, and AdamW - at the workload's full size.

Two ways to fill the compute events:
  * `path_executor` - a synthetic gradient (one elementwise pass over the
    gathered layer).  The driving model's GEMMs are NOT run: the reference has
    no model compute, and a 1-13B model's forward/backward on CPU takes minutes
    per step.  Leaving it out only makes the CPU number faster.
  * `CpuModelCompute` - the driving model's real forward/backward on the host
    cores (torch CPU) for every simulated rank: a full training step, used for
    config C1 (tiny, 2 simulated ranks; FCDP vs ZeRO-3).
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from oracle import cpu_executor as cx


def preset_layers(mc, seq: int):
    from paper_2602_06499_b200.trainer import activation_bytes
    defs = mc.layer_defs()
    eb = mc.dtype_bytes
    return defs, {"params": [d.numel for d in defs], "masks": [d.chunk_mask(eb) for d in defs],
                  "act_bytes": [activation_bytes(mc, d, seq) for d in defs],
                  "init_ranges": [d.init_ranges() for d in defs]}


def path_executor(preset: str, N: int, g: int, strategy: str, tau: float, gpu_capacity_bytes: int, batch: int,
                  seq: int | None = None, threads: int | None = None, seed: int = 0x5EED) -> cx.CpuExecutor:
    from paper_2602_06499_b200.driving_model import PRESETS
    mc = PRESETS[preset]
    _, lay = preset_layers(mc, seq or mc.seq)
    return cx.CpuExecutor(lay["params"], lay["masks"], nodes=N, local=g, strategy=strategy,
                          elem_bytes=mc.dtype_bytes, tau=tau, gpu_capacity_bytes=gpu_capacity_bytes,
                          act_bytes=lay["act_bytes"], batch_per_gpu=batch, seed=seed,
                          threads=threads or len(os.sched_getaffinity(0)), lr=1e-4, weight_decay=0.0,
                          init_ranges=lay["init_ranges"])


def host_bytes_needed(preset: str, N: int, g: int) -> int:
    """Host memory the executor allocates for a preset (all ranks)."""
    from paper_2602_06499_b200.driving_model import PRESETS
    mc = PRESETS[preset]
    defs = mc.layer_defs()
    eb = mc.dtype_bytes
    W = sum(d.numel for d in defs) * eb
    Wt = sum(d.trainable_params() for d in defs) * 4
    big = max(d.numel for d in defs) * eb
    # shards + host cache + slices + retained copies; fp32 master/m/v/grad; per-rank gathered/grad buffers
    return 4 * W + 4 * Wt + N * g * 4 * big


class CpuModelCompute:
    """The executor's compute callback running the driving model on the host
    cores (torch CPU autograd), one activation chain per simulated rank - the
    same per-layer forward / backward split the B200 trainer uses
    (paper_2602_06499_b200/trainer.py)."""

    def __init__(self, mc, batch: int, seq: int, seed: int, world: int, threads: int | None = None):
        import torch
        torch.set_num_threads(threads or len(os.sched_getaffinity(0)))
        self.torch = torch
        self.mc, self.batch, self.seq, self.seed, self.world = mc, batch, seq, seed, world
        self.defs = mc.layer_defs()
        self.dtype = torch.bfloat16 if mc.dtype_bytes == 2 else torch.float32
        self.saved, self.out, self.grad_act = {}, {}, {}
        self.losses = {}
        self.cb = cx.COMPUTE_FN(self._call)

    def set_step(self, step: int):
        from paper_2602_06499_b200.trainer import synthetic_batch
        self.batches = {r: synthetic_batch(self.mc.vocab, self.batch, self.seq, self.seed, step, r)
                        for r in range(self.world)}

    def _call(self, user, kind, rank, layer, w, g):
        try:
            self._compute(kind, rank, layer, w, g)
            return 0
        except Exception:
            import traceback
            traceback.print_exc()
            return 1

    def _compute(self, kind, rank, layer, w, g):
        torch = self.torch
        from paper_2602_06499_b200.driving_model import layer_forward
        d = self.defs[layer]
        eb = self.mc.dtype_bytes
        raw = np.frombuffer(C.string_at(w, d.numel * eb), np.int16 if eb == 2 else np.float32).copy()
        flat = torch.from_numpy(raw).view(self.dtype) if eb == 2 else torch.from_numpy(raw)
        x, y = self.batches[rank]
        if kind == 4:  # forward
            p = {t.name: flat[d.offsets[t.name]:d.offsets[t.name] + t.numel].view(t.shape).requires_grad_(t.trainable)
                 for t in d.tensors}
            x_in = self.out[rank].detach().requires_grad_(True) if layer > 0 else None
            out = layer_forward(self.mc, d, p, x_in, x, y)
            self.saved[(rank, layer)] = (x_in, out, p)
            if d.kind == "head":
                self.losses[rank] = float(out.detach())
            else:
                self.out[rank] = out
            return
        x_in, out, p = self.saved.pop((rank, layer))
        train = [t.name for t in d.tensors if t.trainable]
        inputs = ([x_in] if x_in is not None else []) + [p[n] for n in train]
        if not inputs or not out.requires_grad:
            self.grad_act[rank] = None
            return
        grads = torch.autograd.grad(out, inputs, grad_outputs=None if d.kind == "head" else self.grad_act[rank],
                                    allow_unused=True)
        if x_in is not None:
            self.grad_act[rank] = grads[0]
            grads = grads[1:]
        if g:
            gflat = torch.zeros(d.numel, dtype=self.dtype)
            for n, gr in zip(train, grads):
                if gr is not None:
                    gflat[d.offsets[n]:d.offsets[n] + gr.numel()] = gr.reshape(-1)
            buf = gflat.view(torch.int16).numpy() if eb == 2 else gflat.numpy()
            C.memmove(g, buf.ctypes.data, d.numel * eb)


def full_step_executor(preset: str, N: int, g: int, strategy: str, batch: int, seed: int = 0x5EED,
                       lr: float = 1e-3, wd: float = 0.01, threads: int | None = None):
    """Executor + real driving-model compute (config C1: a full CPU training step)."""
    from paper_2602_06499_b200.driving_model import PRESETS
    mc = PRESETS[preset]
    _, lay = preset_layers(mc, mc.seq)
    ex = cx.CpuExecutor(lay["params"], lay["masks"], nodes=N, local=g, strategy=strategy,
                        elem_bytes=mc.dtype_bytes, act_bytes=lay["act_bytes"], batch_per_gpu=batch, seed=seed,
                        threads=threads or len(os.sched_getaffinity(0)), lr=lr, weight_decay=wd,
                        init_ranges=lay["init_ranges"])
    comp = CpuModelCompute(mc, batch, mc.seq, seed, N * g, threads)
    ex._cb = comp.cb
    cx._check(cx.lib().fce_set_compute(ex._h, comp.cb, None))
    return ex, comp


def c1_tiny_timing(steps: int = 5, warmup: int = 2, batch: int = 2) -> dict:
    """BASELINE config C1: the tiny 2-layer h=256 fp32 model, 2 simulated ranks
    (2 emulated nodes x 1 GPU), one FULL training step (model compute + the
    whole path) on the C++ CPU executor, FCDP vs ZeRO-3."""
    out = {}
    # one discarded pass first: torch's CPU thread pool and allocator warm up
    # once per process, which would otherwise be charged to whichever runs first
    for strategy in ("zero3", "fcdp", "zero3"):
        ex, comp = full_step_executor("tiny", 2, 1, strategy, batch)
        ts, losses, st = [], [], None
        for s in range(1, warmup + steps + 1):
            comp.set_step(s)
            t0 = time.perf_counter()
            st = ex.step()
            if s > warmup:
                ts.append(time.perf_counter() - t0)
            losses.append(float(np.mean(list(comp.losses.values()))))
        ex.close()
        tokens = 2 * batch * comp.seq
        out[strategy] = {"ms_per_step": 1e3 * float(np.median(ts)), "tokens_per_s": tokens / float(np.median(ts)),
                         "loss_last": losses[-1], "nic_bytes_per_node": st["nic_tx_fwd_ag"] + st["nic_tx_bwd_ag"] +
                         st["nic_tx_rs"], "bwd_ag_bytes_per_node": st["nic_tx_bwd_ag"]}
    out["sample"] = (f"tiny h=256 fp32, 2 simulated ranks (2x1), {batch} x {comp.seq} tokens per rank, "
                     f"{steps} timed full steps (torch-CPU model compute + C++ executor data plane)")
    return out
