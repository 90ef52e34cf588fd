"""FCDP training loop on B200: shardsim programs executed by the engine, with
the driving model's compute bound to the engine's compute stream.

This is the public API a user calls (bench.py's e2e path goes through it):

    t = FcdpTrainer(PRESETS["gpt2-1.3b"], topo, StrategyPlan(StrategyKind.Fcdp), rank=..., ...)
    loss = t.step(tokens, labels)      # one iteration: build_iteration -> engine.run

Backward without re-gathering through autograd: each layer's forward graph is
kept, but the saved weight tensors are swapped out at pack time (they alias
the gathered-layer buffer, which is reused) and re-materialised at unpack time
from the buffer the backward pass re-gathered - ZeRO-3/FCDP semantics
(forward gathers, backward reconstructs from the host cache).
"""
from __future__ import annotations

import os
from typing import Dict, List, Optional

import torch

from . import shardsim as S
from .driving_model import LayerDef, ModelConfig, layer_forward
from .engine import FWD, Engine
from .tensors import device_view


class FcdpTrainer:
    def __init__(self, cfg: ModelConfig, topo: S.ClusterTopology, plan: S.StrategyPlan, *, rank: int,
                 world_size: int, device: int, shm_name: str, batch_per_gpu: int, seq_len: Optional[int] = None,
                 seed: int = 0x5EED, nic_pacing: bool = True, lr: float = 1e-4, weight_decay: float = 0.0,
                 gpu_capacity_bytes: int = 0, use_copy_engine: bool = False, timeout_s: float = 600.0,
                 activation_bytes_per_sample: Optional[int] = None):
        self.cfg = cfg
        self.topo, self.plan = topo, plan
        self.rank, self.world = rank, world_size
        self.device = torch.device("cuda", device)
        self.batch, self.seq = batch_per_gpu, seq_len or cfg.seq
        self.dtype = torch.bfloat16 if cfg.dtype_bytes == 2 else torch.float32
        self.defs: List[LayerDef] = cfg.layer_defs()
        # activation bytes per sample per layer feed the tau-admission projection;
        # a measured figure (bench.py's ZeRO-3 max-batch probe) overrides the estimate
        layers = [S.LayerSpec(i, d.numel, d.trainable_params() / d.numel,
                              activation_bytes_per_sample=(activation_bytes_per_sample
                                                           if activation_bytes_per_sample is not None
                                                           else activation_bytes(cfg, d, self.seq)))
                  for i, d in enumerate(self.defs)]
        self.model = S.ModelSpec(layers, cfg.dtype_bytes, batch_per_gpu=batch_per_gpu)
        self.gpu_capacity_bytes = gpu_capacity_bytes
        self.engine = Engine(self.model, topo, plan, rank=rank, world_size=world_size, device=device,
                             shm_name=shm_name, chunk_masks=[d.chunk_mask(cfg.dtype_bytes) for d in self.defs],
                             nic_pacing=nic_pacing, use_copy_engine=use_copy_engine, timeout_s=timeout_s)
        self.engine.init_params(seed, [d.init_ranges() for d in self.defs])
        self.engine.set_adam(lr=lr, weight_decay=weight_decay)
        self.engine.set_compute(self._compute)
        self.stream = torch.cuda.ExternalStream(self.engine.compute_stream(), device=self.device)
        self.states = S.init_param_states(self.model)
        self.iteration = 0
        self._saved: Dict[int, tuple] = {}
        self._bwd_w: Dict[int, torch.Tensor] = {}
        self._cur = None
        self._grad_act = None
        self.loss: Optional[torch.Tensor] = None
        self._held_grads: List[torch.Tensor] = []
        self._segments_ok = os.environ.get("FCDP_GRAD_SEGMENTS", "1") != "0"
        self.last_program: Optional[S.EventProgram] = None

    # -------------------------------------------------------------- API
    def step(self, tokens: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        """One training iteration.  tokens/labels: int64 [batch, seq] on this GPU.
        Returns the loss as a device tensor (enqueued on the compute stream)."""
        self.iteration += 1
        prog = S.build_iteration(self.plan, self.model, self.topo, self.states, self.iteration,
                                 gpu_capacity_bytes=self.gpu_capacity_bytes)
        self.tokens, self.labels = tokens, labels
        self.states = self.engine.run(prog, self.states)
        self._held_grads.clear()  # the program (incl. its fused updates) is enqueued before the join
        self.last_program = prog
        return self.loss

    def sync(self) -> None:
        self.engine.sync()

    def close(self) -> None:
        self.engine.close()

    # ----------------------------------------------------------- compute
    def _pack(self, t: torch.Tensor):
        cur = self._cur
        if cur is not None and t.device.type == "cuda":
            try:
                ptr = t.untyped_storage().data_ptr()
            except Exception:
                return t
            if ptr == cur[1]:
                return ("fcdp-w", cur[0], t.storage_offset(), tuple(t.shape), tuple(t.stride()))
        return t

    def _unpack(self, obj):
        if isinstance(obj, tuple) and len(obj) == 5 and obj[0] == "fcdp-w":
            _, layer, off, shape, stride = obj
            return torch.as_strided(self._bwd_w[layer], shape, stride, off)
        return obj

    def _hand_over(self, layer: int, ldef: LayerDef, train, grads) -> bool:
        """G = 1: give the engine autograd's own gradient buffers (no copy into
        the natural gradient slot; the fused RS + AdamW reads them in place).
        They stay referenced until step() returns (engine.run enqueued the
        program's end, which orders the compute stream after the update)."""
        if not self._segments_ok or not self.engine.takes_grad_segments(layer):
            return False
        segs = []
        for n, gr in zip(train, grads):
            if gr is None:
                continue  # an unused tensor: gradient 0 (chunks no segment covers)
            if not gr.is_contiguous() or gr.dtype != self.dtype or gr.data_ptr() % 16:
                return False
            segs.append((ldef.offsets[n], gr.data_ptr(), gr.numel()))
        segs.sort()
        if len(segs) > 24:
            return False
        self.engine.grad_segments(layer, segs)
        self._held_grads.extend(g for g in grads if g is not None)
        return True

    def _copy_grads(self, g: int, ldef: LayerDef, train, grads, p) -> None:
        """Autograd's gradients into the engine's natural gradient slot: every
        16-byte aligned contiguous tensor in one fcdp_copy_segments launch."""
        import ctypes as C
        from ._capi import check, lib
        G = device_view(g, ldef.numel, self.dtype, self.device)
        eb = G.element_size()
        src, dst, nbytes = [], [], []
        for n, gr in zip(train, grads):
            o = ldef.offsets[n]
            if gr is None:
                G[o:o + p[n].numel()].zero_()
            elif gr.is_contiguous() and gr.dtype == self.dtype and gr.data_ptr() % 16 == 0 and \
                    (o * eb) % 16 == 0 and (gr.numel() * eb) % 16 == 0:
                src.append(gr.data_ptr())
                dst.append(g + o * eb)
                nbytes.append(gr.numel() * eb)
            else:
                G[o:o + gr.numel()].copy_(gr.reshape(-1))
        if src:
            n = len(src)
            check(lib().fcdp_copy_segments(n, (C.c_void_p * n)(*src), (C.c_void_p * n)(*dst),
                                           (C.c_int64 * n)(*nbytes),
                                           C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)))

    def _params(self, flat: torch.Tensor, ldef: LayerDef, grad: bool):
        out = {}
        for t in ldef.tensors:
            v = flat[ldef.offsets[t.name]:ldef.offsets[t.name] + t.numel].view(t.shape)
            out[t.name] = v.detach().requires_grad_(grad and t.trainable)
        return out

    def _compute(self, kind: int, layer: int, w: int, g: Optional[int], stream: int) -> None:
        ldef = self.defs[layer]
        with torch.cuda.stream(self.stream):
            W = device_view(w, ldef.numel, self.dtype, self.device)
            if kind == FWD:
                p = self._params(W, ldef, True)
                x_in = None
                if layer > 0:
                    x_in = self._saved_out.detach().requires_grad_(True)
                self._cur = (layer, w)
                with torch.autograd.graph.saved_tensors_hooks(self._pack, self._unpack):
                    y = layer_forward(self.cfg, ldef, p, x_in, self.tokens, self.labels)
                self._cur = None
                self._saved[layer] = (x_in, y, p)
                if ldef.kind == "head":
                    self.loss = y.detach()
                else:
                    self._saved_out = y
            else:
                x_in, y, p = self._saved.pop(layer)
                self._bwd_w[layer] = W
                train = [t.name for t in ldef.tensors if t.trainable]
                inputs = ([x_in] if x_in is not None else []) + [p[n] for n in train]
                grad_out = None if ldef.kind == "head" else self._grad_act
                if not inputs or not y.requires_grad:
                    # nothing upstream needs a gradient (e.g. a frozen embedding under PEFT)
                    self._bwd_w.pop(layer, None)
                    self._grad_act = None
                    if layer == 0:
                        self._saved_out = None
                    return
                grads = torch.autograd.grad(y, inputs, grad_outputs=grad_out, allow_unused=True)
                self._bwd_w.pop(layer, None)
                if x_in is not None:
                    self._grad_act = grads[0]
                    grads = grads[1:]
                if g:
                    if not self._hand_over(layer, ldef, train, grads):
                        self._copy_grads(g, ldef, train, grads, p)
                if layer == 0:
                    self._grad_act = None
                    self._saved_out = None


def activation_bytes(cfg: ModelConfig, d: LayerDef, seq: int) -> int:
    """Activation bytes per sample of one layer, fed to the tau-admission
    projection (reference schedule.cpp:196-208): a bf16 transformer block with
    flash attention keeps about 34 * seq * hidden bytes, the head its bf16 logits
    and their gradient (the fused cross-entropy keeps no fp32 copy)."""
    ffn = cfg.ffn or 4 * cfg.hidden
    if d.kind == "head":
        return seq * cfg.vocab_rows * (4 if cfg.dtype_bytes == 2 else 8)
    if d.kind == "embed":
        return seq * cfg.hidden * 2
    return int(seq * cfg.hidden * 34 * max(1.0, ffn / (4 * cfg.hidden)))


def synthetic_batch(vocab: int, batch: int, seq: int, seed: int, step: int, rank: int,
                    device=None, pin: bool = False):
    """Counter-based synthetic tokens: (seed, step, rank) -> [batch, seq+1] ids."""
    g = torch.Generator().manual_seed((seed * 1_000_003 + step * 8191 + rank) & 0x7FFFFFFFFFFFFFFF)
    ids = torch.randint(0, vocab, (batch, seq + 1), generator=g, dtype=torch.int64)
    if pin:
        ids = ids.pin_memory()
    if device is not None:
        ids = ids.to(device, non_blocking=True)
    return ids[:, :-1], ids[:, 1:]
