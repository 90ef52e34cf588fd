"""Driving models for the FCDP data plane (the compute behind ComputeFwd/Bwd).

The reference models a layer only by its size (workload.hpp:13-33); to train
something real the B200 build needs the layers themselves.  Each layer is ONE
flat natural-order buffer (the unit the shard store gathers) carved into
named tensors, so a ModelSpec layer list and the PEFT chunk mask fall out of
the tensor list:

    GPT-2 (LayerNorm, GELU, biased MHA)        - configs C1 (tiny) and C2 (1.3B)
    Llama (RMSNorm, SwiGLU, RoPE) + LoRA q,k,v,o - configs C3 (7B r=16) and C4 (13B)

Explicit layer lists: [embedding] + blocks + [final norm + untied head].  The
compute uses torch (cuBLAS GEMMs on tensor cores, SDPA attention) on the
engine's compute stream: it is the consumer of the hot path, not the hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

CHUNK = 16


@dataclass
class TensorSpec:
    name: str
    shape: Tuple[int, ...]
    init: str = "uniform"   # uniform(-scale, scale) | const
    scale: float = 0.02
    trainable: bool = True

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape))


@dataclass
class LayerDef:
    kind: str                       # "embed" | "gpt2_block" | "llama_block" | "head"
    tensors: List[TensorSpec]
    offsets: Dict[str, int] = field(default_factory=dict)

    def __post_init__(self):
        off = 0
        for t in self.tensors:
            self.offsets[t.name] = off
            off += t.numel
        self.numel = off

    def chunk_mask(self, elem_bytes: int) -> np.ndarray:
        V = CHUNK // elem_bytes
        if self.numel % V:
            raise ValueError(f"{self.kind}: {self.numel} params is not a whole number of 16-byte chunks")
        m = np.zeros(self.numel // V, np.uint8)
        for t in self.tensors:
            if t.trainable:
                o = self.offsets[t.name]
                if o % V or t.numel % V:
                    raise ValueError(f"trainable tensor {t.name} is not 16-byte aligned")
                m[o // V:(o + t.numel) // V] = 1
        return m

    def trainable_params(self) -> int:
        return sum(t.numel for t in self.tensors if t.trainable)

    def init_ranges(self):
        rs = []
        for t in self.tensors:
            o = self.offsets[t.name]
            rs.append((o, o + t.numel, 1 if t.init == "const" else 0, float(t.scale)))
        return rs


@dataclass
class ModelConfig:
    family: str          # "gpt2" | "llama"
    hidden: int
    layers: int
    heads: int
    vocab: int
    seq: int
    ffn: int = 0
    lora_rank: int = 0   # > 0: LoRA on q,k,v,o; base weights frozen
    dtype_bytes: int = 2
    name: str = ""
    pad_vocab_to: int = 1  # embedding/head rows rounded up (GPT-2: 50257 -> 50304) for aligned GEMMs

    @property
    def vocab_rows(self) -> int:
        m = self.pad_vocab_to
        return (self.vocab + m - 1) // m * m

    def layer_defs(self) -> List[LayerDef]:
        h, V = self.hidden, self.vocab_rows
        peft = self.lora_rank > 0
        defs = []
        if self.family == "gpt2":
            defs.append(LayerDef("embed", [TensorSpec("wte", (V, h), scale=0.02, trainable=not peft),
                                           TensorSpec("wpe", (self.seq, h), scale=0.01, trainable=not peft)]))
            s = 0.02
            for _ in range(self.layers):
                defs.append(LayerDef("gpt2_block", [
                    TensorSpec("ln1_w", (h,), "const", 1.0), TensorSpec("ln1_b", (h,), "const", 0.0),
                    TensorSpec("qkv_w", (3 * h, h), scale=s), TensorSpec("qkv_b", (3 * h,), "const", 0.0),
                    TensorSpec("proj_w", (h, h), scale=s / math.sqrt(2 * self.layers)),
                    TensorSpec("proj_b", (h,), "const", 0.0),
                    TensorSpec("ln2_w", (h,), "const", 1.0), TensorSpec("ln2_b", (h,), "const", 0.0),
                    TensorSpec("fc_w", (4 * h, h), scale=s), TensorSpec("fc_b", (4 * h,), "const", 0.0),
                    TensorSpec("fc2_w", (h, 4 * h), scale=s / math.sqrt(2 * self.layers)),
                    TensorSpec("fc2_b", (h,), "const", 0.0)]))
            defs.append(LayerDef("head", [TensorSpec("lnf_w", (h,), "const", 1.0),
                                          TensorSpec("lnf_b", (h,), "const", 0.0),
                                          TensorSpec("lm_w", (V, h), scale=0.02)]))
        elif self.family == "llama":
            f, r = self.ffn, self.lora_rank
            defs.append(LayerDef("embed", [TensorSpec("wte", (V, h), scale=0.02, trainable=not peft)]))
            for _ in range(self.layers):
                ts = [TensorSpec("attn_norm", (h,), "const", 1.0, trainable=not peft)]
                # q, k, v (and their LoRA A's) adjacent in the layer buffer: one
                # [tokens x 3h] projection GEMM and one [tokens x 3r] LoRA-A GEMM
                for p in ("q", "k", "v", "o"):
                    ts.append(TensorSpec(f"{p}_w", (h, h), scale=0.02, trainable=not peft))
                if peft:
                    for p in ("q", "k", "v", "o"):
                        ts.append(TensorSpec(f"{p}_A", (r, h), scale=0.02, trainable=True))
                    for p in ("q", "k", "v", "o"):
                        # B != 0 so that A receives gradient from step 1 (parity runs)
                        ts.append(TensorSpec(f"{p}_B", (h, r), scale=1e-3, trainable=True))
                ts += [TensorSpec("mlp_norm", (h,), "const", 1.0, trainable=not peft),
                       TensorSpec("gate_w", (f, h), scale=0.02, trainable=not peft),
                       TensorSpec("up_w", (f, h), scale=0.02, trainable=not peft),
                       TensorSpec("down_w", (h, f), scale=0.02, trainable=not peft)]
                defs.append(LayerDef("llama_block", ts))
            defs.append(LayerDef("head", [TensorSpec("norm_w", (h,), "const", 1.0, trainable=not peft),
                                          TensorSpec("lm_w", (V, h), scale=0.02, trainable=not peft)]))
        else:
            raise ValueError(f"unknown family {self.family}")
        return defs


PRESETS: Dict[str, ModelConfig] = {
    # C1: tiny 2-layer transformer, hidden 256, fp32 (12h^2 + 13h = 789,760 params per block)
    "tiny": ModelConfig("gpt2", 256, 2, 4, 1024, 64, dtype_bytes=4, name="tiny-h256-fp32"),
    # C2: GPT-2 1.3B (h=2048, 24 layers, 16 heads, 50,358,272 params per block)
    "gpt2-1.3b": ModelConfig("gpt2", 2048, 24, 16, 50257, 1024, name="gpt2-1.3b", pad_vocab_to=64),
    # C3: Llama-style 7B + LoRA r=16 on q,k,v,o (202,907,648 params per block, 524,288 trainable)
    "llama7b-lora16": ModelConfig("llama", 4096, 32, 32, 32000, 2048, ffn=11008, lora_rank=16,
                                  name="llama7b-lora16"),
    # C4: Llama-style 13B, full training (317,204,480 params per block)
    "llama13b": ModelConfig("llama", 5120, 40, 40, 32000, 2048, ffn=13824, name="llama13b"),
    # small variants for tests / smoke
    "gpt2-small-test": ModelConfig("gpt2", 128, 3, 4, 512, 32, name="gpt2-small-test"),
    "llama-lora-test": ModelConfig("llama", 128, 3, 4, 512, 32, ffn=352, lora_rank=8, name="llama-lora-test"),
}


# ---------------------------------------------------------------- compute

def _views(flat, ldef: LayerDef):
    return {t.name: flat[ldef.offsets[t.name]:ldef.offsets[t.name] + t.numel].view(t.shape)
            for t in ldef.tensors}


def _rope(x, base=10000.0):
    """Rotary embedding of x [b, s, nh, d] (rotated pairs (0,1), (2,3), ...)."""
    import torch
    b, s, nh, d = x.shape
    pos = torch.arange(s, device=x.device, dtype=torch.float32)
    inv = base ** (-torch.arange(0, d, 2, device=x.device, dtype=torch.float32) / d)
    ang = (pos[:, None] * inv[None, :])[:, None, :]  # [s, 1, d/2]: broadcast over heads
    cos, sin = ang.cos().to(x.dtype), ang.sin().to(x.dtype)
    x1, x2 = x[..., 0::2], x[..., 1::2]
    out = torch.stack((x1 * cos - x2 * sin, x1 * sin + x2 * cos), dim=-1)
    return out.flatten(-2)


_LN = None


def _layer_norm(x, w, b, eps=1e-5):
    """LayerNorm of the GPT-2 blocks: libfcdp's bandwidth kernels for bf16 rows
    (h a multiple of 256, <= 2048, on the GPU), torch's otherwise."""
    global _LN
    import torch
    import torch.nn.functional as F
    h = x.shape[-1]
    if not (x.is_cuda and x.dtype == torch.bfloat16 and h % 256 == 0 and h <= 2048):
        return F.layer_norm(x, (h,), w, b, eps)
    if _LN is None:
        _LN = _make_layernorm()
    return _LN.apply(x, w, b, eps)


_ALN = None


def _add_layer_norm(x, r, w, b, eps=1e-5):
    """(s, LN(s)) with s = x + r: the residual add fused into libfcdp's LayerNorm
    (forward) and the residual's gradient folded into its dx (backward)."""
    global _ALN
    import torch
    import torch.nn.functional as F
    h = x.shape[-1]
    if not (x.is_cuda and x.dtype == torch.bfloat16 and r.dtype == torch.bfloat16 and h % 256 == 0 and h <= 2048):
        s = x + r
        return s, F.layer_norm(s, (h,), w, b, eps)
    if _ALN is None:
        _ALN = _make_add_layernorm()
    return _ALN.apply(x, r, w, b, eps)


def _make_add_layernorm():
    import ctypes as C
    import torch
    from ._capi import check, lib

    P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None

    class AddLayerNormFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, r, w, b, eps):
            xc, rc = x.contiguous(), r.contiguous()
            h = xc.shape[-1]
            rows = xc.numel() // h
            s_ = torch.empty_like(xc)
            y = torch.empty_like(xc)
            mean = torch.empty(rows, dtype=torch.float32, device=x.device)
            rstd = torch.empty_like(mean)
            st = C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
            check(lib().fcdp_add_layernorm_fwd(rows, h, eps, P(xc), P(rc), P(w), P(b), P(s_), P(y), P(mean), P(rstd),
                                               st))
            ctx.save_for_backward(s_, w, mean, rstd)
            return s_, y

        @staticmethod
        def backward(ctx, ds, dy):
            s_, w, mean, rstd = ctx.saved_tensors
            h = s_.shape[-1]
            rows = s_.numel() // h
            dyc = dy.contiguous() if dy is not None else torch.zeros_like(s_)
            dsc = ds.contiguous() if ds is not None else None
            dx = torch.empty_like(s_)
            want_w = ctx.needs_input_grad[2] or ctx.needs_input_grad[3]
            dw = torch.empty(h, dtype=w.dtype, device=w.device) if want_w else None
            db = torch.empty(h, dtype=w.dtype, device=w.device) if want_w else None
            splits = 64
            scratch = torch.empty(2 * splits * h, dtype=torch.float32, device=s_.device) if want_w else None
            st = C.c_void_p(torch.cuda.current_stream(s_.device).cuda_stream)
            check(lib().fcdp_layernorm_bwd_res(rows, h, P(dyc), P(s_), P(w), P(mean), P(rstd), P(dsc), P(dx), P(dw),
                                               P(db), P(scratch), splits, st))
            return dx, dx, dw, db, None

    return AddLayerNormFn


_RMS = None


def _rms_norm(x, w, r=None, eps=1e-5):
    """RMSNorm of x (or of the residual sum s = x + r, returned as (s, y)) on
    libfcdp's kernels for bf16 rows with h a multiple of 1024; torch otherwise."""
    global _RMS
    import torch
    import torch.nn.functional as F
    h = x.shape[-1]
    if not (x.is_cuda and x.dtype == torch.bfloat16 and h % 1024 == 0 and h <= 8192
            and (r is None or r.dtype == torch.bfloat16)):
        if r is None:
            return F.rms_norm(x, (h,), w, eps=eps)
        s_ = x + r
        return s_, F.rms_norm(s_, (h,), w, eps=eps)
    if _RMS is None:
        _RMS = _make_rmsnorm()
    if r is None:
        return _RMS[0].apply(x, w, eps)
    return _RMS[1].apply(x, r, w, eps)


def _make_rmsnorm():
    import ctypes as C
    import torch
    from ._capi import check, lib

    P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    S = lambda dev: C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def fwd(x, r, w, eps):
        xc = x.contiguous()
        h = xc.shape[-1]
        rows = xc.numel() // h
        y = torch.empty_like(xc)
        s_ = torch.empty_like(xc) if r is not None else None
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        rc = r.contiguous() if r is not None else None
        check(lib().fcdp_rmsnorm_fwd(rows, h, eps, P(xc), P(rc), P(w), P(s_), P(y), P(rstd), S(x.device)))
        return (s_ if r is not None else xc), y, rstd

    def bwd(ctx, dy, dres, want_w):
        xin, w, rstd = ctx.saved_tensors
        h = xin.shape[-1]
        rows = xin.numel() // h
        dyc = dy.contiguous() if dy is not None else torch.zeros_like(xin)
        drc = dres.contiguous() if dres is not None else None
        dx = torch.empty_like(xin)
        splits = 64
        dw = torch.empty(h, dtype=w.dtype, device=w.device) if want_w else None
        scratch = torch.empty(splits * h, dtype=torch.float32, device=xin.device) if want_w else None
        check(lib().fcdp_rmsnorm_bwd(rows, h, P(dyc), P(xin), P(w), P(rstd), P(drc), P(dx), P(dw), P(scratch), splits,
                                     S(xin.device)))
        return dx, dw

    class RMSNormFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w, eps):
            xin, y, rstd = fwd(x, None, w, eps)
            ctx.save_for_backward(xin, w, rstd)
            return y

        @staticmethod
        def backward(ctx, dy):
            dx, dw = bwd(ctx, dy, None, ctx.needs_input_grad[1])
            return dx, dw, None

    class AddRMSNormFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, r, w, eps):
            s_, y, rstd = fwd(x, r, w, eps)
            ctx.save_for_backward(s_, w, rstd)
            return s_, y

        @staticmethod
        def backward(ctx, ds, dy):
            dx, dw = bwd(ctx, dy, ds, ctx.needs_input_grad[2])
            return dx, dx, dw, None

    return RMSNormFn, AddRMSNormFn


def _make_layernorm():
    import ctypes as C
    import torch
    from ._capi import check, lib

    P = lambda t: C.c_void_p(t.data_ptr())

    class LayerNormFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x, w, b, eps):
            xc = x.contiguous()
            h = xc.shape[-1]
            rows = xc.numel() // h
            y = torch.empty_like(xc)
            mean = torch.empty(rows, dtype=torch.float32, device=x.device)
            rstd = torch.empty_like(mean)
            s = C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
            check(lib().fcdp_layernorm_fwd(rows, h, eps, P(xc), P(w), P(b), P(y), P(mean), P(rstd), s))
            ctx.save_for_backward(xc, w, mean, rstd)
            return y

        @staticmethod
        def backward(ctx, dy):
            xc, w, mean, rstd = ctx.saved_tensors
            h = xc.shape[-1]
            rows = xc.numel() // h
            dyc = dy.contiguous()
            dx = torch.empty_like(xc)
            want_w = ctx.needs_input_grad[1] or ctx.needs_input_grad[2]
            dw = torch.empty(h, dtype=w.dtype, device=w.device) if want_w else None
            db = torch.empty(h, dtype=w.dtype, device=w.device) if want_w else None
            splits = 64
            scratch = torch.empty(2 * splits * h, dtype=torch.float32, device=xc.device) if want_w else None
            s = C.c_void_p(torch.cuda.current_stream(xc.device).cuda_stream)
            check(lib().fcdp_layernorm_bwd(rows, h, P(dyc), P(xc), P(w), P(mean), P(rstd), P(dx),
                                           P(dw) if want_w else None, P(db) if want_w else None,
                                           P(scratch) if want_w else None, splits, s))
            return dx, dw, db, None

    return LayerNormFn


_FNS = None


def _fused_ok(*ts) -> bool:
    import torch
    return all(t.is_cuda and t.dtype == torch.bfloat16 for t in ts)


def _fns():
    """autograd Functions over libfcdp's driving-model kernels (model_kernels.cu)."""
    global _FNS
    if _FNS is not None:
        return _FNS
    import ctypes as C
    import torch
    from ._capi import check, lib

    P = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    S = lambda dev: C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)

    def bias_grad(dy2):
        rows, cols = dy2.shape
        splits = lib().fcdp_colsum_splits(rows, cols)
        part = torch.empty(splits * cols, dtype=torch.float32, device=dy2.device)
        db = torch.empty(cols, dtype=dy2.dtype, device=dy2.device)
        check(lib().fcdp_bias_grad(rows, cols, P(dy2), P(db), P(part), splits, S(dy2.device)))
        return db

    class LinearBias(torch.autograd.Function):
        """y = x W^T + b (cuBLAS, bias in the GEMM epilogue); backward: the two
        cuBLAS GEMMs torch's addmm backward issues, and db by fcdp_bias_grad
        (torch's column reduction ran at ~2 TB/s)."""

        @staticmethod
        def forward(ctx, x, w, b):
            ctx.save_for_backward(x, w)
            return torch.nn.functional.linear(x, w, b)

        @staticmethod
        def backward(ctx, dy):
            x, w = ctx.saved_tensors
            dy2 = dy.reshape(-1, dy.shape[-1])
            if not dy2.is_contiguous():
                dy2 = dy2.contiguous()
            dx = dw = db = None
            if ctx.needs_input_grad[0]:
                dx = dy2.mm(w).view(x.shape)
            if ctx.needs_input_grad[1]:
                dw = dy2.t().mm(x.reshape(-1, x.shape[-1]))
            if ctx.needs_input_grad[2]:
                db = bias_grad(dy2)
            return dx, dw, db

    class BiasGelu(torch.autograd.Function):
        """y = gelu_tanh(h + b) in one pass; backward dh and db = sum_r dh in one pass."""

        @staticmethod
        def forward(ctx, h, b):
            hc = h.contiguous()
            cols = hc.shape[-1]
            rows = hc.numel() // cols
            y = torch.empty_like(hc)
            check(lib().fcdp_bias_gelu_fwd(rows, cols, P(hc), P(b), P(y), S(hc.device)))
            ctx.save_for_backward(hc, b)
            return y

        @staticmethod
        def backward(ctx, dy):
            hc, b = ctx.saved_tensors
            cols = hc.shape[-1]
            rows = hc.numel() // cols
            dyc = dy.contiguous()
            dh = torch.empty_like(hc)
            splits = lib().fcdp_colsum_splits(rows, cols)
            part = torch.empty(splits * cols, dtype=torch.float32, device=hc.device)
            db = torch.empty(cols, dtype=b.dtype, device=b.device)
            check(lib().fcdp_bias_gelu_bwd(rows, cols, P(dyc), P(hc), P(b), P(dh), P(db), P(part), splits,
                                           S(hc.device)))
            return dh, (db if ctx.needs_input_grad[1] else None)

    class CrossEntropy(torch.autograd.Function):
        """Mean cross-entropy of bf16 logits in fp32 without an fp32 copy of the
        logits: one read forward, one read + one write backward."""

        @staticmethod
        def forward(ctx, logits, labels):
            lc = logits.contiguous()
            V = lc.shape[-1]
            rows = lc.numel() // V
            lab = labels.reshape(-1).to(torch.int64).contiguous()  # the kernel reads int64 labels
            loss = torch.empty(rows, dtype=torch.float32, device=lc.device)
            lse = torch.empty_like(loss)
            check(lib().fcdp_xent_fwd(rows, V, P(lc), P(lab), P(loss), P(lse), S(lc.device)))
            valid = (lab >= 0).sum().clamp_min(1).to(torch.float32)
            ctx.save_for_backward(lc, lab, lse, valid)
            return loss.sum() / valid

        @staticmethod
        def backward(ctx, g):
            lc, lab, lse, valid = ctx.saved_tensors
            V = lc.shape[-1]
            rows = lc.numel() // V
            scale = (g.float() / valid).reshape(1).contiguous()
            dl = torch.empty_like(lc)
            check(lib().fcdp_xent_bwd(rows, V, P(lc), P(lab), P(lse), P(scale), P(dl), S(lc.device)))
            return dl, None

    tables = {}

    def rope_tables(seq, dim, device, base=10000.0):
        key = (seq, dim, device, base)
        if key not in tables:
            pos = torch.arange(seq, device=device, dtype=torch.float32)
            inv = base ** (-torch.arange(0, dim, 2, device=device, dtype=torch.float32) / dim)
            ang = pos[:, None] * inv[None, :]
            tables[key] = (ang.cos().contiguous(), ang.sin().contiguous())
        return tables[key]

    class Rope(torch.autograd.Function):
        """Rotary embedding of [b, s, nh, d] in one pass (fp32 tables); the
        backward is the inverse rotation."""

        @staticmethod
        def forward(ctx, x):
            xc = x.contiguous()
            b, sq, nh, d = xc.shape
            cs, sn = rope_tables(sq, d, xc.device)
            y = torch.empty_like(xc)
            check(lib().fcdp_rope(b, sq, nh, d, P(xc), 0, P(cs), P(sn), 0, P(y), 0, S(xc.device)))
            ctx.shape = (b, sq, nh, d)
            return y

        @staticmethod
        def backward(ctx, dy):
            b, sq, nh, d = ctx.shape
            dyc = dy.contiguous()
            cs, sn = rope_tables(sq, d, dyc.device)
            dx = torch.empty_like(dyc)
            check(lib().fcdp_rope(b, sq, nh, d, P(dyc), 0, P(cs), P(sn), 1, P(dx), 0, S(dyc.device)))
            return dx

    class GateUpSwiGLU(torch.autograd.Function):
        """silu(m Wg^T) * (m Wu^T) with Wg, Wu adjacent in the layer buffer: ONE
        [rows x 2f] GEMM, one fused SwiGLU pass; backward one fused pass giving
        d[gate|up], then one GEMM each for dm and (if trainable) d[Wg|Wu]."""

        @staticmethod
        def forward(ctx, m, wg, wu):
            f, hdim = wg.shape
            w2 = torch.as_strided(wg, (2 * f, hdim), (hdim, 1))
            m2 = m.reshape(-1, hdim)
            h2 = m2.mm(w2.t())
            rows = h2.shape[0]
            y = torch.empty(rows, f, dtype=m.dtype, device=m.device)
            check(lib().fcdp_swiglu_fwd(rows, f, P(h2), 2 * f, C.c_void_p(h2.data_ptr() + f * h2.element_size()), 2 * f,
                                        P(y), S(m.device)))
            ctx.save_for_backward(m, wg, wu, h2)
            return y.view(*m.shape[:-1], f)

        @staticmethod
        def backward(ctx, dy):
            m, wg, wu, h2 = ctx.saved_tensors
            f, hdim = wg.shape
            rows = h2.shape[0]
            dyc = dy.reshape(rows, f).contiguous()
            dh2 = torch.empty_like(h2)
            off = f * h2.element_size()
            check(lib().fcdp_swiglu_bwd(rows, f, P(dyc), P(h2), 2 * f, C.c_void_p(h2.data_ptr() + off), 2 * f,
                                        P(dh2), 2 * f, C.c_void_p(dh2.data_ptr() + off), 2 * f, S(m.device)))
            w2 = torch.as_strided(wg, (2 * f, hdim), (hdim, 1))
            dm = dwg = dwu = None
            if ctx.needs_input_grad[0]:
                dm = dh2.mm(w2).view(m.shape)
            if ctx.needs_input_grad[1] or ctx.needs_input_grad[2]:
                dw2 = dh2.t().mm(m.reshape(-1, hdim))
                dwg, dwu = dw2[:f], dw2[f:]
            return dm, dwg, dwu

    class LlamaQKV(torch.autograd.Function):
        """q, k, v of a Llama block from ONE [tokens x 3h] GEMM over the adjacent
        q|k|v weights (+ LoRA: one [tokens x 3r] GEMM over the adjacent A's and
        the three B's accumulated into their thirds in the GEMM epilogue), RoPE
        applied to the q and k thirds in place of a copy.  Backward by hand:
        one dgrad GEMM for the input (+ one for the LoRA path) instead of three
        (+ three) and the autograd accumulations between them."""

        @staticmethod
        def forward(ctx, a, wq, wk, wv, aq, ak, av, bq, bk, bv, nh):
            b, sq, h = a.shape
            hd = h // nh
            a2 = a.reshape(-1, h)
            w3 = torch.as_strided(wq, (3 * h, h), (h, 1))
            y3 = a2.mm(w3.t())
            xa3 = None
            if aq is not None:
                r = aq.shape[0]
                xa3 = a2.mm(torch.as_strided(aq, (3 * r, h), (h, 1)).t())
                for i, bb in enumerate((bq, bk, bv)):
                    y3[:, i * h:(i + 1) * h].addmm_(xa3[:, i * r:(i + 1) * r], bb.t())
            cs, sn = rope_tables(sq, hd, a.device)
            q = torch.empty(b, sq, nh, hd, dtype=a.dtype, device=a.device)
            k = torch.empty_like(q)
            st = S(a.device)
            rows_of = lambda t: t.numel() // t.shape[-1]
            check(lib().fcdp_rope(b, sq, nh, hd, P(y3), 3 * h, P(cs), P(sn), 0, P(q), 0, st))
            check(lib().fcdp_rope(b, sq, nh, hd, C.c_void_p(y3.data_ptr() + h * y3.element_size()), 3 * h, P(cs),
                                  P(sn), 0, P(k), 0, st))
            v = torch.empty(b, sq, nh, hd, dtype=a.dtype, device=a.device)  # dense v: SDPA keeps its cuDNN path
            eb = y3.element_size()
            check(lib().fcdp_copy_rows(rows_of(a), h * eb, C.c_void_p(y3.data_ptr() + 2 * h * eb), 3 * h * eb, P(v),
                                       h * eb, st))
            ctx.save_for_backward(a, wq, aq, bq, bk, bv, xa3)
            ctx.nh = nh
            return q, k, v

        @staticmethod
        def backward(ctx, dq, dk, dv):
            a, wq, aq, bq, bk, bv, xa3 = ctx.saved_tensors
            b, sq, h = a.shape
            nh = ctx.nh
            hd = h // nh
            rows = b * sq
            a2 = a.reshape(-1, h)
            dy3 = torch.empty(rows, 3 * h, dtype=a.dtype, device=a.device)
            cs, sn = rope_tables(sq, hd, a.device)
            st = S(a.device)
            for i, d in enumerate((dq, dk)):
                dc = d.contiguous()
                check(lib().fcdp_rope(b, sq, nh, hd, P(dc), 0, P(cs), P(sn), 1,
                                      C.c_void_p(dy3.data_ptr() + i * h * dy3.element_size()), 3 * h, st))
            dvc = dv.contiguous()
            eb = dy3.element_size()
            check(lib().fcdp_copy_rows(rows, h * eb, P(dvc), h * eb, C.c_void_p(dy3.data_ptr() + 2 * h * eb), 3 * h * eb,
                                       st))
            w3 = torch.as_strided(wq, (3 * h, h), (h, 1))
            ng = ctx.needs_input_grad
            da = dy3.mm(w3) if ng[0] else None
            dw = [None, None, None]
            if ng[1] or ng[2] or ng[3]:
                dw3 = dy3.t().mm(a2)
                dw = [dw3[i * h:(i + 1) * h] for i in range(3)]
            dA = [None, None, None]
            dB = [None, None, None]
            if aq is not None:
                r = aq.shape[0]
                dxa3 = torch.cat([dy3[:, i * h:(i + 1) * h].mm(bb) for i, bb in enumerate((bq, bk, bv))], dim=1)
                if da is not None:
                    da.addmm_(dxa3, torch.as_strided(aq, (3 * r, h), (h, 1)))
                if ng[4] or ng[5] or ng[6]:
                    dA3 = dxa3.t().mm(a2)
                    dA = [dA3[i * r:(i + 1) * r] for i in range(3)]
                if ng[7] or ng[8] or ng[9]:
                    dB = [dy3[:, i * h:(i + 1) * h].t().mm(xa3[:, i * r:(i + 1) * r]) for i in range(3)]
            return (da.view(a.shape) if da is not None else None, *dw, *dA, *dB, None)

    class LoraLinear(torch.autograd.Function):
        """y = x W^T + (x A^T) B^T (the add in the second GEMM's epilogue);
        backward dx = dy W + (dy B) A with the second term accumulated in the
        GEMM epilogue too (no autograd accumulation pass)."""

        @staticmethod
        def forward(ctx, x, w, a_, b_):
            x2 = x.reshape(-1, x.shape[-1])
            xa = x2.mm(a_.t())
            y = torch.addmm(x2.mm(w.t()), xa, b_.t())
            ctx.save_for_backward(x, w, a_, b_, xa)
            return y.view(*x.shape[:-1], w.shape[0])

        @staticmethod
        def backward(ctx, dy):
            x, w, a_, b_, xa = ctx.saved_tensors
            x2 = x.reshape(-1, x.shape[-1])
            dy2 = dy.reshape(-1, dy.shape[-1])
            dxa = dy2.mm(b_)
            ng = ctx.needs_input_grad
            dx = dy2.mm(w).addmm_(dxa, a_).view(x.shape) if ng[0] else None
            dw = dy2.t().mm(x2) if ng[1] else None
            da = dxa.t().mm(x2) if ng[2] else None
            db = dy2.t().mm(xa) if ng[3] else None
            return dx, dw, da, db

    class GptMlp(torch.autograd.Function):
        """fc2(gelu_tanh(fc(m))) with the bias + GELU in the fc GEMM's cuBLASLt
        epilogue (GELU_AUX_BIAS, the pre-activation kept as aux) and, in the
        backward, the GELU derivative and the fc bias gradient in the epilogue of
        the fc2 input-gradient GEMM (DGELU_BGRAD): no separate elementwise pass
        on the [tokens x 4h] activations in either direction."""

        @staticmethod
        def forward(ctx, m, fc_w, fc_b, fc2_w, fc2_b):
            h = m.shape[-1]
            ffn = fc_w.shape[0]
            m2 = m.reshape(-1, h)
            if not m2.is_contiguous():
                m2 = m2.contiguous()
            rows = m2.shape[0]
            act = torch.empty(rows, ffn, dtype=m.dtype, device=m.device)
            aux = torch.empty_like(act)
            check(lib().fcdp_fc_gelu_fwd(rows, h, ffn, P(m2), P(fc_w), P(fc_b), P(act), P(aux), S(m.device)))
            out = torch.nn.functional.linear(act, fc2_w, fc2_b)
            ctx.save_for_backward(m2, fc_w, fc2_w, act, aux)
            ctx.mshape = m.shape
            return out.view(*m.shape[:-1], fc2_w.shape[0])

        @staticmethod
        def backward(ctx, dout):
            m2, fc_w, fc2_w, act, aux = ctx.saved_tensors
            rows, ffn = act.shape
            h = m2.shape[1]
            d2 = dout.reshape(rows, -1)
            if not d2.is_contiguous():
                d2 = d2.contiguous()
            ng = ctx.needs_input_grad
            d_fc2_b = bias_grad(d2) if ng[4] else None
            d_fc2_w = d2.t().mm(act) if ng[3] else None
            dpre = torch.empty_like(aux)
            d_fc_b = torch.empty(ffn, dtype=aux.dtype, device=aux.device)
            check(lib().fcdp_fc2_dgrad_dgelu(rows, d2.shape[1], ffn, P(d2), P(fc2_w), P(aux), P(dpre), P(d_fc_b),
                                             S(aux.device)))
            d_fc_w = dpre.t().mm(m2) if ng[1] else None
            dm = dpre.mm(fc_w).view(ctx.mshape) if ng[0] else None
            return dm, d_fc_w, (d_fc_b if ng[2] else None), d_fc2_w, d_fc2_b

    from types import SimpleNamespace
    _FNS = SimpleNamespace(GptMlp=GptMlp, LinearBias=LinearBias, BiasGelu=BiasGelu, CrossEntropy=CrossEntropy, Rope=Rope,
                           GateUpSwiGLU=GateUpSwiGLU, LlamaQKV=LlamaQKV, LoraLinear=LoraLinear)
    return _FNS


def _llama_qkv(p, a, nh):
    """(q, k, v) [b, s, nh, hd] with RoPE on q, k: the joint projection when the
    q|k|v weights (and LoRA A's) are adjacent in the layer buffer, else per tensor."""
    lora = "q_A" in p
    if (_fused_ok(a, p["q_w"]) and a.shape[-1] // nh % 8 == 0 and _adjacent(p["q_w"], p["k_w"])
            and _adjacent(p["k_w"], p["v_w"])
            and (not lora or (_adjacent(p["q_A"], p["k_A"]) and _adjacent(p["k_A"], p["v_A"])))):
        args = [p[f"{n}_A"] for n in "qkv"] + [p[f"{n}_B"] for n in "qkv"] if lora else [None] * 6
        return _fns().LlamaQKV.apply(a, p["q_w"], p["k_w"], p["v_w"], *args, nh)
    return None


def _adjacent(a, b) -> bool:
    """b starts where a ends in the same storage (consecutive tensors of a layer buffer)."""
    return (a.is_contiguous() and b.is_contiguous() and a.untyped_storage().data_ptr() == b.untyped_storage().data_ptr()
            and b.data_ptr() == a.data_ptr() + a.numel() * a.element_size() and a.shape == b.shape)


def _swiglu_mlp(m, wg, wu):
    import torch.nn.functional as F
    if _fused_ok(m, wg, wu) and wg.shape[0] % 8 == 0 and _adjacent(wg, wu):
        return _fns().GateUpSwiGLU.apply(m, wg, wu)
    return F.silu(F.linear(m, wg)) * F.linear(m, wu)


def _rope_fn(x):
    if _fused_ok(x) and x.shape[-1] % 8 == 0:
        return _fns().Rope.apply(x)
    return _rope(x)


def _linear_bias(x, w, b):
    import torch.nn.functional as F
    if _fused_ok(x, w, b) and w.shape[0] % 8 == 0:
        return _fns().LinearBias.apply(x, w, b)
    return F.linear(x, w, b)


def _mlp_gelu(m, w, b):
    """gelu_tanh(m W^T + b): the GEMM without its bias, bias + GELU fused."""
    import torch.nn.functional as F
    if _fused_ok(m, w, b) and w.shape[0] % 8 == 0:
        return _fns().BiasGelu.apply(F.linear(m, w), b)
    return F.gelu(F.linear(m, w, b), approximate="tanh")


_MLP_LT = None


def _gpt2_mlp(m, p):
    """fc2(gelu_tanh(fc(m) + b1)) + b2 with the bias + GELU kernels.  FCDP_MLP_LT=1
    selects the cuBLASLt epilogue fusion instead (GptMlp): correct, but the
    epilogue GEMMs the heuristic picks are slower on B200 - 80.4-82.0 ms per
    GPT-2 1.3B step against 68.5-68.7 ms (profiles/r02_ab_mlp_epilogue.json)."""
    global _MLP_LT
    if _fused_ok(m, p["fc_w"]) and p["fc_w"].shape[0] % 8 == 0 and m.shape[-1] % 8 == 0:
        if _MLP_LT is None:
            import os
            from ._capi import lib
            _MLP_LT = os.environ.get("FCDP_MLP_LT", "0") != "0" and lib().fcdp_mlp_gemm_available() == 1
        if _MLP_LT:
            return _fns().GptMlp.apply(m, p["fc_w"], p["fc_b"], p["fc2_w"], p["fc2_b"])
    return _linear_bias(_mlp_gelu(m, p["fc_w"], p["fc_b"]), p["fc2_w"], p["fc2_b"])


def _cross_entropy(logits, labels):
    import torch.nn.functional as F
    if _fused_ok(logits) and logits.shape[-1] % 8 == 0:
        return _fns().CrossEntropy.apply(logits.reshape(-1, logits.shape[-1]), labels.reshape(-1))
    return F.cross_entropy(logits.float().view(-1, logits.shape[-1]), labels.reshape(-1))


def layer_forward(cfg: ModelConfig, ldef: LayerDef, p, x, tokens=None, labels=None):
    """Forward of one layer.  x: [b, s, h] (None for the embedding)."""
    import torch
    import torch.nn.functional as F
    h, nh = cfg.hidden, cfg.heads
    if ldef.kind == "embed":
        y = F.embedding(tokens, p["wte"])
        if "wpe" in p:
            y = y + p["wpe"][: tokens.shape[1]].unsqueeze(0)
        return y
    if ldef.kind == "gpt2_block":
        b, s, _ = x.shape
        a = _layer_norm(x, p["ln1_w"], p["ln1_b"])
        # q, k, v stay [b, s, nh, hd] in memory and reach SDPA as transposed views;
        # the output comes back in the same layout, so neither direction needs a
        # strided copy (tools/attn_layout_probe.py: 0.85 vs 1.29 ms per block fwd+bwd)
        q, k, v = _linear_bias(a, p["qkv_w"], p["qkv_b"]).view(b, s, 3, nh, h // nh).unbind(2)
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), is_causal=True)
        x, m = _add_layer_norm(x, _linear_bias(o.transpose(1, 2).reshape(b, s, h), p["proj_w"], p["proj_b"]),
                               p["ln2_w"], p["ln2_b"])
        return x + _gpt2_mlp(m, p)
    if ldef.kind == "llama_block":
        b, s, _ = x.shape
        a = _rms_norm(x, p["attn_norm"])

        def proj(name, inp):
            if f"{name}_A" in p and _fused_ok(inp, p[f"{name}_w"]):
                return _fns().LoraLinear.apply(inp, p[f"{name}_w"], p[f"{name}_A"], p[f"{name}_B"])
            y = F.linear(inp, p[f"{name}_w"])
            if f"{name}_A" in p:
                # y + (x A^T) B^T with the add in the LoRA GEMM's epilogue (addmm, beta = 1)
                xa = F.linear(inp, p[f"{name}_A"])
                y = torch.addmm(y.reshape(-1, y.shape[-1]), xa.reshape(-1, xa.shape[-1]),
                                p[f"{name}_B"].t()).view(y.shape)
            return y
        qkv = _llama_qkv(p, a, nh)
        if qkv is not None:
            q, k, v = (t.transpose(1, 2) for t in qkv)
        else:
            q = _rope_fn(proj("q", a).view(b, s, nh, h // nh)).transpose(1, 2)
            k = _rope_fn(proj("k", a).view(b, s, nh, h // nh)).transpose(1, 2)
            v = proj("v", a).view(b, s, nh, h // nh).transpose(1, 2)
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x, m = _rms_norm(x, p["mlp_norm"], r=proj("o", o.transpose(1, 2).reshape(b, s, h)))
        return x + F.linear(_swiglu_mlp(m, p["gate_w"], p["up_w"]), p["down_w"])
    if ldef.kind == "head":
        if "lnf_w" in p:
            a = _layer_norm(x, p["lnf_w"], p["lnf_b"])
        else:
            a = _rms_norm(x, p["norm_w"])
        logits = F.linear(a, p["lm_w"])
        return _cross_entropy(logits, labels)
    raise ValueError(ldef.kind)
