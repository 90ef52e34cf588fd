"""Kernel parity at BASELINE.json's full layer sizes, through size-independent
properties (the CPU oracle would take minutes per layer at these sizes).

* partition -> expand round trip is the identity on the natural layer, for a
  C2 GPT-2 1.3B block (dense), a C3 Llama-7B block with its LoRA r=16 q,k,v,o
  chunk mask, and a C4 Llama-13B block, at the 2x4 geometry (G = 8);
* the fused reduce-scatter of g identical gradients with scale 1/g returns the
  gradient exactly (a sum of <= 8 equal bf16 values is exact in fp32 and 1/g is
  a power of two) - every shard, every slice, full C2 block;
* AdamW over a 100M-element shard agrees bit-exactly with the C oracle on a
  random sample of positions (elementwise op: sampling loses nothing).
All calls go through the C ABI.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _block_mask(preset, eb=2):
    from paper_2602_06499_b200.driving_model import PRESETS
    defs = PRESETS[preset].layer_defs()
    block = next(d for d in defs if d.kind.endswith("_block"))
    return block.chunk_mask(eb)


@pytest.mark.parametrize("preset,params", [("gpt2-1.3b", 50_358_272), ("llama7b-lora16", 202_907_648),
                                           ("llama13b", 317_204_480)])
def test_roundtrip_full_layer(built, preset, params):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    m = _block_mask(preset)
    chunks = m.size
    assert chunks * 8 == params  # SURVEY §8 sizes
    N, g = 2, 4
    lay = C.c_void_p()
    check(lib.fcdp_layout_create(chunks, m.ctypes.data_as(C.POINTER(C.c_uint8)), 2, N, g, C.byref(lay)))
    geo = O.geom(chunks, m, N, g)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0x5EED)
    nat = torch.randint(0, 256, (chunks * 16,), dtype=torch.uint8, device=dev, generator=gen)
    t = torch.zeros(max(geo.slice_t * g, 1) * 16, dtype=torch.uint8, device=dev)
    f = torch.zeros(max(geo.slice_f * g, 1) * 16, dtype=torch.uint8, device=dev)
    check(lib.fcdp_partition(lay, _ptr(nat), _ptr(t), _ptr(f), None))
    T = (C.c_void_p * g)(*[t.data_ptr() + j * geo.slice_t * 16 for j in range(g)])
    F = (C.c_void_p * g)(*[f.data_ptr() + j * geo.slice_f * 16 for j in range(g)])
    out = torch.zeros_like(nat)
    check(lib.fcdp_expand(lay, T, F, _ptr(out), 0, None))  # set All
    torch.cuda.synchronize()
    assert torch.equal(out, nat)
    if geo.pt and geo.pf:  # trainable-only expand leaves frozen chunks untouched
        out2 = torch.zeros_like(nat)
        check(lib.fcdp_expand(lay, T, F, _ptr(out2), 1, None))
        torch.cuda.synchronize()
        mk = torch.from_numpy(m.astype(bool)).to(dev).repeat_interleave(16)
        assert torch.equal(out2[mk], nat[mk])
        assert int(out2[~mk].count_nonzero()) == 0
    lib.fcdp_layout_destroy(lay)


def test_rs_identical_grads_full_layer(built):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    chunks = 50_358_272 // 8
    m = np.ones(chunks, np.uint8)
    N, g = 1, 4
    lay = C.c_void_p()
    check(lib.fcdp_layout_create(chunks, m.ctypes.data_as(C.POINTER(C.c_uint8)), 2, N, g, C.byref(lay)))
    geo = O.geom(chunks, m, N, g)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    x = torch.randn(chunks * 8, device=dev, generator=gen).to(torch.bfloat16)
    G = (C.c_void_p * g)(*([x.data_ptr()] * g))
    own = torch.empty(geo.shard_t * 8, dtype=torch.float32, device=dev)
    wire = torch.empty(geo.slice_t * 16, dtype=torch.uint8, device=dev)
    for j in range(g):
        check(lib.fcdp_rs_slice(lay, G, j, 0, 1.0 / g, 1, _ptr(own), _ptr(wire), None))
        torch.cuda.synchronize()
        lo = j * geo.slice_t * 8
        n = min(geo.slice_t * 8, x.numel() - lo)
        assert torch.equal(own[:n], x[lo:lo + n].float()), j
    lib.fcdp_layout_destroy(lay)


def test_adam_full_shard_sampled(built):
    from paper_2602_06499_b200 import _capi
    dev = _dev()
    lib = built
    n = 100_000_000
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    w = torch.randn(n, device=dev, generator=gen)
    mm = torch.randn(n, device=dev, generator=gen).mul_(1e-3)
    vv = torch.rand(n, device=dev, generator=gen).mul_(1e-6)
    gr = torch.randn(n, device=dev, generator=gen).mul_(1e-2)
    idx = torch.from_numpy(np.random.default_rng(3).choice(n, 200_000, replace=False)).to(dev)
    w0, m0, v0, g0 = (a[idx].cpu().numpy().copy() for a in (w, mm, vv, gr))
    p = torch.zeros(n * 2, dtype=torch.uint8, device=dev)
    cfg = _capi.AdamConfig(1e-3, 0.9, 0.95, 1e-8, 0.1, 7)
    _capi.check(lib.fcdp_adam_step(n, C.byref(cfg), _ptr(w), _ptr(mm), _ptr(vv), _ptr(gr), _ptr(p), 2, None))
    torch.cuda.synchronize()
    pr = np.zeros(w0.size, np.uint16)
    O.adam(w0, m0, v0, g0, pr, 1e-3, 0.9, 0.95, 1e-8, 0.1, 7)
    assert np.array_equal(w[idx].cpu().numpy().view(np.uint32), w0.view(np.uint32))
    assert np.array_equal(mm[idx].cpu().numpy().view(np.uint32), m0.view(np.uint32))
    assert np.array_equal(vv[idx].cpu().numpy().view(np.uint32), v0.view(np.uint32))
    assert np.array_equal(p.view(torch.int16)[idx].cpu().numpy().view(np.uint16), pr)
