"""Parity of each sm_100a data-plane kernel with the CPU oracle (bit-exact).

All calls go through the C ABI (include/fcdp.h) on cuda:0; slices that in a
real job live on NVLink peers are separate local allocations here (the
multi-GPU path is covered by tests/test_engine_gpu.py).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from tests.maskgen import masks

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _layout(lib, chunks, mask, eb, N, g):
    from paper_2602_06499_b200._capi import check
    m = (C.c_uint8 * chunks)(*mask.tolist())
    out = C.c_void_p()
    check(lib.fcdp_layout_create(chunks, m, eb, N, g, C.byref(out)))
    return out


def _u8(a: np.ndarray, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8).copy()).to(dev)


SIZES = [1, 33, 4096 + 7]
GEOS = [(1, 1), (2, 1), (1, 4), (2, 2), (2, 4), (4, 2), (1, 8), (8, 1), (1, 3)]


@pytest.mark.parametrize("chunks", SIZES)
@pytest.mark.parametrize("N,g", GEOS)
def test_expand_bit_exact(built, chunks, N, g):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    rng = np.random.default_rng(chunks * 31 + N * 7 + g)
    for name, m in masks(chunks, chunks + g):
        geo = O.geom(chunks, m, N, g)
        lay = _layout(lib, chunks, m, 2, N, g)
        ts = [rng.integers(0, 256, max(geo.slice_t, 1) * 16, dtype=np.uint8) for _ in range(g)]
        fs = [rng.integers(0, 256, max(geo.slice_f, 1) * 16, dtype=np.uint8) for _ in range(g)]
        dts = [_u8(x, dev) for x in ts]
        dfs = [_u8(x, dev) for x in fs]
        for pset in (0, 1, 2):
            ref = np.full(chunks * 16, 0x5A, np.uint8)
            O.expand(geo, m, ts, fs, ref, pset)
            out = torch.full((chunks * 16,), 0x5A, dtype=torch.uint8, device=dev)
            T = (C.c_void_p * g)(*[t.data_ptr() for t in dts])
            F = (C.c_void_p * g)(*[t.data_ptr() for t in dfs])
            check(lib.fcdp_expand(lay, T, F, _ptr(out), pset, None))
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), ref), (name, pset)
        lib.fcdp_layout_destroy(lay)


@pytest.mark.parametrize("chunks", SIZES)
def test_partition_bit_exact(built, chunks):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    rng = np.random.default_rng(chunks)
    for name, m in masks(chunks, chunks):
        nat = rng.integers(0, 256, chunks * 16, dtype=np.uint8)
        t, f = O.partition(nat, m)
        lay = _layout(lib, chunks, m, 2, 2, 2)
        dt = torch.zeros(max(t.size, 16), dtype=torch.uint8, device=dev)
        df = torch.zeros(max(f.size, 16), dtype=torch.uint8, device=dev)
        dnat = _u8(nat, dev)
        check(lib.fcdp_partition(lay, _ptr(dnat), _ptr(dt), _ptr(df), None))
        torch.cuda.synchronize()
        assert np.array_equal(dt.cpu().numpy()[:t.size], t), name
        assert np.array_equal(df.cpu().numpy()[:f.size], f), name
        lib.fcdp_layout_destroy(lay)


@pytest.mark.parametrize("eb", [2, 4])
@pytest.mark.parametrize("N,g", [(1, 1), (2, 1), (1, 4), (2, 2), (2, 4), (1, 8), (1, 3)])
def test_rs_slice_bit_exact(built, eb, N, g):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    chunks = 777
    V = 16 // eb
    rng = np.random.default_rng(eb * 100 + N * 10 + g)
    for name, m in masks(chunks, 11):
        geo = O.geom(chunks, m, N, g)
        lay = _layout(lib, chunks, m, eb, N, g)
        x = [rng.standard_normal(chunks * V).astype(np.float32) for _ in range(g)]
        grads = [O.f32_to_bf16(a) for a in x] if eb == 2 else x
        dg = [_u8(a, dev) for a in grads]
        G = (C.c_void_p * g)(*[t.data_ptr() for t in dg])
        for j in range(g):
            for n in range(N):
                for final in (False, True):
                    own, wire = O.rs_slice(geo, m, eb, grads, j, n, 1.0 / (N * g), final)
                    down = torch.zeros(max(own.size, 4), dtype=torch.float32, device=dev)
                    dwire = torch.zeros(max(wire.nbytes, 16), dtype=torch.uint8, device=dev)
                    check(lib.fcdp_rs_slice(lay, G, j, n, 1.0 / (N * g), int(final), _ptr(down), _ptr(dwire), None))
                    torch.cuda.synchronize()
                    assert np.array_equal(down.cpu().numpy()[:own.size].view(np.uint32), own.view(np.uint32)), (name, j, n)
                    # only non-own shard chunks of the wire buffer are defined
                    w = dwire.cpu().numpy()[:wire.nbytes].view(wire.dtype)
                    sel = np.ones(wire.size, bool)
                    sel[n * geo.shard_t * V:(n + 1) * geo.shard_t * V] = False
                    real = np.zeros(wire.size, bool)
                    real[:max(0, min(geo.slice_t, geo.pt - j * geo.slice_t)) * V] = True
                    sel &= real
                    assert np.array_equal(w[sel].view(np.uint8), wire[sel].view(np.uint8)), (name, j, n)
        lib.fcdp_layout_destroy(lay)


@pytest.mark.parametrize("eb", [2, 4])
def test_rs_finalize_bit_exact(built, eb):
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    rng = np.random.default_rng(5)
    n, N = 10008, 4  # whole 16-byte chunks (multiple of 4 elements)
    own = rng.standard_normal(n).astype(np.float32)
    wf = rng.standard_normal(N * n).astype(np.float32)
    wire = O.f32_to_bf16(wf) if eb == 2 else wf
    for node in range(N):
        ref = O.rs_finalize(own, wire, N, node, eb, n, 0.125)
        out = torch.zeros(n, dtype=torch.float32, device=dev)
        down, dwire = _u8(own, dev), _u8(wire, dev)  # keep alive until the kernel ran
        check(lib.fcdp_rs_finalize(n, N, node, eb, _ptr(down), _ptr(dwire), n, 0.125, _ptr(out), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("eb", [2, 4])
def test_adam_bit_exact(built, eb):
    from paper_2602_06499_b200 import _capi
    dev = _dev()
    lib = built
    rng = np.random.default_rng(9)
    n = 50001
    w = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    p = np.zeros(n, np.uint16 if eb == 2 else np.float32)
    dw, dm, dv = (torch.from_numpy(a.copy()).to(dev) for a in (w, m, v))
    dp = torch.zeros(n * eb, dtype=torch.uint8, device=dev)
    for step in range(1, 4):
        g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        O.adam(w, m, v, g, p, 1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        cfg = _capi.AdamConfig(1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        dg = torch.from_numpy(g).to(dev)
        _capi.check(lib.fcdp_adam_step(n, C.byref(cfg), _ptr(dw), _ptr(dm), _ptr(dv), _ptr(dg), _ptr(dp),
                                       eb, None))
        torch.cuda.synchronize()
        assert np.array_equal(dw.cpu().numpy().view(np.uint32), w.view(np.uint32)), step
        assert np.array_equal(dv.cpu().numpy().view(np.uint32), v.view(np.uint32)), step
        assert np.array_equal(dp.cpu().numpy(), p.view(np.uint8)), step


@pytest.mark.parametrize("eb", [2, 4])
def test_fused_grad_adam_bit_exact(built, eb):
    """G = 1 fused RS + AdamW (the engine's one-GPU path) vs the oracle's RS
    (g = 1, final scale) followed by its AdamW: masters, moments, parameter
    shard and the kept fp32 gradient bit for bit, with the gradient handed over
    as segments that leave gaps (uncovered elements = gradient 0) and include
    -0.0 / zero gradients."""
    from paper_2602_06499_b200 import _capi
    dev = _dev()
    lib = built
    V = 16 // eb
    rng = np.random.default_rng(23)
    chunks = 9001
    n = chunks * V
    mask = np.ones(chunks, np.uint8)
    geo = O.geom(chunks, mask, 1, 1)
    w = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    p = np.zeros(n, np.uint16 if eb == 2 else np.float32)
    dw, dm, dv = (torch.from_numpy(a.copy()).to(dev) for a in (w, m, v))
    dp = torch.zeros(n * eb, dtype=torch.uint8, device=dev)
    keep = torch.zeros(n, dtype=torch.float32, device=dev)
    segs = [(0, 1000 * V), (1000 * V, 3000 * V), (4500 * V, 4000 * V), (8600 * V, 401 * V)]  # gap 4000..4500
    for step in range(1, 4):
        x = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        x[:64] = 0.0
        x[64:128] = -0.0
        nat = O.f32_to_bf16(x) if eb == 2 else x
        covered = np.zeros(n, bool)
        for o, c in segs:
            covered[o:o + c] = True
        nat = np.where(covered, nat, np.zeros_like(nat))
        own, _ = O.rs_slice(geo, mask, eb, [nat], 0, 0, 1.0, True)
        O.adam(w, m, v, own, p, 1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        dnat = torch.from_numpy(nat.view(np.uint8).copy()).to(dev)
        base = dnat.data_ptr()
        offs = (C.c_int64 * len(segs))(*[o for o, _ in segs])
        ptrs = (C.c_void_p * len(segs))(*[base + o * eb for o, _ in segs])
        cnts = (C.c_int64 * len(segs))(*[c for _, c in segs])
        cfg = _capi.AdamConfig(1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        _capi.check(lib.fcdp_adam_grad_step(n, C.byref(cfg), 1.0, len(segs), offs, ptrs, cnts, _ptr(dw), _ptr(dm),
                                            _ptr(dv), _ptr(dp), eb, _ptr(keep), None))
        torch.cuda.synchronize()
        assert np.array_equal(keep.cpu().numpy().view(np.uint32), own.view(np.uint32)), step
        assert np.array_equal(dw.cpu().numpy().view(np.uint32), w.view(np.uint32)), step
        assert np.array_equal(dm.cpu().numpy().view(np.uint32), m.view(np.uint32)), step
        assert np.array_equal(dv.cpu().numpy().view(np.uint32), v.view(np.uint32)), step
        assert np.array_equal(dp.cpu().numpy(), p.view(np.uint8)), step


@pytest.mark.parametrize("eb", [2, 4])
def test_init_bit_exact(built, eb):
    from paper_2602_06499_b200 import _capi
    dev = _dev()
    lib = built
    chunks = 5000
    n = chunks * 16 // eb
    lay = _layout(lib, chunks, np.ones(chunks, np.uint8), eb, 1, 1)
    ranges = [(0, n // 2, 0, 0.02), (n // 2, n // 2 + 100, 1, 1.0), (n // 2 + 100, n, 0, 0.5)]
    ref = O.init_natural(n, eb, 0x5EED, 7, ranges)
    R = (_capi.InitRange * 3)(*[_capi.InitRange(*r) for r in ranges])
    out = torch.zeros(n * eb, dtype=torch.uint8, device=dev)
    _capi.check(lib.fcdp_init_natural(lay, 0x5EED, 7, R, 3, _ptr(out), None))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref.view(np.uint8))
    lib.fcdp_layout_destroy(lay)


_TMA_SCRIPT = r"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import oracle as O
from paper_2602_06499_b200 import _capi
lib = _capi.lib()
dev = torch.device("cuda", 0)
rng = np.random.default_rng(3)
for chunks, g in ((4099, 1), (100003, 4), (7, 2)):
    m = np.ones(chunks, np.uint8)
    geo = O.geom(chunks, m, 1, g)
    lay = C.c_void_p()
    _capi.check(lib.fcdp_layout_create(chunks, m.ctypes.data_as(C.POINTER(C.c_uint8)), 2, 1, g, C.byref(lay)))
    ts = [rng.integers(0, 256, geo.slice_t * 16, dtype=np.uint8) for _ in range(g)]
    ref = np.zeros(chunks * 16, np.uint8)
    O.expand(geo, m, ts, [None] * g, ref, 0)
    dts = [torch.from_numpy(x).to(dev) for x in ts]
    out = torch.zeros(chunks * 16, dtype=torch.uint8, device=dev)
    _capi.check(lib.fcdp_expand(lay, (C.c_void_p * g)(*[t.data_ptr() for t in dts]), None, C.c_void_p(out.data_ptr()), 0, None))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref), (chunks, g)
print("tma-ok")
"""


def test_tma_bulk_copy_path(built):
    """The TMA bulk-copy gather (FCDP_COPY=tma, read once per process) is bit-exact too."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    _dev()
    root = str(Path(__file__).resolve().parents[1])
    r = subprocess.run([sys.executable, "-c", _TMA_SCRIPT, root], env=dict(os.environ, FCDP_COPY="tma"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "tma-ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("eb", [2, 4])
def test_adam_special_values_bit_exact(built, eb):
    """AdamW on gradients that exercise the IEEE division / sqrt edge paths:
    exact zeros (0/eps), denormal squares, huge and tiny magnitudes."""
    from paper_2602_06499_b200 import _capi
    dev = _dev()
    lib = built
    rng = np.random.default_rng(17)
    n = 4096
    g = np.concatenate([np.zeros(1024, np.float32),                               # 0 -> m = v = 0 paths
                        (rng.standard_normal(1024) * 1e-22).astype(np.float32),   # g*g underflows to denormal/0
                        (rng.standard_normal(1024) * 1e18).astype(np.float32),    # g*g near the fp32 max
                        (rng.standard_normal(1024) * 1e-3).astype(np.float32)])
    w = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    p = np.zeros(n, np.uint16 if eb == 2 else np.float32)
    dw, dm, dv, dg = (torch.from_numpy(a.copy()).to(dev) for a in (w, m, v, g))
    dp = torch.zeros(n * eb, dtype=torch.uint8, device=dev)
    for step in (1, 2):
        O.adam(w, m, v, g, p, 1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        cfg = _capi.AdamConfig(1e-3, 0.9, 0.95, 1e-8, 0.1, step)
        _capi.check(lib.fcdp_adam_step(n, C.byref(cfg), _ptr(dw), _ptr(dm), _ptr(dv), _ptr(dg), _ptr(dp), eb, None))
        torch.cuda.synchronize()
        assert np.array_equal(dw.cpu().numpy().view(np.uint32), w.view(np.uint32)), step
        assert np.array_equal(dm.cpu().numpy().view(np.uint32), m.view(np.uint32)), step
        assert np.array_equal(dv.cpu().numpy().view(np.uint32), v.view(np.uint32)), step
        assert np.array_equal(dp.cpu().numpy(), p.view(np.uint8)), step


def test_expand_partition_random_shapes_bit_exact(built):
    """Randomised: sizes 1..3000 chunks, any mask density, every node x GPU shape
    up to 8 GPUs, every portion set - CUDA expand and partition vs the oracle."""
    hyp = pytest.importorskip("hypothesis")
    from hypothesis import given, settings, strategies as st
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built

    @settings(max_examples=40, deadline=None, derandomize=True)
    @given(chunks=st.integers(1, 3000), density=st.floats(0.0, 1.0),
           shape=st.sampled_from([(1, 1), (2, 1), (1, 2), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8), (8, 1), (2, 3)]),
           seed=st.integers(0, 2**31 - 1), pset=st.sampled_from([0, 1, 2]))
    def run(chunks, density, shape, seed, pset):
        N, g = shape
        rng = np.random.default_rng(seed)
        m = (rng.random(chunks) < density).astype(np.uint8)
        geo = O.geom(chunks, m, N, g)
        lay = _layout(lib, chunks, m, 2, N, g)
        try:
            nat = rng.integers(0, 256, chunks * 16, dtype=np.uint8)
            t, f = O.partition(nat, m)
            dnat = _u8(nat, dev)
            dt = torch.zeros(max(geo.slice_t * g, 1) * 16, dtype=torch.uint8, device=dev)
            df = torch.zeros(max(geo.slice_f * g, 1) * 16, dtype=torch.uint8, device=dev)
            check(lib.fcdp_partition(lay, _ptr(dnat), _ptr(dt), _ptr(df), None))
            torch.cuda.synchronize()
            assert np.array_equal(dt.cpu().numpy()[:t.size], t)
            assert np.array_equal(df.cpu().numpy()[:f.size], f)
            T = (C.c_void_p * g)(*[dt.data_ptr() + j * geo.slice_t * 16 for j in range(g)])
            F = (C.c_void_p * g)(*[df.data_ptr() + j * geo.slice_f * 16 for j in range(g)])
            out = torch.full((chunks * 16,), 0x5A, dtype=torch.uint8, device=dev)
            check(lib.fcdp_expand(lay, T, F, _ptr(out), pset, None))
            torch.cuda.synchronize()
            tp = dt.cpu().numpy(); fp = df.cpu().numpy()
            ref = np.full(chunks * 16, 0x5A, np.uint8)
            O.expand(geo, m, [tp[j * geo.slice_t * 16:(j + 1) * geo.slice_t * 16] for j in range(g)],
                     [fp[j * geo.slice_f * 16:(j + 1) * geo.slice_f * 16] for j in range(g)], ref, pset)
            assert np.array_equal(out.cpu().numpy(), ref)
        finally:
            lib.fcdp_layout_destroy(lay)

    run()


def test_rs_random_shapes_bit_exact(built):
    """Randomised reduce-scatter: random masks / sizes / shapes (g up to 8) and
    both dtypes; intra-node RS kernel (own fp32 shard + wire) then the
    inter-node epilogue, each vs the oracle bit for bit."""
    pytest.importorskip("hypothesis")
    from hypothesis import given, settings, strategies as st
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built

    @settings(max_examples=25, deadline=None, derandomize=True)
    @given(chunks=st.integers(1, 1500), density=st.floats(0.01, 1.0),
           shape=st.sampled_from([(1, 1), (2, 1), (1, 2), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8), (3, 2)]),
           eb=st.sampled_from([2, 4]), seed=st.integers(0, 2**31 - 1))
    def run(chunks, density, shape, eb, seed):
        N, g = shape
        V = 16 // eb
        rng = np.random.default_rng(seed)
        m = (rng.random(chunks) < density).astype(np.uint8)
        geo = O.geom(chunks, m, N, g)
        lay = _layout(lib, chunks, m, eb, N, g)
        try:
            xs = [rng.standard_normal(chunks * V).astype(np.float32) for _ in range(g)]
            grads = [O.f32_to_bf16(a) for a in xs] if eb == 2 else xs
            dg = [_u8(a, dev) for a in grads]
            G = (C.c_void_p * g)(*[t.data_ptr() for t in dg])
            j, n = int(rng.integers(0, g)), int(rng.integers(0, N))
            scale = 1.0 / (N * g)
            own, wire = O.rs_slice(geo, m, eb, grads, j, n, scale, N == 1)
            down = torch.zeros(max(own.size, 4), dtype=torch.float32, device=dev)
            dwire = torch.zeros(max(wire.nbytes, 16), dtype=torch.uint8, device=dev)
            check(lib.fcdp_rs_slice(lay, G, j, n, scale, int(N == 1), _ptr(down), _ptr(dwire), None))
            torch.cuda.synchronize()
            assert np.array_equal(down.cpu().numpy()[:own.size].view(np.uint32), own.view(np.uint32))
            # the wire: real chunks of the other nodes' shards, cast to the param dtype
            w = dwire.cpu().numpy()[:wire.nbytes].view(wire.dtype)
            sel = np.zeros(wire.size, bool)
            sel[:max(0, min(geo.slice_t, geo.pt - j * geo.slice_t)) * V] = True
            sel[n * geo.shard_t * V:(n + 1) * geo.shard_t * V] = False
            assert np.array_equal(w[sel].view(np.uint8), wire[sel].view(np.uint8))
            if N > 1 and geo.shard_t:
                sh = geo.shard_t * V
                # the epilogue's input is the kernel's own wire output, as a peer node would send it
                rx = np.zeros(N * sh, wire.dtype)
                for m_ in range(N):
                    if m_ != n:
                        rx[m_ * sh:(m_ + 1) * sh] = w[m_ * sh:(m_ + 1) * sh]
                ref = O.rs_finalize(own[:sh].copy(), rx, N, n, eb, sh, scale)
                drx, downs = _u8(rx, dev), down[:sh].contiguous()
                out = torch.zeros(sh, dtype=torch.float32, device=dev)
                check(lib.fcdp_rs_finalize(sh, N, n, eb, _ptr(downs), _ptr(drx), sh, scale, _ptr(out), None))
                torch.cuda.synchronize()
                assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        finally:
            lib.fcdp_layout_destroy(lay)

    run()


def test_copy_segments_exact(built):
    """fcdp_copy_segments (the masked-layer gradient hand-off): 40 random
    16-byte aligned segments (two launches) land exactly, nothing else is touched."""
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    rng = np.random.default_rng(7)
    sizes = [int(x) * 16 for x in rng.integers(0, 5000, 40)]
    srcs = [torch.from_numpy(rng.integers(0, 256, max(n, 16), dtype=np.uint8)).to(dev) for n in sizes]
    out = torch.full((sum(sizes) + 16 * 41,), 0xA5, dtype=torch.uint8, device=dev)
    offs, o = [], 0
    for n in sizes:
        offs.append(o)
        o += n + 16
    n = len(sizes)
    check(lib.fcdp_copy_segments(n, (C.c_void_p * n)(*[t.data_ptr() for t in srcs]),
                                 (C.c_void_p * n)(*[out.data_ptr() + x for x in offs]), (C.c_int64 * n)(*sizes), None))
    torch.cuda.synchronize()
    host = out.cpu().numpy()
    ref = np.full_like(host, 0xA5)
    for t, x, sz in zip(srcs, offs, sizes):
        ref[x:x + sz] = t.cpu().numpy()[:sz]
    assert np.array_equal(host, ref)


def test_copy_rows_exact(built):
    """fcdp_copy_rows: a strided third of a [rows x 3h] matrix to a dense [rows x h] and back."""
    from paper_2602_06499_b200._capi import check
    dev = _dev()
    lib = built
    rows, h = 333, 264
    src = torch.randint(-30000, 30000, (rows, 3 * h), dtype=torch.int16, device=dev)
    dst = torch.zeros(rows, h, dtype=torch.int16, device=dev)
    check(lib.fcdp_copy_rows(rows, h * 2, C.c_void_p(src.data_ptr() + 2 * h * 2), 3 * h * 2, _ptr(dst), h * 2, None))
    back = torch.zeros_like(src)
    check(lib.fcdp_copy_rows(rows, h * 2, _ptr(dst), h * 2, C.c_void_p(back.data_ptr() + h * 2), 3 * h * 2, None))
    torch.cuda.synchronize()
    assert torch.equal(dst, src[:, 2 * h:])
    assert torch.equal(back[:, h:2 * h], src[:, 2 * h:]) and int(back[:, :h].abs().sum()) == 0
