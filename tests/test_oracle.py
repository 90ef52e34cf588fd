"""CPU oracle self-checks (no GPU): the restatement is consistent with itself
and with independent numpy formulations before it is trusted as the checker."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.maskgen import masks


@pytest.mark.parametrize("chunks", [1, 31, 32, 33, 1000])
def test_partition_roundtrip(chunks):
    rng = np.random.default_rng(chunks)
    nat = rng.integers(0, 256, chunks * 16, dtype=np.uint8)
    for name, m in masks(chunks, chunks):
        t, f = O.partition(nat, m)
        back = O.unpartition(t, f, m, chunks)
        assert np.array_equal(back, nat), name
        # numpy formulation of the compaction
        c = nat.reshape(chunks, 16)
        assert np.array_equal(t.reshape(-1, 16), c[m.astype(bool)])
        assert np.array_equal(f.reshape(-1, 16), c[~m.astype(bool)])


@pytest.mark.parametrize("N,g", [(1, 1), (2, 1), (1, 4), (2, 2), (2, 4), (4, 2), (1, 8), (8, 1), (2, 3)])
def test_expand_equals_unpartition_of_slices(N, g):
    chunks = 517
    rng = np.random.default_rng(7)
    for name, m in masks(chunks, 3):
        geo = O.geom(chunks, m, N, g)
        nat = rng.integers(0, 256, chunks * 16, dtype=np.uint8)
        t, f = O.partition(nat, m)
        tp = np.zeros(geo.slice_t * g * 16, np.uint8); tp[:t.size] = t
        fp = np.zeros(geo.slice_f * g * 16, np.uint8); fp[:f.size] = f
        ts = [tp[j * geo.slice_t * 16:(j + 1) * geo.slice_t * 16] for j in range(g)]
        fs = [fp[j * geo.slice_f * 16:(j + 1) * geo.slice_f * 16] for j in range(g)]
        out = np.zeros(chunks * 16, np.uint8)
        O.expand(geo, m, ts, fs, out, 0)
        assert np.array_equal(out, nat), name
        # FrozenOnly leaves trainable chunks untouched
        out2 = np.full(chunks * 16, 0xAB, np.uint8)
        O.expand(geo, m, ts, fs, out2, 2)
        keep = np.repeat(m.astype(bool), 16)
        assert np.all(out2[keep] == 0xAB) and np.array_equal(out2[~keep], nat[~keep])


def test_rs_slice_against_numpy():
    chunks, N, g = 300, 2, 4
    rng = np.random.default_rng(1)
    for name, m in masks(chunks, 5):
        geo = O.geom(chunks, m, N, g)
        grads = [O.f32_to_bf16(rng.standard_normal(chunks * 8).astype(np.float32)) for _ in range(g)]
        full = np.zeros(chunks * 8, np.float32)
        for x in grads:  # same order, fp32
            full = (full + O.bf16_to_f32(x)).astype(np.float32)
        tvec = full.reshape(chunks, 8)[m.astype(bool)].reshape(-1)
        for j in range(g):
            for n in range(N):
                own, wire = O.rs_slice(geo, m, 2, grads, j, n, 0.125, False)
                k0 = j * geo.slice_t
                lo = k0 + n * geo.shard_t
                hi = min(lo + geo.shard_t, geo.pt)
                if hi > lo:
                    assert np.array_equal(own[:(hi - lo) * 8], tvec[lo * 8:hi * 8]), name
                ownf, _ = O.rs_slice(geo, m, 2, grads, j, n, 0.125, True)
                if hi > lo:
                    assert np.array_equal(ownf[:(hi - lo) * 8], (tvec[lo * 8:hi * 8] * np.float32(0.125)))


def test_mics_replica_sum_against_numpy():
    """MiCS replica gradient sync (engine mics_grad_sync): rs_slice with no own
    shard puts the whole node-reduced slice on the wire; rs_finalize with
    node = -1 sums every node's wire contribution in node order, so all
    replicas produce identical bits."""
    chunks, N, g = 200, 3, 2
    rng = np.random.default_rng(4)
    m = np.ones(chunks, np.uint8)
    geo = O.geom(chunks, m, 1, g)  # MiCS: shards over the node's g GPUs only
    per_node = [[O.f32_to_bf16(rng.standard_normal(chunks * 8).astype(np.float32)) for _ in range(g)]
                for _ in range(N)]
    sh = geo.shard_t * 8
    for j in range(g):
        wires = []
        for n in range(N):
            own, wire = O.rs_slice(geo, m, 2, per_node[n], j, -1, 1.0 / (N * g), False)
            assert not own.any()  # nothing kept back in fp32
            acc = np.zeros(chunks * 8, np.float32)
            for x in per_node[n]:
                acc = (acc + O.bf16_to_f32(x)).astype(np.float32)
            assert np.array_equal(wire[:sh], O.f32_to_bf16(acc[j * sh:(j + 1) * sh]))
            wires.append(wire[:sh])
        rx = np.concatenate(wires)
        got = O.rs_finalize(np.zeros(sh, np.float32), rx, N, -1, 2, sh, 1.0 / (N * g))
        exp = np.zeros(sh, np.float32)
        for w in wires:
            exp = (exp + O.bf16_to_f32(w)).astype(np.float32)
        assert np.array_equal(got, (exp * np.float32(1.0 / (N * g))).astype(np.float32))


def test_adam_against_numpy():
    rng = np.random.default_rng(2)
    n = 1000
    w = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32); v = np.zeros(n, np.float32)
    p = np.zeros(n, np.uint16)
    g = rng.standard_normal(n).astype(np.float32)
    w0 = w.copy()
    O.adam(w, m, v, g, p, 1e-3, 0.9, 0.999, 1e-8, 0.01, 1)
    m_ref = 0.1 * g; v_ref = 0.001 * g * g
    upd = (m_ref / 0.1) / (np.sqrt(v_ref / 0.001) + 1e-8) + 0.01 * w0
    np.testing.assert_allclose(w, w0 - 1e-3 * upd, rtol=1e-6, atol=1e-7)
    assert np.array_equal(p, O.f32_to_bf16(w))


def test_bf16_rounding_matches_torch():
    import torch
    x = np.random.default_rng(3).standard_normal(10000).astype(np.float32) * 1e3
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.f32_to_bf16(x), ref)
    lib = O.lib()
    assert all(lib.fo_f32_to_bf16(float(v)) == r for v, r in zip(x[:200], ref[:200]))


def test_init_deterministic():
    a = O.init_natural(1000, 2, 0x5EED, 3, [(0, 500, 0, 0.02), (500, 600, 1, 1.0)])
    b = O.init_natural(1000, 2, 0x5EED, 3, [(0, 500, 0, 0.02), (500, 600, 1, 1.0)])
    assert np.array_equal(a, b)
    f = O.bf16_to_f32(a)
    assert np.all(np.abs(f[:500]) <= 0.0201) and np.all(f[500:600] == 1.0) and np.all(f[600:] == 0)
