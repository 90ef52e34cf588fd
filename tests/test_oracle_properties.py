"""Property tests of the CPU oracle (hypothesis): the layout geometry and the
partition / expand pair over random sizes, masks and node x GPU shapes.  These
pin the checker itself before it is used to judge the GPU path."""
import numpy as np
import pytest

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402

from oracle import oracle as O  # noqa: E402

shapes = st.sampled_from([(1, 1), (2, 1), (1, 2), (2, 2), (1, 4), (4, 1), (2, 4), (4, 2), (1, 8), (8, 1), (3, 1),
                          (1, 3), (2, 3)])


@settings(max_examples=60, deadline=None)
@given(chunks=st.integers(1, 700), density=st.floats(0.0, 1.0), shape=shapes, seed=st.integers(0, 2**31 - 1))
def test_geometry_covers_each_portion_exactly_once(chunks, density, shape, seed):
    N, g = shape
    m = (np.random.default_rng(seed).random(chunks) < density).astype(np.uint8)
    geo = O.geom(chunks, m, N, g)
    G = N * g
    assert geo.pt == int(m.sum()) and geo.pf == chunks - geo.pt
    for per, total, sl in ((geo.shard_t, geo.pt, geo.slice_t), (geo.shard_f, geo.pf, geo.slice_f)):
        assert per * G >= total and (per - 1) * G < max(total, 1)  # ceil split, padding < G chunks
        assert sl == per * N                                      # slice j = shards j*N .. j*N+N-1


@settings(max_examples=40, deadline=None)
@given(chunks=st.integers(1, 400), density=st.floats(0.0, 1.0), shape=shapes, seed=st.integers(0, 2**31 - 1),
       pset=st.sampled_from([0, 1, 2]))
def test_expand_inverts_partition(chunks, density, shape, seed, pset):
    N, g = shape
    rng = np.random.default_rng(seed)
    m = (rng.random(chunks) < density).astype(np.uint8)
    nat = rng.integers(0, 256, chunks * 16, dtype=np.uint8)
    geo = O.geom(chunks, m, N, g)
    t, f = O.partition(nat, m)
    tp = np.zeros(max(geo.slice_t * g, 1) * 16, np.uint8); tp[:t.size] = t
    fp = np.zeros(max(geo.slice_f * g, 1) * 16, np.uint8); fp[:f.size] = f
    ts = [tp[j * geo.slice_t * 16:(j + 1) * geo.slice_t * 16] for j in range(g)]
    fs = [fp[j * geo.slice_f * 16:(j + 1) * geo.slice_f * 16] for j in range(g)]
    out = np.full(chunks * 16, 0x5A, np.uint8)
    O.expand(geo, m, ts, fs, out, pset)
    sel = np.repeat(m.astype(bool), 16)
    want = {0: np.ones_like(sel), 1: sel, 2: ~sel}[pset]
    assert np.array_equal(out[want], nat[want])
    assert np.all(out[~want] == 0x5A)
