"""The engine-parity oracle (tests/engine_oracle.py) checked on CPU against
the compiled-reference-pinned byte oracle: over 3 iterations, the NIC and host
bytes the CPU re-derivation expects per node equal shardsim comm_volume exactly
(the same identity tests/test_engine_gpu.py then demands of the GPUs)."""
import numpy as np
import pytest

from tests.engine_oracle import Sim


def _masks(chunks, kind, G=1, seed=0):
    """Dense, or LoRA-like: a few trainable runs whose total is a multiple of G
    (so no shard is padded and the closed form applies), one frozen-only layer."""
    rng = np.random.default_rng(seed)
    out = []
    for i, c in enumerate(chunks):
        if kind == "dense":
            m = np.ones(c, np.uint8)
        else:
            m = np.zeros(c, np.uint8)
            if i != 1:
                for r in range(3):  # disjoint thirds, one run of G * k chunks in each
                    lo = r * (c // 3)
                    k = int(rng.integers(1, 3)) * G
                    a = lo + int(rng.integers(0, c // 3 - k))
                    m[a:a + k] = 1
        out.append(m.tolist())
    return out


@pytest.mark.parametrize("N,g", [(2, 1), (2, 2), (4, 1), (2, 4), (1, 2)])
@pytest.mark.parametrize("strategy,kind", [("zero3", "dense"), ("fcdp", "dense"), ("fcdp", "lora"),
                                           ("fcdp-comm", "lora"), ("zeropp", "dense")])
def test_sim_bytes_equal_comm_volume(built, N, g, strategy, kind):
    G = N * g
    chunks = (64 * G, 96 * G, 32 * G)
    cfg = {"N": N, "g": g, "world": G, "strategy": strategy, "eb": 2, "iters": 3, "seed": 0x5EED,
           "params": [c * 8 for c in chunks], "masks": _masks(chunks, kind, G)}
    sim = Sim(cfg)
    S = sim.S
    states = S.init_param_states(sim.model)
    for it in (1, 2, 3):
        exp, states, _ = sim.iteration(it, states)
        vol = S.comm_volume(sim.plan, sim.model, sim.topo, it)
        for n in range(N):
            node = [exp[n * g + j]["counters"] for j in range(g)]
            assert sum(c["nic_tx_fwd_ag"] for c in node) == vol.fwd_ag_inter
            assert sum(c["nic_tx_bwd_ag"] for c in node) == vol.bwd_ag_inter
            assert sum(c["nic_tx_rs"] for c in node) == vol.reduce_scatter_inter
            assert sum(c["cache_h2d"] for c in node) == vol.h2d_total
            assert sum(c["cache_d2h"] for c in node) == vol.d2h_total


def test_sim_mics_replicas_identical(built):
    """MiCS (subgroup = g): every node's replica of every shard stays bit-identical."""
    N, g = 2, 2
    chunks = (1000, 1537, 777)
    cfg = {"N": N, "g": g, "world": N * g, "strategy": "mics", "eb": 2, "iters": 3, "seed": 0x5EED,
           "params": [c * 8 for c in chunks], "masks": _masks(chunks, "dense")}
    sim = Sim(cfg)
    states = sim.S.init_param_states(sim.model)
    for it in (1, 2, 3):
        _, states, _ = sim.iteration(it, states)
        for r in range(g, N * g):
            for l in range(sim.L):
                assert np.array_equal(sim.shard_t[r][l], sim.shard_t[r % g][l])
                assert np.array_equal(sim.master[r][l], sim.master[r % g][l])
