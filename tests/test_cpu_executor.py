"""The C++ CPU executor (oracle/cpu_executor.cpp, the timed CPU reference of the
path) against the Python engine oracle (tests/engine_oracle.py): the same
reference-built programs, every value bit-exact - shards, host caches, reduced
gradients, AdamW masters - and the byte counters.  It is the second,
independent CPU restatement of the data plane, and the one bench.py times.
Also: FCDP vs ZeRO-3 inter-group bytes == the reference comm_volume, and the
SPEC.md:357 freshness rule (a stale host-cache reload is a ProtocolError)."""
import numpy as np
import pytest

from tests.engine_oracle import Sim
from tests.test_engine_gpu import _masks

cx = pytest.importorskip("oracle.cpu_executor")
if not cx.available():
    try:
        cx.lib()
    except Exception:
        pytest.skip("cpu executor not built (needs /root/reference)", allow_module_level=True)


def _cfg(N, g, strategy, eb, kind, chunks=(1000, 1537, 777), tau=0.0, capacity=0, iters=3):
    V = 16 // eb
    return {"N": N, "g": g, "world": N * g, "strategy": strategy, "eb": eb, "iters": iters, "seed": 0x5EED,
            "params": [c * V for c in chunks], "masks": _masks(chunks, kind), "tau": tau, "capacity": capacity}


def _executor(cfg, threads=4, **kw):
    return cx.CpuExecutor(cfg["params"], [np.array(m, np.uint8) for m in cfg["masks"]], nodes=cfg["N"],
                          local=cfg["g"], strategy=cfg["strategy"], elem_bytes=cfg["eb"], tau=cfg["tau"],
                          gpu_capacity_bytes=cfg["capacity"], seed=cfg["seed"], threads=threads, **kw)


def run_and_check(cfg, threads=4):
    sim = Sim(cfg)
    S = sim.S
    states = S.init_param_states(sim.model)
    ex = _executor(cfg, threads)
    V = sim.V
    try:
        for it in range(1, cfg["iters"] + 1):
            exp, states, prog = sim.iteration(it, states)
            st = ex.step()
            assert st["events"] == len(prog.events)
            for r in range(sim.G):
                e = exp[r]
                s = sim.shard_index(r)
                j = r % sim.g
                for l in range(sim.L):
                    geo = sim.geo[l]
                    ht, hf = e["host"][l]
                    if ht is not None:
                        n = sim._real_slice(l, False, j) * 16
                        assert np.array_equal(ex.read(r, l, "host_t", n), ht[:n]), (it, r, l)
                    if hf is not None:
                        n = sim._real_slice(l, True, j) * 16
                        assert np.array_equal(ex.read(r, l, "host_f", n), hf[:n]), (it, r, l)
                    rt = sim._real(l, False, s)
                    if rt:
                        got = ex.read(r, l, "grad", rt * V * 4).view(np.uint32)
                        assert np.array_equal(got, e["grad"][l][:rt * V].view(np.uint32)), ("grad", it, r, l)
                        got = ex.read(r, l, "master", rt * V * 4).view(np.uint32)
                        assert np.array_equal(got, e["master"][l][:rt * V].view(np.uint32)), ("master", it, r, l)
                        assert np.array_equal(ex.read(r, l, "shard_t", rt * 16), e["shard_t"][l][:rt * 16])
                    rf = sim._real(l, True, s)
                    if rf:
                        assert np.array_equal(ex.read(r, l, "shard_f", rf * 16), e["shard_f"][l][:rf * 16])
            for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs", "cache_h2d", "cache_d2h", "nvlink_rx",
                      "nic_tx_grad_sync"):
                assert st[k] * sim.N == sum(exp[r]["counters"][k] for r in range(sim.G)), (k, it)
    finally:
        ex.close()


CASES = [(1, 1, "fcdp", 2, "dense"), (1, 1, "fcdp-comm", 4, "random"), (2, 1, "zero3", 2, "dense"),
         (2, 1, "fcdp", 2, "dense"), (2, 1, "fcdp-comm", 2, "lora"), (1, 2, "fcdp", 2, "dense"),
         (2, 2, "fcdp", 2, "lora"), (2, 2, "zero3", 4, "random"), (2, 2, "fcdp-comm", 2, "random"),
         (2, 2, "zeropp", 2, "dense"), (2, 2, "mics", 2, "lora"), (4, 1, "fcdp-comm", 2, "lora"),
         (2, 4, "fcdp", 2, "dense"), (4, 2, "fcdp-comm", 2, "lora")]


@pytest.mark.parametrize("N,g,strategy,eb,kind", CASES)
def test_cpu_executor_matches_engine_oracle(N, g, strategy, eb, kind):
    run_and_check(_cfg(N, g, strategy, eb, kind))


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_cpu_executor_thread_split_is_exact(threads):
    """Work split inside a rank (kBlock chunks per item) never changes a bit."""
    run_and_check(_cfg(2, 1, "fcdp-comm", 2, "random", chunks=(20000, 9001, 4099)), threads=threads)


@pytest.mark.parametrize("N,g", [(1, 1), (2, 2)])
def test_cpu_executor_tau_retention(N, g):
    run_and_check(_cfg(N, g, "fcdp-comm", 2, "lora", tau=1.0))


def test_cpu_executor_bytes_equal_comm_volume():
    """Divisible sizes at 2x2: per-node NIC bytes == the reference comm_volume,
    FCDP's backward AG bytes are 0, and ZeRO-3 moves 1.5x FCDP's (fwd+bwd+RS)."""
    from paper_2602_06499_b200 import shardsim as S
    G = 4
    res = {}
    for strategy in ("zero3", "fcdp"):
        cfg = _cfg(2, 2, strategy, 2, "dense", chunks=(64 * G, 96 * G, 32 * G))
        sim = Sim(cfg)
        ex = _executor(cfg)
        for it in range(1, 4):
            st = ex.step()
            vol = S.comm_volume(sim.plan, sim.model, sim.topo, it)
            assert st["nic_tx_fwd_ag"] == vol.fwd_ag_inter
            assert st["nic_tx_bwd_ag"] == vol.bwd_ag_inter
            assert st["nic_tx_rs"] == vol.reduce_scatter_inter
            if strategy == "fcdp":
                assert st["cache_h2d"] == vol.h2d_total and st["cache_d2h"] == vol.d2h_total
        res[strategy] = st
        ex.close()
    assert res["fcdp"]["nic_tx_bwd_ag"] == 0 and res["zero3"]["nic_tx_bwd_ag"] > 0
    z = sum(res["zero3"][k] for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs"))
    f = sum(res["fcdp"][k] for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs"))
    assert 2 * z == 3 * f


def test_cpu_executor_stale_reload_is_protocol_error():
    """SPEC.md:357 freshness (mutation): iteration 2 loses rank 1's FCDP-Cache
    store of layer 1, so its host copy is one version old when the backward
    reloads it - a ProtocolError (-2), with every rank thread still coming home."""
    cfg = _cfg(2, 1, "fcdp", 2, "dense")
    ex = _executor(cfg)
    ex.step()
    ex.drop_d2h(1, 1)
    with pytest.raises(cx.ExecError) as ei:
        ex.step()
    assert ei.value.code == -2 and "freshness" in str(ei.value) and "stale host cache" in str(ei.value)
    ex.close()


def test_cpu_executor_compute_callback_sees_gathered_layers():
    """The compute callback receives the gathered natural layer (bit-exact vs the
    oracle's natural parameters) and returns the gradient in the natural buffer."""
    import ctypes as C
    from oracle import oracle as O
    cfg = _cfg(2, 2, "fcdp-comm", 2, "lora", iters=2)
    sim = Sim(cfg)
    states = sim.S.init_param_states(sim.model)
    ex = _executor(cfg)
    seen = []

    def cb(user, kind, rank, layer, w, g):
        n = cfg["params"][layer] * 2
        W = np.frombuffer(C.string_at(w, n), np.uint16)
        seen.append((kind, rank, layer, W.copy()))
        if g:
            gr = O.f32_to_bf16(O.bf16_to_f32(W) * np.float32((1 + rank) / 8.0))
            C.memmove(g, gr.ctypes.data, n)
        return 0
    ex.set_compute(cb)
    for it in range(1, 3):
        exp, states, prog = sim.iteration(it, states)
        seen.clear()
        ex.step()
        for r in range(sim.G):
            mine = [(k, l, W) for k, rr, l, W in seen if rr == r]
            assert len(mine) == len(exp[r]["captures"])
            for (k1, l1, w1), (k2, l2, w2) in zip(mine, exp[r]["captures"]):
                assert (k1, l1) == (k2, l2) and np.array_equal(w1.view(np.uint8), w2.view(np.uint8))
            l = 1
            rt = sim._real(l, False, sim.shard_index(r))
            if rt:
                got = ex.read(r, l, "master", rt * 8 * 4).view(np.uint32)
                assert np.array_equal(got, exp[r]["master"][l][:rt * 8].view(np.uint32))
    ex.close()
