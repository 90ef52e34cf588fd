"""Engine parity on the B200: gathered layers, FCDP-Cache contents, gradient
reduce-scatter, AdamW updates and NIC byte counters vs the CPU oracle.

Each case launches one process per rank (tests/engine_worker.py), runs a few
iterations of a shardsim program, and re-derives every value on the CPU
(tests/engine_oracle.py).  Gathered / cached parameters and the fp32
reduction + optimizer arithmetic are compared BIT-EXACT.
"""
import json
import os
import pickle
import subprocess
import sys
import uuid
from pathlib import Path

import numpy as np
import pytest

from tests.engine_oracle import Sim

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _need_gpu():
    # Ranks are placed round-robin on the visible GPUs (rank % device_count,
    # engine_worker.py), so an N x g job runs on any box with >= 1 GPU: CUDA IPC,
    # the shared control block and stream memory ops all work between processes
    # that share a device.  Same-device "NVLink" pulls then read local HBM.
    if _ngpu() < 1:
        pytest.skip("needs a GPU")


def _masks(chunks_list, kind, seed=0):
    rng = np.random.default_rng(seed)
    out = []
    for i, c in enumerate(chunks_list):
        if kind == "dense":
            m = np.ones(c, np.uint8)
        elif kind == "lora":
            m = np.zeros(c, np.uint8)
            for _ in range(3):
                a = int(rng.integers(0, c - 8))
                m[a:a + int(rng.integers(2, 9))] = 1
            if i == 1:
                m[:] = 0  # a frozen-only layer (reference workload.cpp:52-53)
        else:
            m = (rng.random(c) < 0.3).astype(np.uint8)
        out.append(m.tolist())
    return out


def run_job(tmp_path, N, g, strategy, eb=2, kind="dense", iters=3, chunks=(1000, 1537, 777), pacing=False,
            use_ce=False, tau=0.0, capacity=0, stepwise=False, trace=False, mutate=None, nic_log=False,
            inter="ib100-rdma-measured"):
    world = N * g
    V = 16 // eb
    cfg = {"N": N, "g": g, "world": world, "inter": inter, "strategy": strategy, "eb": eb, "iters": iters, "seed": 0x5EED,
           "params": [c * V for c in chunks], "masks": _masks(chunks, kind), "shm": f"fcdp_test_{uuid.uuid4().hex[:12]}",
           "out": str(tmp_path), "pacing": pacing, "use_ce": use_ce, "tau": tau, "capacity": capacity,
           "stepwise": stepwise, "trace": trace, "mutate": mutate, "nic_log": nic_log}
    procs = []
    for r in range(world):
        c = dict(cfg, rank=r)
        procs.append(subprocess.Popen([sys.executable, str(ROOT / "tests" / "engine_worker.py"), json.dumps(c)],
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{out[-4000:]}"
    dumps = []
    for r in range(world):
        with open(tmp_path / f"rank{r}.pkl", "rb") as f:
            dumps.append(pickle.load(f))
    return cfg, dumps


def check_job(cfg, dumps):
    sim = Sim(cfg)
    S = sim.S
    states = S.init_param_states(sim.model)
    V = sim.V
    for it in range(1, cfg["iters"] + 1):
        exp, states, prog = sim.iteration(it, states)
        for r in range(sim.G):
            got = dumps[r][it - 1]
            e = exp[r]
            # gathered layers at every compute event, bit-exact
            assert len(got["captures"]) == len(e["captures"]), (it, r)
            for (k1, l1, w1), (k2, l2, w2) in zip(got["captures"], e["captures"]):
                assert (k1, l1) == (k2, l2)
                assert np.array_equal(w1.view(np.uint8), w2.view(np.uint8)), f"gathered layer {l1} kind {k1} it {it} rank {r}"
            j = r % sim.g
            s = sim.shard_index(r)
            for l in range(sim.L):
                geo = sim.geo[l]
                ht, hf = e["host"][l]
                if ht is not None:
                    n = sim._real_slice(l, False, j) * 16
                    assert np.array_equal(got["host"][l][0][:n], ht[:n]), f"host cache t layer {l} it {it} rank {r}"
                if hf is not None:
                    n = sim._real_slice(l, True, j) * 16
                    assert np.array_equal(got["host"][l][1][:n], hf[:n]), f"host cache f layer {l} it {it} rank {r}"
                rt = sim._real(l, False, s)
                if rt:
                    assert np.array_equal(got["grad"][l][:rt * V].view(np.uint32),
                                          e["grad"][l][:rt * V].view(np.uint32)), f"grad layer {l} it {it} rank {r}"
                    assert np.array_equal(got["master"][l][:rt * V].view(np.uint32),
                                          e["master"][l][:rt * V].view(np.uint32)), f"master layer {l} it {it} rank {r}"
                    assert np.array_equal(got["shard_t"][l][:rt * 16], e["shard_t"][l][:rt * 16]), f"param layer {l}"
                rf = sim._real(l, True, s)
                if rf:
                    assert np.array_equal(got["shard_f"][l][:rf * 16], e["shard_f"][l][:rf * 16])
            for k, v in e["counters"].items():
                assert got["counters"][k] == v, (k, got["counters"][k], v, it, r)
        # per node NIC totals vs the reference closed form, when shards divide evenly
        vol = S.comm_volume(sim.plan, sim.model, sim.topo, it)
        if all(sim._real(l, False, 0) == sim.geo[l].shard_t and sim.geo[l].pt % sim.G == 0 and
               sim.geo[l].pf % sim.G == 0 for l in range(sim.L)):
            for n in range(sim.N):
                node = [dumps[n * sim.g + j][it - 1]["counters"] for j in range(sim.g)]
                assert sum(c["nic_tx_fwd_ag"] for c in node) == vol.fwd_ag_inter
                assert sum(c["nic_tx_bwd_ag"] for c in node) == vol.bwd_ag_inter
                assert sum(c["nic_tx_rs"] for c in node) == vol.reduce_scatter_inter
                if sim.plan.tau == 0:
                    assert sum(c["cache_h2d"] for c in node) == vol.h2d_total
                    assert sum(c["cache_d2h"] for c in node) == vol.d2h_total


CASES_1 = [(1, 1, "zeropp", 2, "dense"), (1, 1, "zero3", 2, "dense"), (1, 1, "fcdp", 2, "dense"), (1, 1, "fcdp-comm", 2, "lora"),
           (1, 1, "fcdp-comm", 4, "random"), (1, 1, "fcdp", 4, "lora")]
CASES_2 = [(2, 1, "zero3", 2, "dense"), (2, 1, "fcdp", 2, "dense"), (2, 1, "fcdp-comm", 2, "lora"),
           (1, 2, "fcdp", 2, "dense"), (1, 2, "fcdp-comm", 2, "random"), (2, 1, "fcdp-comm", 4, "random"),
           (1, 2, "zeropp", 2, "lora"), (2, 1, "mics", 2, "dense"), (1, 2, "mics", 4, "random")]
CASES_4 = [(2, 2, "zeropp", 2, "dense"), (2, 2, "zero3", 2, "dense"), (2, 2, "fcdp", 2, "dense"), (2, 2, "fcdp-comm", 2, "lora"),
           (4, 1, "fcdp-comm", 2, "random"), (1, 4, "fcdp", 4, "lora"), (2, 2, "mics", 2, "lora"),
           (4, 1, "mics", 4, "dense")]
# 8 ranks: the g = 8 intra-node paths and the 4-node NIC fan-in (emulated 2x4, 4x2, 1x8)
CASES_8 = [(2, 4, "fcdp", 2, "dense"), (4, 2, "fcdp-comm", 2, "lora"), (1, 8, "fcdp", 4, "random")]


@pytest.mark.parametrize("N,g,strategy,eb,kind", CASES_1 + CASES_2 + CASES_4 + CASES_8)
def test_engine_parity(tmp_path, built, N, g, strategy, eb, kind):
    _need_gpu()
    cfg, dumps = run_job(tmp_path, N, g, strategy, eb, kind)
    check_job(cfg, dumps)


def test_engine_even_shards_match_comm_volume(tmp_path, built):
    """Divisible sizes: per-node NIC counters equal comm_volume exactly."""
    _need_gpu()
    N, g = 2, 2
    G = N * g
    cfg, dumps = run_job(tmp_path, N, g, "fcdp-comm", 2, "lora", chunks=(64 * G, 96 * G, 32 * G))
    check_job(cfg, dumps)


@pytest.mark.parametrize("N,g,strategy", [(2, 2, "zero3"), (2, 2, "fcdp"), (4, 1, "fcdp-comm")])
def test_engine_nic_wire_log(tmp_path, built, N, g, strategy):
    """NIC bandwidth profile (Fig. 10) from the paced emulator's wire
    log: per rank, the logged bytes of each kind equal the NIC counters; the
    payloads of one node never overlap on its wire (one NIC per node,
    topology.hpp:23-25) and each occupies bytes / B_nic of it; FCDP puts no
    backward all-gather on the wire, ZeRO-3 does."""
    _need_gpu()
    cfg, dumps = run_job(tmp_path, N, g, strategy, 2, "lora" if strategy == "fcdp-comm" else "dense",
                         pacing=True, nic_log=True, inter="eth10g-measured")
    check_job(cfg, dumps)
    from paper_2602_06499_b200 import shardsim as S
    bw = S.make_topology(N, g, inter_preset="eth10g-measured").inter_node.bandwidth_bytes_per_s
    kinds = {0: "nic_tx_fwd_ag", 1: "nic_tx_bwd_ag", 2: "nic_tx_rs", 15: "nic_tx_grad_sync"}
    for it in range(cfg["iters"]):
        bwd_ag = 0
        for n in range(N):
            recs = np.concatenate([dumps[n * g + j][it]["nic_log"] for j in range(g)])
            for j in range(g):
                d = dumps[n * g + j][it]
                log = d["nic_log"]
                assert set(np.unique(log["kind"]).tolist()) <= set(kinds)
                for k, name in kinds.items():
                    assert int(log["bytes"][log["kind"] == k].sum()) == d["counters"][name], (n, j, name)
            recs = np.sort(recs, order="start_ns")
            dur = (recs["end_ns"] - recs["start_ns"]).astype(np.float64)
            assert np.all(np.abs(dur - recs["bytes"] / bw * 1e9) <= 1.0 + 1e-6 * dur)
            assert np.all(recs["start_ns"][1:] >= recs["end_ns"][:-1]), "two payloads overlap on one node's NIC"
            bwd_ag += int(recs["bytes"][recs["kind"] == 1].sum())
        if strategy == "zero3":
            assert bwd_ag > 0
        else:
            assert bwd_ag == 0


@pytest.mark.parametrize("N,g,strategy,kind", [(1, 1, "fcdp", "dense"), (1, 1, "fcdp-comm", "lora"),
                                                (2, 1, "fcdp-comm", "lora"), (2, 2, "fcdp", "lora"),
                                                (2, 2, "fcdp-comm", "random")])
def test_engine_tau_retention(tmp_path, built, N, g, strategy, kind):
    """tau = 1, unlimited capacity: every layer retained, no backward reload
    (FCDP-Cache adaptive GPU caching; schedule.cpp:196-223)."""
    _need_gpu()
    cfg, dumps = run_job(tmp_path, N, g, strategy, 2, kind, tau=1.0)
    check_job(cfg, dumps)
    for d in dumps[0]:
        assert all(f & 1 for f in d["retained"])
    if strategy == "fcdp-comm":
        # from iteration 2 on, every frozen reload is satisfied by the resident buffer
        assert all(d["counters"]["resident_hits"] > 0 for d in dumps[0][1:])
        assert all(d["counters"]["cache_h2d"] == 0 for d in dumps[0][1:])


def test_engine_tau_partial_capacity(tmp_path, built):
    """A capacity that admits only some layers: mixed retained / host-cache layers."""
    cfg, dumps = run_job(tmp_path, 1, 1, "fcdp", 2, "dense", tau=0.5, capacity=900_000)  # retains the last layer only
    check_job(cfg, dumps)
    flags = dumps[0][-1]["retained"]
    assert any(f & 1 for f in flags) and not all(f & 1 for f in flags), flags


@pytest.mark.parametrize("N,g,strategy,kind", [(1, 1, "fcdp-comm", "lora"), (2, 1, "fcdp", "random")])
def test_engine_stepwise_executor(tmp_path, built, N, g, strategy, kind):
    """fcdp_engine_begin / exec (one event at a time, id order) / end gives the
    same bit-exact results as fcdp_engine_run (the caller is an
    executor walking EventProgram.events)."""
    _need_gpu()
    cfg, dumps = run_job(tmp_path, N, g, strategy, 2, kind, stepwise=True)
    check_job(cfg, dumps)


_ORDER_SCRIPT = r"""
import sys, uuid
sys.path.insert(0, sys.argv[1])
from paper_2602_06499_b200 import shardsim as S
from paper_2602_06499_b200.engine import Engine, _States
from paper_2602_06499_b200._capi import lib
PROTOCOL = -2  # FCDP_ERR_PROTOCOL
model = S.ModelSpec([S.LayerSpec(i, 8 * 64, 1.0) for i in range(3)], 2)
topo = S.make_topology(1, 1)
plan = S.StrategyPlan(S.StrategyKind.Fcdp)
eng = Engine(model, topo, plan, rank=0, world_size=1, device=0, shm_name=f"fcdp_order_{uuid.uuid4().hex[:10]}",
             timeout_s=60.0)
eng.init_params(1, [])
states = S.init_param_states(model)
prog = S.build_iteration(plan, model, topo, states, 1)
assert lib().fcdp_engine_exec(eng._h, 0) == PROTOCOL        # exec outside begin/end
assert lib().fcdp_engine_begin(eng._h, prog.ptr) == 0
assert lib().fcdp_engine_exec(eng._h, 1) == PROTOCOL        # id 0 must come first
assert lib().fcdp_engine_begin(eng._h, prog.ptr) == PROTOCOL  # a program is already in progress
st = _States.from_list(states)
assert lib().fcdp_engine_end(eng._h, st.ptr) == PROTOCOL     # end before every event ran
for e in prog.events:
    assert lib().fcdp_engine_exec(eng._h, e.id) == 0
assert lib().fcdp_engine_exec(eng._h, len(prog.events)) == PROTOCOL  # past the end
assert lib().fcdp_engine_end(eng._h, st.ptr) == 0
eng.sync()
assert all(p.version == 1 and p.host_cached_version == 0 for p in st.to_list())  # step_state applied
print("order-ok")
"""


def test_engine_exec_order_enforced(tmp_path, built):
    """fcdp_engine_exec rejects out-of-order / repeated / past-the-end ids and a
    second begin with FCDP_ERR_PROTOCOL (the stepwise executor contract)."""
    if _ngpu() < 1:
        pytest.skip("needs a GPU")
    r = subprocess.run([sys.executable, "-c", _ORDER_SCRIPT, str(ROOT)], capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "order-ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- mutations
# SPEC.md:389-409 mutation harness applied to EXECUTED programs: each mutation
# must be rejected by the engine on the GPU with the error class its rule
# names, every rank must come home (abort flag, no hang), and the engine must
# refuse further programs (failure latch).

def _errors(tmp_path, world):
    return [pickle.load(open(tmp_path / f"rank{r}.pkl", "rb"))["errors"] for r in range(world)]


@pytest.mark.parametrize("N,g,strategy,kind", [(2, 1, "fcdp", "dense"), (2, 2, "fcdp-comm", "lora")])
def test_engine_rejects_stale_host_cache_reload(tmp_path, built, N, g, strategy, kind):
    """Iteration 2 loses layer 0's FCDP-Cache store (its D2H is dropped from the
    executed program): the backward reload of layer 0 would read the version-0
    host copy after AdamW moved the shard to version 1 -> FCDP_ERR_PROTOCOL
    ("freshness"; Algorithm 1 line 10)."""
    _need_gpu()
    run_job(tmp_path, N, g, strategy, 2, kind, iters=2, mutate={"it": 2, "kind": "drop_d2h", "layer": 0})
    for errs in _errors(tmp_path, N * g):
        assert errs and errs[0][0] == "ProtocolError" and "stale host cache" in errs[0][2], errs
        assert errs[1][0] == "ProtocolError" and "earlier program failed" in errs[1][2], errs


def test_engine_rejects_backward_ag_inter(tmp_path, built):
    """A backward AgInter injected into an FCDP program (layer 1's reload + intra
    gather replaced by an inter-node gather) -> FCDP_ERR_PROTOCOL
    (zero_bwd_ag_inter)."""
    _need_gpu()
    run_job(tmp_path, 2, 1, "fcdp", 2, "dense", iters=1, mutate={"it": 1, "kind": "bwd_ag_inter", "layer": 1})
    for errs in _errors(tmp_path, 2):
        assert errs and errs[0][0] == "ProtocolError" and "zero_bwd_ag_inter" in errs[0][2], errs


def test_engine_rejects_divergent_programs(tmp_path, built):
    """Rank 1 builds its program with another GPU capacity, so tau retention (and
    the cross-rank sequence numbers) differ: begin() compares program hashes
    across ranks and both ranks answer FCDP_ERR_CONFIG instead of reading a
    peer's slot of another layer."""
    _need_gpu()
    run_job(tmp_path, 2, 1, "fcdp", 2, "dense", iters=1, tau=0.5,
            mutate={"it": 1, "kind": "capacity_mismatch", "capacity": 300_000})
    for errs in _errors(tmp_path, 2):
        assert errs and errs[0][0] == "ConfigError" and "different programs" in errs[0][2], errs


# ------------------------------------------------------- executed-trace verify
@pytest.mark.parametrize("N,g,strategy,kind", [(2, 1, "fcdp", "dense"), (2, 2, "fcdp-comm", "lora"),
                                                (2, 2, "zero3", "dense")])
def test_engine_executed_trace_verifies(tmp_path, built, N, g, strategy, kind):
    """verify.py over what the GPUs EXECUTED (fcdp_engine_trace + counters):
    every event started after its dependencies finished on the device, FCDP
    executed 0 backward inter-node gathers, and the per-node NIC bytes equal
    the reference comm_volume."""
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200 import verify as Vf
    _need_gpu()
    G = N * g
    cfg, dumps = run_job(tmp_path, N, g, strategy, 2, kind, trace=True, chunks=(64 * G, 96 * G, 32 * G))
    check_job(cfg, dumps)
    for r in range(G):
        for d in dumps[r]:
            tr = d["trace"]
            evs = [S.Event(i, S.EventKind(k), l, S.ParamSet.All, 0, deps) for i, k, l, deps, _, _ in tr]
            begin = [b for *_, b, _ in tr]
            end = [e for *_, e in tr]
            assert all(e >= b for b, e in zip(begin, end))
            assert Vf.check_trace_respects_deps(evs, begin, end) == []
            assert Vf.check_zero_bwd_ag_inter(S.StrategyKind.from_string(strategy), evs) == []
            if strategy != "zero3":
                assert d["counters"]["ag_inter_events_bwd"] == 0
                assert d["counters"]["nic_tx_bwd_ag"] == 0
