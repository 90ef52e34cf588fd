"""Control plane parity: our shardsim vs the compiled reference.

* tests/golden/control_plane.txt.gz is the output of tests/cpp/golden_driver.cpp
  linked against the reference sources (/root/reference/proj/src/*.cpp, built
  by oracle/Makefile).  It covers serialize_program (schedule.cpp:389-416) for
  every strategy x topology x model x iteration 1-3, comm_volume
  (costmodel.cpp:21-98), memory_footprint / max_feasible_batch
  (strategy.cpp:74-137), iteration_time_estimate (costmodel.cpp:100-129),
  presets and error messages.
* The same driver linked against libfcdp.so through include/shardsim must
  reproduce it byte for byte (drop-in proof).
"""
import gzip
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden" / "control_plane.txt.gz"


def test_golden_driver_against_libfcdp(built, tmp_path):
    exe = tmp_path / "golden_ours"
    pkg = ROOT / "paper_2602_06499_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/golden_driver.cpp"),
                    f"-L{pkg}", "-lfcdp", f"-Wl,-rpath,{pkg}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True).stdout
    gold = gzip.decompress(GOLDEN.read_bytes())
    assert out == gold, "control plane diverges from the reference goldens"


@pytest.mark.skipif(not Path("/root/reference/proj/src").exists(), reason="reference sources absent")
def test_golden_file_pinned_by_reference():
    """The committed golden file is what the reference itself produces."""
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], check=True, capture_output=True)
    out = subprocess.run([str(ROOT / "oracle/_ref/golden_ref")], check=True, capture_output=True).stdout
    assert out == gzip.decompress(GOLDEN.read_bytes())


# ---- SPEC / SURVEY known-answer tests through the Python mirror -------------

def _gpt2_blocks():
    from paper_2602_06499_b200.shardsim import LayerSpec, ModelSpec
    return ModelSpec([LayerSpec(i, 50358272) for i in range(24)], 2)


def test_survey_byte_targets(built):
    from paper_2602_06499_b200 import shardsim as S
    m = _gpt2_blocks()
    topo = S.make_topology(2, 4)
    z3 = S.comm_volume(S.StrategyPlan(S.StrategyKind.Zero3), m, topo, 2)
    fc = S.comm_volume(S.StrategyPlan(S.StrategyKind.Fcdp), m, topo, 2)
    assert z3.fwd_ag_inter + z3.bwd_ag_inter == 2_417_197_056
    assert fc.fwd_ag_inter == 1_208_598_528 and fc.bwd_ag_inter == 0
    assert fc.h2d_total == 2_417_197_056 and fc.d2h_total == 2_417_197_056
    # Llama-7B + LoRA r=16
    lora = S.ModelSpec([S.LayerSpec(i, 202907648, 524288 / 202907648) for i in range(32)], 2)
    z3 = S.comm_volume(S.StrategyPlan(S.StrategyKind.Zero3), lora, topo, 2)
    fcc = S.comm_volume(S.StrategyPlan(S.StrategyKind.FcdpComm), lora, topo, 2)
    assert z3.fwd_ag_inter + z3.bwd_ag_inter == 12_986_089_472
    assert fcc.fwd_ag_inter == 16_777_216 and fcc.bwd_ag_inter == 0
    assert fcc.reduce_scatter_inter == 16_777_216
    assert 1 - fcc.fwd_ag_inter / (z3.fwd_ag_inter + z3.bwd_ag_inter) > 0.998


def test_spec_examples(built):
    from paper_2602_06499_b200 import shardsim as S
    # topology: calibration round trip
    topo = S.make_topology(2, 8, inter_preset="eth1g-measured")
    assert abs(S.transfer_time(16 * S.kGiB, S.LinkKind.InterNode, topo) - 67.66) < 1e-9
    assert S.transfer_time(0, S.LinkKind.HostGpu, topo) == 0.0
    # workload presets
    g30 = S.model_preset("gpt30b")
    assert g30.num_layers() == 40 and g30.total_params() == 30_000_000_000
    assert S.model_preset("gpt25b").num_layers() == 39
    with pytest.raises(S.ConfigError):
        S.model_preset("gpt99b")
    with pytest.raises(S.ConfigError):
        S.apply_lora_mask(g30, 0.0)
    # strategy footprint
    g10 = S.model_preset("gpt10b")
    fp = S.memory_footprint(S.StrategyPlan(S.StrategyKind.Fcdp), g10, S.make_topology(4, 8))
    assert fp.host_cache_bytes_per_node == 20_000_000_000
    z3 = S.memory_footprint(S.StrategyPlan(S.StrategyKind.Zero3), g10, S.make_topology(4, 8))
    assert z3.gpu_total_bytes() == fp.gpu_total_bytes()
    # schedule: FCDP iteration 1 -> L AgInter + L D2H fwd, 0 backward AgInter
    m = _gpt2_blocks()
    plan = S.StrategyPlan(S.StrategyKind.Fcdp)
    st = S.init_param_states(m)
    prog = S.build_iteration(plan, m, S.make_topology(2, 4), st, 1)
    ev = prog.events
    last_fwd = max(e.id for e in ev if e.kind == S.EventKind.ComputeFwd)
    assert sum(e.kind == S.EventKind.AgInter for e in ev) == 24
    assert sum(e.kind == S.EventKind.D2H for e in ev) == 24
    assert not any(e.kind == S.EventKind.AgInter and e.id > last_fwd for e in ev)
    # ZeRO-3: 2L AgInter
    p3 = S.build_iteration(S.StrategyPlan(S.StrategyKind.Zero3), m, S.make_topology(2, 4), st, 1)
    assert sum(e.kind == S.EventKind.AgInter for e in p3.events) == 48
    # step_state: after FcdpComm iteration 1, frozen portions are clean forever
    lora = S.ModelSpec([S.LayerSpec(i, 4096, 0.25) for i in range(3)], 2)
    pc = S.StrategyPlan(S.StrategyKind.FcdpComm)
    st = S.init_param_states(lora)
    for it in range(1, 5):
        prog = S.build_iteration(pc, lora, S.make_topology(2, 2), st, it)
        frozen_gathers = [e for e in prog.events if e.kind == S.EventKind.AgInter
                          and e.param_set in (S.ParamSet.All, S.ParamSet.FrozenOnly)]
        assert (len(frozen_gathers) == 3) == (it == 1)
        st = S.step_state(st, prog)
        assert all((not s.dirty) and s.host_cached_version == 0 for s in st if s.frozen)
    # protocol errors
    bad = S.init_param_states(lora)
    bad[0].dirty = False
    with pytest.raises(S.ProtocolError):
        S.build_iteration(pc, lora, S.make_topology(2, 2), bad, 1)


def test_serialize_matches_python_events(built):
    from paper_2602_06499_b200 import shardsim as S
    m = S.ModelSpec([S.LayerSpec(i, 789760) for i in range(2)], 4)
    prog = S.build_iteration(S.StrategyPlan(S.StrategyKind.Fcdp), m, S.make_topology(2, 1),
                             S.init_param_states(m), 1)
    text = S.serialize_program(prog).splitlines()
    assert text[0] == f"program iteration=1 strategy=fcdp events={len(prog.events)}"
    names = {0: "ag_inter", 1: "ag_intra", 2: "h2d", 3: "d2h", 4: "compute_fwd", 5: "compute_bwd",
             6: "reduce_scatter", 7: "optimizer_step", 8: "mask_dirty", 9: "broadcast"}
    for line, e in zip(text[1:], prog.events):
        f = line.split(" ")
        assert int(f[0]) == e.id and f[1] == names[int(e.kind)]
        assert f[4] == str(e.bytes_total)
        assert f[5] == "deps=" + ",".join(map(str, e.deps))


def test_control_plane_timer_reference_vs_ours(built):
    """BASELINE.md §3 "Timing 1": the same timing driver linked against the
    compiled reference and against libfcdp walks identical programs (events per
    step, comm_volume checksum)."""
    import json
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    ref, ours = root / "oracle" / "_ref" / "time_ref", root / "oracle" / "_ref" / "time_ours"
    if not ref.exists() or not ours.exists():
        pytest.skip("timing drivers not built (needs /root/reference)")
    args = ["fcdp-comm", "2", "4", "20", "2"] + [str(x) for x in (131072000, *([202907648] * 4), 131076096)]
    a = json.loads(subprocess.run([str(ref)] + args, capture_output=True, text=True, check=True).stdout)
    b = json.loads(subprocess.run([str(ours)] + args, capture_output=True, text=True, check=True).stdout)
    assert a["events_per_step"] == b["events_per_step"] and a["check"] == b["check"]
