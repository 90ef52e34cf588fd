"""verify rules hold on real programs and fire on mutated ones."""
import copy

import pytest

from paper_2602_06499_b200 import shardsim as S
from paper_2602_06499_b200 import verify as V


def lora_model():
    return S.ModelSpec([S.LayerSpec(0, 4096, 0.0)] + [S.LayerSpec(i, 4096, 0.25) for i in range(1, 4)], 2)


def programs(strategy, iters=4, model=None):
    model = model or lora_model()
    plan = S.StrategyPlan(strategy)
    st = S.init_param_states(model)
    out = []
    for it in range(1, iters + 1):
        p = S.build_iteration(plan, model, S.make_topology(2, 2), st, it)
        out.append(p)
        st = S.step_state(st, p)
        assert not V.check_dirty_iff_stale(st) or strategy == S.StrategyKind.Zero3
    return out, st


@pytest.mark.parametrize("kind", [S.StrategyKind.Fcdp, S.StrategyKind.FcdpComm])
def test_rules_hold(built, kind):
    progs, st = programs(kind)
    for p in progs:
        assert V.check_program(kind, p.events) == []
    if kind == S.StrategyKind.FcdpComm:
        assert V.check_frozen_gather_once([p.events for p in progs], [0, 1, 2, 3]) == []
    assert V.check_dirty_iff_stale(st) == []


def test_mutation_backward_ag_inter(built):
    progs, _ = programs(S.StrategyKind.Fcdp, 1)
    ev = copy.deepcopy(progs[0].events)
    bwd_h2d = next(e for e in ev if e.kind == S.EventKind.H2D)
    bwd_h2d.kind = S.EventKind.AgInter  # inject a backward inter-node gather
    v = V.check_program(S.StrategyKind.Fcdp, ev)
    assert [x.rule for x in v] == ["zero_bwd_ag_inter"]


def test_mutation_frozen_regather(built):
    progs, _ = programs(S.StrategyKind.FcdpComm, 3)
    evs = [copy.deepcopy(p.events) for p in progs]
    ag = next(e for e in evs[2] if e.kind == S.EventKind.AgInter)
    ag.param_set = S.ParamSet.All  # iteration 3 re-gathers a frozen portion
    v = V.check_frozen_gather_once(evs, [1, 2, 3])
    assert v and all(x.rule == "frozen_gather_once" for x in v)


def test_mutation_dirty_flag(built):
    _, st = programs(S.StrategyKind.FcdpComm, 2)
    st = copy.deepcopy(st)
    frozen = next(s for s in st if s.frozen)
    frozen.dirty = True
    assert [x.rule for x in V.check_dirty_iff_stale(st)] == ["dirty_iff_stale"]


def test_mutation_compute_without_gather(built):
    progs, _ = programs(S.StrategyKind.Zero3, 1)
    ev = copy.deepcopy(progs[0].events)
    c = next(e for e in ev if e.kind == S.EventKind.ComputeFwd and e.layer == 2)
    c.deps = [d for d in c.deps if ev[d].kind not in V.RECONSTRUCT]
    assert [x.rule for x in V.check_program(S.StrategyKind.Zero3, ev)] == ["compute_has_params"]


def test_bytes_conserved():
    assert V.check_bytes_conserved({"fwd": 10}, {"fwd": 10}) == []
    assert [x.rule for x in V.check_bytes_conserved({"fwd": 9}, {"fwd": 10})] == ["bytes_conserved"]
