"""Protocol invariant checker over executed programs ("verify").

The reference specifies these rules but ships no checker.  Here they run over
the event programs the B200 engine executed plus its measured byte counters:

    zero_bwd_ag_inter   no AgInter between the last ComputeFwd and the end of
                        the program for fcdp / fcdp-comm / zeropp
    frozen_gather_once  over K >= 2 iterations of fcdp-comm every frozen portion
                        is inter-gathered exactly once (iteration 1)
    dirty_iff_stale     dirty <=> host_cached_version != version (schedule.hpp:43-50)
    compute_has_params  every ComputeFwd/Bwd of a layer transitively depends on
                        an event that reconstructs it, unless the layer was
                        retained (freshness)
    bytes_conserved     per-node measured NIC bytes == comm_volume
    trace_respects_deps over an EXECUTED trace (fcdp_engine_trace): no event's
                        stream reached it before every dependency had finished
                        on the device (the DAG edges were honoured at run time)

check_* functions return a list of Violation(rule, event_id, detail); an
empty list means the rule holds.  tests/test_verify.py mutates programs to
show every rule fires on exactly the violation class it names.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence

from .shardsim import Event, EventKind, ParamSet, ParamState, StrategyKind


@dataclass
class Violation:
    rule: str
    event_id: Optional[int]
    detail: str


RECONSTRUCT = (EventKind.AgInter, EventKind.AgIntra, EventKind.H2D)


def check_zero_bwd_ag_inter(strategy: StrategyKind, events: Sequence[Event]) -> List[Violation]:
    if strategy not in (StrategyKind.Fcdp, StrategyKind.FcdpComm, StrategyKind.ZeroPP):
        return []
    fwd = [e.id for e in events if e.kind == EventKind.ComputeFwd]
    if not fwd:
        return []
    last = max(fwd)
    return [Violation("zero_bwd_ag_inter", e.id, f"backward AgInter of layer {e.layer}")
            for e in events if e.kind == EventKind.AgInter and e.id > last]


def check_frozen_gather_once(programs: Sequence[Sequence[Event]], frozen_layers: Iterable[int]) -> List[Violation]:
    frozen_layers = set(frozen_layers)
    seen: Dict[int, int] = {}
    out = []
    for it, events in enumerate(programs, start=1):
        for e in events:
            if e.kind == EventKind.AgInter and e.layer in frozen_layers and e.param_set != ParamSet.TrainableOnly:
                seen[e.layer] = seen.get(e.layer, 0) + 1
                if it > 1:
                    out.append(Violation("frozen_gather_once", e.id,
                                         f"frozen portion of layer {e.layer} re-gathered in iteration {it}"))
    for l in frozen_layers:
        if programs and seen.get(l, 0) != 1:
            out.append(Violation("frozen_gather_once", None, f"layer {l} frozen portion gathered {seen.get(l, 0)} times"))
    return out


def check_dirty_iff_stale(states: Sequence[ParamState]) -> List[Violation]:
    out = []
    for i, s in enumerate(states):
        stale = s.host_cached_version is None or s.host_cached_version != s.version
        if s.dirty != stale:
            out.append(Violation("dirty_iff_stale", None, f"portion {i} (layer {s.layer}, frozen={s.frozen}) "
                                                          f"dirty={s.dirty} but stale={stale}"))
    return out


def check_compute_has_params(events: Sequence[Event], retained: Sequence[int] = ()) -> List[Violation]:
    by_id = {e.id: e for e in events}
    out = []

    def reaches(eid: int, layer: int, seen: set) -> bool:
        if eid in seen:
            return False
        seen.add(eid)
        e = by_id[eid]
        if e.kind in RECONSTRUCT and e.layer == layer:
            return True
        return any(reaches(d, layer, seen) for d in e.deps
                   if by_id[d].kind in RECONSTRUCT and by_id[d].layer == layer)

    for e in events:
        if e.kind not in (EventKind.ComputeFwd, EventKind.ComputeBwd):
            continue
        if e.kind == EventKind.ComputeBwd and e.layer in retained:
            continue
        if not any(reaches(d, e.layer, set()) for d in e.deps):
            out.append(Violation("compute_has_params", e.id, f"{e.kind.name} of layer {e.layer} has no "
                                                             "reconstruction dependency"))
    return out


def check_bytes_conserved(measured: Dict[str, int], expected: Dict[str, int]) -> List[Violation]:
    return [Violation("bytes_conserved", None, f"{k}: measured {measured.get(k)} != oracle {v}")
            for k, v in expected.items() if measured.get(k) != v]


def check_trace_respects_deps(events: Sequence[Event], begin_ms: Sequence[float], end_ms: Sequence[float],
                              tol_ms: float = 0.05) -> List[Violation]:
    """Executed-trace rule: every event began (its stream reached it, after its
    dependency waits) no earlier than each dependency finished."""
    out = []
    for e in events:
        for d in e.deps:
            if begin_ms[e.id] + tol_ms < end_ms[d]:
                out.append(Violation("trace_respects_deps", e.id,
                                     f"{e.kind.name} L{e.layer} began at {begin_ms[e.id]:.3f} ms before dependency "
                                     f"{d} finished at {end_ms[d]:.3f} ms"))
    return out


def overlap_fraction(events: Sequence[Event], begin_ms: Sequence[float], end_ms: Sequence[float],
                     kinds: Iterable[EventKind], against: Iterable[EventKind]) -> Optional[float]:
    """Fraction of the device time of events of `kinds` (e.g. the FCDP-Cache
    D2H stores) that overlaps the union of events of `against` (e.g. compute):
    north_star's "overlapped with compute", measured on an executed trace."""
    kinds, against = set(kinds), set(against)
    busy = sorted((begin_ms[e.id], end_ms[e.id]) for e in events if e.kind in against)
    merged: List[List[float]] = []
    for a, b in busy:
        if merged and a <= merged[-1][1]:
            merged[-1][1] = max(merged[-1][1], b)
        else:
            merged.append([a, b])
    total = covered = 0.0
    for e in events:
        if e.kind not in kinds:
            continue
        a, b = begin_ms[e.id], end_ms[e.id]
        total += b - a
        for x, y in merged:
            covered += max(0.0, min(b, y) - max(a, x))
    return covered / total if total > 0 else None


def check_program(strategy: StrategyKind, events: Sequence[Event], retained: Sequence[int] = ()) -> List[Violation]:
    return check_zero_bwd_ag_inter(strategy, events) + check_compute_has_params(events, retained)
