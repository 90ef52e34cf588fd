"""Read an engine trace (tools/trace_step.py output) and explain the step time.

    python tools/trace_report.py gpurun_out/trace_fcdp_2x1.json

Prints, for the compute stream, every idle gap > 0.2 ms and the event that was
running late (the dependency the compute waited for).
"""
import json
import sys
from collections import defaultdict

STREAM = {"AgInter": "gather", "AgIntra": "gather", "H2D": "gather", "D2H": "cache", "ReduceScatter": "rs",
          "ComputeFwd": "comp", "ComputeBwd": "comp", "OptimizerStep": "comp", "MaskDirty": "comp"}


def main(path):
    d = json.load(open(path))
    ev = d["events"]
    print(f"{path}: step {d['step_ms']:.1f} ms, {len(ev)} events")
    busy = defaultdict(float)
    for e in ev:
        busy[STREAM[e["kind"]]] += e["end_ms"] - e["begin_ms"]
    print("stream busy (ms):", {k: round(v, 1) for k, v in busy.items()})
    comp = [e for e in ev if STREAM[e["kind"]] == "comp" and e["kind"] != "MaskDirty"]
    t = 0.0
    idle = 0.0
    for e in comp:
        gap = e["begin_ms"] - t
        # the compute event's own end minus duration tells when it could start; gaps show waiting
        if gap > 0.2:
            idle += gap
            print(f"  compute idle {gap:6.2f} ms before {e['kind']} L{e['layer']}")
        t = max(t, e["end_ms"])
    kinds = defaultdict(list)
    for e in ev:
        kinds[e["kind"]].append(e["end_ms"] - e["begin_ms"])
    for k, v in kinds.items():
        print(f"  {k:14s} n={len(v):3d} mean {sum(v)/len(v):6.2f} ms  max {max(v):6.2f}")
    print(f"compute idle total {idle:.1f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
