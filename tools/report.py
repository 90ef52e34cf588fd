"""Render bench.py JSON lines (profiles/r01_bench_*.json) as the markdown rows
of DESIGN.md §10: throughput per strategy, inter-node AG bytes, link floor,
dominant-kernel roofline and host-link copies.

    python tools/report.py profiles/r01_bench_n1.json profiles/r01_bench_n2.json ...
"""
import json
import sys


def fmt(x, nd=0):
    return "—" if x is None else f"{x:,.{nd}f}"


def row(d):
    cfg = d.get("config", {})
    z3, zpp, mics, var = (d.get(k) or {} for k in ("zero3", "zeropp", "mics", "fcdp_variant"))
    ag = d.get("ag_inter_bytes_per_step_per_node") or {}
    lb = d.get("link_bound") or {}
    rf = d.get("roofline") or {}
    iso = rf.get("isolated") or {}
    fwd_bwd = (ag.get("fcdp_fwd") or 0) + (ag.get("fcdp_bwd") or 0)
    z3_ag = (ag.get("zero3_fwd") or 0) + (ag.get("zero3_bwd") or 0)
    return ("| {model} {topo} | {v} | {tau0} | {z3} | {zpp} | {mics} | {ag} / {z3ag} GB | {lbf} | {k} {frac} (alone {iso}) |"
            .format(model=cfg.get("model"), topo=cfg.get("topology"), v=fmt(d.get("value")),
                    tau0=fmt(var.get("tokens_per_s")), z3=fmt(z3.get("tokens_per_s")), zpp=fmt(zpp.get("tokens_per_s")),
                    mics=fmt(mics.get("tokens_per_s")), ag=fmt(fwd_bwd / 1e9, 3), z3ag=fmt(z3_ag / 1e9, 3) if z3_ag else "—",
                    lbf=fmt(lb.get("frac"), 3), k=rf.get("kernel"), frac=fmt(rf.get("frac"), 2),
                    iso=fmt(iso.get("frac"), 2)))


def main(paths):
    print("| config | FCDP tok/s | τ=0 | ZeRO-3 | ZeRO++ | MiCS | AG bytes/node FCDP / ZeRO-3 | link floor frac | dominant kernel frac |")
    print("|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        with open(p) as f:
            lines = [l for l in f.read().splitlines() if l.startswith("{")]
        if lines:
            print(row(json.loads(lines[-1])))


if __name__ == "__main__":
    main(sys.argv[1:])
