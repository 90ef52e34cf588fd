"""Summarise ncu reports for profiles/: per kernel class, dram bytes and duration per launch.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv] > profiles/...

Kernel classes follow the engine's accounting: gather_expand (concat/expand/copy),
rs_slice, rs_finalize, adamw.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

CLASSES = [("adamw_fused_rs", r"adam_grad_kernel"), ("adamw", r"adam_kernel"), ("rs_finalize", r"rs_finalize_kernel"),
           ("rs_slice", r"rs_(dense|masked)_kernel"),
           ("gather_expand", r"(expand_kernel|concat_kernel|copy_kernel|bulk_copy_kernel)"),
           ("partition", r"partition_kernel"), ("fcdp_setup", r"(init_kernel|widen_kernel)"),
           ("grad_handoff", r"seg_copy_kernel"),
           # driving-model kernels (model_kernels.cu): the path's consumer, not the path
           ("model_bias_gelu_fwd", r"bias_gelu_fwd_kernel"), ("model_gelu_bwd_bias_grad", r"colsum_partial_kernel<(true|1)>"),
           ("model_bias_grad", r"colsum_(partial|final)_kernel"), ("model_layernorm", r"ln_(fwd|bwd)"),
           ("model_xent", r"xent_(fwd|bwd)_kernel"), ("model_rope", r"rope_kernel"), ("model_swiglu", r"swiglu_"),
           ("model_rmsnorm", r"rms_(fwd|bwd)")]


def ours(name):
    """A kernel of libfcdp: namespace fcdp::(anonymous); ncu prints it either as
    "fcdp::<unnamed>::k" or, shortened, "unnamed>::k" at the start of the name."""
    return "fcdp::" in name or re.match(r"^(void )?unnamed>::", name) is not None


def klass(name):
    if not ours(name):
        return None
    for c, pat in CLASSES:
        if re.search(pat, name):
            return c
    return None


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {}
        for h, u, v in zip(hdr, units, r):
            f = num(v)
            d[h] = f * UNIT[u] if (f is not None and u in UNIT) else v
        recs.append(d)
    return recs


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarise_full(rep):
    acc = defaultdict(lambda: defaultdict(list))
    for r in raw_rows(rep):
        name = r.get("Kernel Name") or r.get("Function Name") or ""
        c = klass(name)
        if not c:
            continue
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
                    "launch__grid_size", "launch__block_size"):
            v = num(r.get(key))
            if v is not None:
                acc[c][key].append(v)
        acc[c]["names"].append(name[:120])
    res = {}
    for c, d in acc.items():
        mean = {k: sum(v) / len(v) for k, v in d.items() if k != "names" and v}
        rb, wb = mean.get("dram__bytes_read.sum"), mean.get("dram__bytes_write.sum")
        res[c] = {"launches_profiled": len(d["names"]), "kernel": d["names"][0],
                  "duration_s": mean.get("gpu__time_duration.sum"),
                  "dram_bytes_per_launch": (rb or 0) + (wb or 0) if rb is not None else None,
                  "dram_read": rb, "dram_write": wb, **{k: v for k, v in mean.items()}}
    return res


def summarise_launches(path):
    """ncu --metrics gpu__time_duration.sum --csv launch list: time share per kernel."""
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = num(d.get("Metric Value"))
        if v is None:
            continue
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
        name = d["Kernel Name"]
        key = klass(name) or (("fcdp:" if ours(name) else "torch/cublas:") + name[:60])
        tot[key] += v * scale
        cnt[key] += 1
    all_ms = sum(tot.values())
    return {k: {"launches": cnt[k], "ms": tot[k], "share": tot[k] / all_ms if all_ms else None}
            for k in sorted(tot, key=lambda k: -tot[k])}


if __name__ == "__main__":
    out = {}
    args = sys.argv[1:]
    if "--launches" in args:
        i = args.index("--launches")
        out["launch_list"] = summarise_launches(args[i + 1])
        del args[i:i + 2]
    for rep in args:
        out.update(summarise_full(rep))
    print(json.dumps(out, indent=1))
