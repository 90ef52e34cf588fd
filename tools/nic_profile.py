"""Inter-node NIC bandwidth profile of one training step (Fig. 10:
"peak inter-node network bandwidth during forward and backward passes").

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/nic_profile.py [--preset gpt2-1.3b] [--strategies zero3,fcdp] [--bin-ms 2]

One process per GPU, emulated topology as bench.py (2 -> 2x1, 4 -> 2x2).  For
each strategy the same trainer runs warm-up steps, then ONE step with every
rank's NIC emulator logging the payloads it paces onto its node's wire
(fcdp_engine_nic_log).  Rank 0 bins node 0's wire intervals into a time series
of NIC bandwidth per traffic kind (forward all-gather, backward all-gather,
reduce-scatter) and prints one JSON object: per strategy the step time, the
bytes per kind, the NIC busy fraction, the peak / mean bandwidth of the
forward-phase and backward-phase traffic and the series itself.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import uuid
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KINDS = {0: "fwd_ag", 1: "bwd_ag", 2: "rs", 15: "grad_sync"}
TOPOLOGY = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}


def series(recs, t0: int, bin_ns: int, nbins: int):
    """Bytes of each kind that cross the wire inside each bin (intervals split pro rata)."""
    import numpy as np
    out = {name: np.zeros(nbins) for name in KINDS.values()}
    for r in recs:
        s, e, b, k = int(r["start_ns"]) - t0, int(r["end_ns"]) - t0, float(r["bytes"]), KINDS[int(r["kind"])]
        if e <= s:
            out[k][min(max(s // bin_ns, 0), nbins - 1)] += b
            continue
        rate = b / (e - s)
        i = s // bin_ns
        while s < e and i < nbins:
            hi = min(e, (i + 1) * bin_ns)
            out[k][i] += rate * (hi - s)
            s, i = hi, i + 1
    return out


def summarise(recs, step_ms: float, bin_ms: float):
    import numpy as np
    if len(recs) == 0:
        return {"step_ms": step_ms, "bytes": {k: 0 for k in KINDS.values()}, "nic_busy_frac_of_step": 0.0}
    t0 = int(recs["start_ns"].min())
    t1 = int(recs["end_ns"].max())
    bin_ns = int(bin_ms * 1e6)
    nbins = max(1, -(-(t1 - t0) // bin_ns))
    ser = series(recs, t0, bin_ns, nbins)
    gbs = {k: v / (bin_ns / 1e9) / 1e9 for k, v in ser.items()}
    fwd = gbs["fwd_ag"]
    bwd = gbs["bwd_ag"] + gbs["rs"] + gbs["grad_sync"]
    busy_ns = float((recs["end_ns"] - recs["start_ns"]).sum())

    def stats(x):
        nz = x[x > 0]
        return {"peak_gbs": float(x.max()), "mean_gbs_while_active": float(nz.mean()) if nz.size else 0.0,
                "active_ms": float(nz.size * bin_ms)}

    return {
        "step_ms": step_ms,
        "wire_span_ms": (t1 - t0) / 1e6,
        "bytes": {name: int(recs["bytes"][recs["kind"] == k].sum()) for k, name in KINDS.items()},
        "nic_busy_frac_of_step": busy_ns / 1e6 / step_ms,
        "forward_phase": stats(fwd),
        "backward_phase": stats(bwd),
        "series": {"bin_ms": bin_ms, **{k: [round(float(x), 3) for x in v] for k, v in gbs.items()}},
    }


def spark(x, width=100):
    import numpy as np
    x = np.asarray(x, dtype=float)
    if x.size == 0 or x.max() <= 0:
        return ""
    idx = np.linspace(0, x.size, min(width, x.size) + 1).astype(int)
    vals = [x[a:b].mean() if b > a else 0.0 for a, b in zip(idx[:-1], idx[1:])]
    ch = " .:-=+*#%@"
    return "".join(ch[min(len(ch) - 1, int(round(v / x.max() * (len(ch) - 1))))] for v in vals)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="gpt2-1.3b")
    ap.add_argument("--strategies", default="zero3,fcdp")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--inter", default="ib100-rdma-measured")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--bin-ms", type=float, default=2.0)
    ap.add_argument("--topology", default="")
    ap.add_argument("--tau", type=float, default=0.9)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.driving_model import PRESETS
    from paper_2602_06499_b200.trainer import FcdpTrainer, synthetic_batch

    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N, g = (int(x) for x in a.topology.split("x")) if a.topology else TOPOLOGY[world]
    mc = PRESETS[a.preset]
    topo = S.make_topology(N, g, inter_preset=a.inter)
    cap = torch.cuda.get_device_properties(dev).total_memory
    result = {"preset": a.preset, "topology": f"{N}x{g}", "inter_link": a.inter,
              "nic_gbs": topo.inter_node.bandwidth_bytes_per_s / 1e9, "strategies": {}}
    for strat in a.strategies.split(","):
        box = [f"fcdp_nicprof_{uuid.uuid4().hex[:12]}" if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        plan = S.StrategyPlan(S.StrategyKind.from_string(strat), tau=a.tau if strat.startswith("fcdp") else 0.0)
        tr = FcdpTrainer(mc, topo, plan, rank=rank, world_size=world, device=local, shm_name=box[0],
                         batch_per_gpu=a.batch, gpu_capacity_bytes=cap if plan.tau > 0 else 0)
        for i in range(a.warmup):
            tr.step(*synthetic_batch(mc.vocab, a.batch, mc.seq, 0x5EED, i, rank, device=dev))
        tr.sync()
        torch.cuda.synchronize()
        x, y = synthetic_batch(mc.vocab, a.batch, mc.seq, 0x5EED, a.warmup, rank, device=dev)
        tr.engine.set_nic_log(True)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(tr.stream)
        tr.step(x, y)
        e1.record(tr.stream)
        tr.sync()
        torch.cuda.synchronize()
        log = tr.engine.nic_log()
        tr.engine.set_nic_log(False)
        step_ms = e0.elapsed_time(e1)
        logs = [None] * world
        if world > 1:
            dist.all_gather_object(logs, (log, step_ms))
        else:
            logs = [(log, step_ms)]
        tr.close()
        del tr
        torch.cuda.empty_cache()
        if rank == 0:
            node0 = np.concatenate([logs[j][0] for j in range(g)])  # ranks of node 0
            step = max(s for _, s in logs)
            result["strategies"][strat] = summarise(node0, step, a.bin_ms)
    if rank == 0:
        for strat, r in result["strategies"].items():
            ser = r.get("series", {})
            print(f"[nic] {strat:9s} step {r['step_ms']:.1f} ms, NIC busy {r['nic_busy_frac_of_step']:.2f} of the step",
                  file=sys.stderr)
            for k in ("fwd_ag", "bwd_ag", "rs"):
                if ser.get(k) and max(ser[k]) > 0:
                    print(f"    {k:7s} |{spark(ser[k])}|", file=sys.stderr)
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
