"""Executed-event timeline of one training step (engine trace) on the GPU box.

    python tools/trace_step.py [--preset gpt2-1.3b] [--strategy fcdp] [--batch 8] [--topology 1x1]

Prints per-kind totals and the per-event begin/end (device ms from the
iteration start) of the last step; with torchrun, rank 0 prints.
"""
import argparse
import json
import os
import sys
os_env_set = __import__('os').environ.setdefault('CUDA_DEVICE_MAX_CONNECTIONS', '32')
import uuid
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="gpt2-1.3b")
    ap.add_argument("--strategy", default="fcdp")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--topology", default="1x1")
    ap.add_argument("--inter", default="ib100-rdma-measured")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--copy-engine", action="store_true")
    ap.add_argument("--tau", type=float, default=0.0, help="FCDP-Cache retention threshold (capacity = GPU memory)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.driving_model import PRESETS
    from paper_2602_06499_b200.trainer import FcdpTrainer, synthetic_batch
    rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    N, g = (int(x) for x in a.topology.split("x"))
    if world > 1:
        dist.init_process_group("gloo")
    name = [f"fcdp_trace_{uuid.uuid4().hex[:10]}"]
    if world > 1:
        dist.broadcast_object_list(name, src=0)
    mc = PRESETS[a.preset]
    tr = FcdpTrainer(mc, S.make_topology(N, g, inter_preset=a.inter),
                     S.StrategyPlan(S.StrategyKind.from_string(a.strategy), tau=a.tau), rank=rank, world_size=world,
                     device=local, shm_name=name[0], batch_per_gpu=a.batch, use_copy_engine=a.copy_engine,
                     gpu_capacity_bytes=torch.cuda.get_device_properties(local).total_memory if a.tau > 0 else 0)
    dev = torch.device("cuda", local)
    for i in range(a.steps):
        if i == a.steps - 1:
            tr.engine.set_trace(True)
        x, y = synthetic_batch(mc.vocab, a.batch, mc.seq, 1, i, rank, device=dev)
        tr.step(x, y)
    tr.sync()
    rows = tr.engine.trace(tr.last_program)
    if rank == 0:
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for ev, b, e in rows:
            tot[ev.kind.name] += e - b
            cnt[ev.kind.name] += 1
        step_ms = max(e for _, _, e in rows)
        print(f"step (last event end) {step_ms:.2f} ms")
        for k in sorted(tot, key=lambda k: -tot[k]):
            print(f"  {k:14s} n={cnt[k]:3d} busy={tot[k]:8.2f} ms")
        out = [{"id": ev.id, "kind": ev.kind.name, "layer": ev.layer, "set": ev.param_set.name,
                "bytes": ev.bytes_total, "begin_ms": b, "end_ms": e} for ev, b, e in rows]
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps({"step_ms": step_ms, "events": out}, indent=0))
        for r in out[:12] + out[-12:]:
            print(r)
    tr.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
