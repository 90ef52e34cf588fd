"""Where the driving model's step time goes (torch.profiler, CUPTI kernels).

    python tools/model_profile.py [--preset gpt2-1.3b] [--strategy fcdp] [--tau 0.9] [--steps 2]

Runs the bench's N=1 trainer for a few steps and prints the CUDA time per
aten op (self device time, summed over the profiled steps / steps) and the top
kernels, so the non-GEMM part of the driving model can be attributed.
"""
import argparse
import os
import sys
import uuid
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="gpt2-1.3b")
    ap.add_argument("--strategy", default="fcdp")
    ap.add_argument("--tau", type=float, default=0.9)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--rows", type=int, default=40)
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.driving_model import PRESETS
    from paper_2602_06499_b200.trainer import FcdpTrainer, synthetic_batch
    mc = PRESETS[a.preset]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cap = torch.cuda.get_device_properties(0).total_memory
    tr = FcdpTrainer(mc, S.make_topology(1, 1), S.StrategyPlan(S.StrategyKind.from_string(a.strategy), tau=a.tau),
                     rank=0, world_size=1, device=0, shm_name=f"fcdp_prof_{uuid.uuid4().hex[:8]}",
                     batch_per_gpu=a.batch, gpu_capacity_bytes=cap if a.tau > 0 else 0)
    batches = [synthetic_batch(mc.vocab, a.batch, mc.seq, 7, i, 0, device=dev) for i in range(3 + a.steps)]
    for i in range(3):
        tr.step(*batches[i])
    tr.sync()
    torch.cuda.synchronize()
    # host enqueue time vs device time per step: is the Python/engine host side
    # keeping ahead of the GPU?
    import time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    e0.record(tr.stream)
    for i in range(a.steps):
        t0 = time.perf_counter()
        tr.step(*batches[3 + i])
        host.append((time.perf_counter() - t0) * 1e3)
    e1.record(tr.stream)
    tr.sync()
    torch.cuda.synchronize()
    print(f"host enqueue ms/step: {sum(host) / len(host):.2f} (each {[round(h, 1) for h in host]}); "
          f"device ms/step: {e0.elapsed_time(e1) / a.steps:.2f}")
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for i in range(a.steps):
            tr.step(*batches[3 + i])
        tr.sync()
        torch.cuda.synchronize()
    # device busy time (union of kernel / memcpy intervals over all streams) vs the span
    import json
    import tempfile
    with tempfile.NamedTemporaryFile(suffix=".json") as f:
        prof.export_chrome_trace(f.name)
        tr_ev = json.load(open(f.name)).get("traceEvents", [])
    iv = sorted((e["ts"], e["ts"] + e.get("dur", 0)) for e in tr_ev
                if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and e.get("dur", 0) > 0)
    if iv:
        busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
        for s_, e_ in iv[1:]:
            if s_ > cur_e:
                busy += cur_e - cur_s
                cur_s, cur_e = s_, e_
            else:
                cur_e = max(cur_e, e_)
        busy += cur_e - cur_s
        span = iv[-1][1] - iv[0][0]
        print(f"device busy (any stream) {busy / 1e3 / a.steps:.2f} ms/step of a {span / 1e3 / a.steps:.2f} ms/step "
              f"span: idle {(span - busy) / 1e3 / a.steps:.2f} ms/step")
    ka = prof.key_averages()
    rows = sorted(ka, key=lambda e: -getattr(e, "self_device_time_total", getattr(e, "self_cuda_time_total", 0)))
    tot = sum(getattr(e, "self_device_time_total", getattr(e, "self_cuda_time_total", 0)) for e in ka)
    print(f"total self device time per step: {tot / a.steps / 1e3:.2f} ms")
    for e in rows[:a.rows]:
        t = getattr(e, "self_device_time_total", getattr(e, "self_cuda_time_total", 0))
        if t <= 0:
            continue
        print(f"{t / a.steps / 1e3:8.3f} ms/step  n={e.count // a.steps:5d}  {e.key[:110]}")
    tr.close()


if __name__ == "__main__":
    main()
