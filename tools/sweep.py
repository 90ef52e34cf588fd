"""Topology / bandwidth sweep (config C5): FCDP vs ZeRO-3 on the same box.

    python tools/sweep.py --gpus 4 [--presets ib100-rdma-measured,eth10g-measured] [--out gpurun_out/sweep.jsonl]

For every emulated topology N x g with N*g == --gpus and every inter-node
preset, runs bench.py (torchrun, one process per GPU) for fcdp and zero3 and
records tokens/s and the measured inter-group bytes per node per step.
"""
import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def topologies(G):
    return [(N, G // N) for N in (1, 2, 4, 8) if G % N == 0 and G // N <= 8]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--presets", default="ib100-rdma-measured,eth100g-theoretical,ib100-ipoib-measured,"
                                         "eth10g-measured,eth1g-measured")
    ap.add_argument("--strategies", default="fcdp,zero3")
    ap.add_argument("--preset-model", default="gpt2-1.3b")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--topologies", default="", help="comma list NxG (default: all with N*G == gpus)")
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    ap.add_argument("--per-run-timeout", type=int, default=240)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tau-variant", default="-1", help="also time this tau (bench --tau-variant); -1 = no")
    a = ap.parse_args()
    out = Path(a.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    port = 29600
    topos = [tuple(int(x) for x in t.split("x")) for t in a.topologies.split(",")] if a.topologies else topologies(a.gpus)
    for (N, g) in topos:
        for preset in a.presets.split(","):
            for strat in a.strategies.split(","):
                port += 1
                cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
                       "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                       "--gpus", str(a.gpus), "--topology", f"{N}x{g}", "--inter", preset, "--strategy", strat,
                       "--preset", a.preset_model, "--batch", str(a.batch), "--steps", str(a.steps),
                       "--warmup", str(a.warmup), "--no-zero3", "--no-e2e", "--no-cpu-baseline",
                       "--tau-variant", a.tau_variant,
                       "--engine-timeout", "120", "--watchdog", str(a.per_run_timeout - 20)]
                if a.gpus == 1:
                    cmd = [sys.executable, str(ROOT / "bench.py")] + cmd[cmd.index("--gpus"):]
                try:
                    r = subprocess.run(cmd, capture_output=True, text=True, timeout=a.per_run_timeout)
                    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
                    rec = json.loads(line[-1]) if line else {"error": r.stderr[-800:]}
                except subprocess.TimeoutExpired:
                    rec = {"error": "timeout"}
                row = {"topology": f"{N}x{g}", "inter": preset, "strategy": strat,
                       "tokens_per_s": rec.get("value"), "ms_per_step": rec.get("ms_per_step"),
                       "ag_bytes_per_node": rec.get("ag_inter_bytes_per_step_per_node"),
                       "error": rec.get("error")}
                print(json.dumps(row), flush=True)
                with out.open("a") as f:
                    f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
