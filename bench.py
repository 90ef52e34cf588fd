#!/usr/bin/env python
"""FCDP on B200: training-step throughput and inter-group all-gather bytes.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fcdp|reference]

Metric (BASELINE.json): train step tokens/s at 1/2/4/8 B200, with the
inter-group AG bytes per step against an on-box ZeRO-3 schedule.  The 8-GPU
config is GPT-2 1.3B as 2 emulated nodes x 4 GPUs behind a throttled
host-staged inter-node link; N GPUs map to the emulated topology
1 -> 1x1, 2 -> 2x1, 4 -> 2x2, 8 -> 2x4 (weak scaling: batch per GPU fixed).

One process per GPU (torchrun for N > 1).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import uuid
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see package __init__)

METRIC = "train step tokens/s at 1/2/4/8 B200; inter-group AG bytes/step vs ZeRO-3"
TOPOLOGY = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="fcdp", choices=["fcdp", "reference"])
    p.add_argument("--preset", default="gpt2-1.3b")
    p.add_argument("--strategy", default="fcdp")
    p.add_argument("--inter", default="ib100-rdma-measured")
    p.add_argument("--batch", type=int, default=8,
                   help="sequences per GPU; 0 = ZeRO-3 max batch (reference max_feasible_batch fed with the "
                        "activation bytes per sample measured on this box)")
    p.add_argument("--seq", type=int, default=0)
    p.add_argument("--topology", default="", help="override NxG, e.g. 1x2")
    p.add_argument("--zero3-steps", type=int, default=3)
    p.add_argument("--no-zero3", action="store_true")
    p.add_argument("--zeropp", action="store_true", help="also measure ZeRO++ (GPU node replica) on the same executor")
    p.add_argument("--mics", action="store_true", help="also measure MiCS (node-local shards + replica gradient sync)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--copy-engine", action="store_true")
    p.add_argument("--watchdog", type=float, default=900.0,
                   help="dump every thread's stack and exit if the run exceeds this many seconds")
    p.add_argument("--engine-timeout", type=float, default=300.0)
    p.add_argument("--no-pacing", action="store_true", help="do not throttle the emulated inter-node link")
    p.add_argument("--tau", type=float, default=0.9,
                   help="FCDP-Cache adaptive GPU-retention threshold of the headline run (PAPER.md:455-462; "
                        "capacity = this GPU's memory).  0 = every layer through the pinned host cache")
    p.add_argument("--tau-variant", type=float, default=0.0,
                   help="tau of the secondary FCDP run reported beside the headline (default 0: the pure "
                        "host-cache path); negative disables")
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region, for the GPUs this job uses."""

    def __init__(self, world: int = 1):
        self.proc = None
        self.lines = []
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        ids = vis.split(",")[:world] if vis else [str(i) for i in range(world)]
        self.ids = ",".join(ids)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.ids,
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "gpus": self.ids}


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def nvlink_peak():
    """Measured NVLink peer-copy rate per direction on this pool's B200s
    (tools/nvlink_probe.py, profiles/r02_nvlink_probe.json), with its source."""
    try:
        d = json.loads((ROOT / "profiles" / "r02_nvlink_probe.json").read_text())
        return float(d["nvlink_peak_GBps_measured"]), ("profiles/r02_nvlink_probe.json: measured copy-engine peer copy "
                                                        "GPU1->GPU0 (tools/nvlink_probe.py); the gather / RS kernels reach "
                                                        "0.99-1.00 of it alone")
    except Exception:
        return 770.0, "B200_PROFILING.md peer copy 770 GB/s per direction (fallback: no committed probe)"


def ncu_traffic(kernel_class: str):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    try:
        s = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        return s.get(kernel_class, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def control_plane_timing(mc, strategy: str, N: int, g: int, iters: int = 1000):
    """BASELINE.md §3 "Timing 1": build_iteration + step_state + comm_volume per
    step on the host, through the compiled reference (oracle/_ref/time_ref, built
    from /root/reference's own sources) and through this project's libfcdp
    (time_ours), same driver source (tests/cpp/control_plane_timer.cpp)."""
    params = [str(d.numel) for d in mc.layer_defs()]
    out = {}
    for key, exe in (("reference_us_per_step", "time_ref"), ("ours_us_per_step", "time_ours")):
        path = ROOT / "oracle" / "_ref" / exe
        if not path.exists():
            continue
        try:
            r = subprocess.run([str(path), strategy, str(N), str(g), str(iters), str(mc.dtype_bytes)] + params,
                               capture_output=True, text=True, timeout=60)
            out[key] = json.loads(r.stdout)["us_per_step"]
        except Exception:
            pass
    if out:
        out["note"] = "host CPU, 1 thread; model = the bench's explicit layer list"
    return out or None


def isolated_rate(kernel_class: str, alg_bytes: float, eb: int, dev, fused_adam: bool = False):
    """The dominant kernel re-timed alone (after the timed region) at the live
    per-launch size: stateless C-ABI launch on synthetic buffers, L2 flushed
    between reps, CUDA events, median.  The live number in `roofline` includes
    any time the kernel spent sharing SMs / HBM with concurrent work (the
    driving model's backward GEMMs at N > 1); this one is the kernel itself."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2602_06499_b200 import _capi
    lib = _capi.lib()
    P = lambda t: C.c_void_p(t.data_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    keep = []

    def dense_layout(chunks):
        m = np.ones(chunks, np.uint8)
        out = C.c_void_p()
        _capi.check(lib.fcdp_layout_create(chunks, m.ctypes.data_as(C.POINTER(C.c_uint8)), eb, 1, 1, C.byref(out)))
        return out

    V = 16 // eb
    if kernel_class == "adamw" and fused_adam:
        # G = 1: the fused RS + AdamW reading the bf16 gradient in place (24 + 2*eb B/param)
        n = int(alg_bytes // (6 * 4 + 2 * eb)) // (16 // eb) * (16 // eb)
        w, m_, v_ = torch.randn(n, device=dev), torch.zeros(n, device=dev), torch.zeros(n, device=dev)
        g_ = torch.randn(n, device=dev).mul_(1e-3).to(torch.bfloat16 if eb == 2 else torch.float32)
        par = torch.empty(n * eb, dtype=torch.uint8, device=dev)
        cfg = _capi.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
        offs, cnts = (C.c_int64 * 1)(0), (C.c_int64 * 1)(n)
        ptrs = (C.c_void_p * 1)(g_.data_ptr())
        keep += [w, m_, v_, g_, par]
        fn = lambda: _capi.check(lib.fcdp_adam_grad_step(n, C.byref(cfg), 1.0, 1, offs, ptrs, cnts, P(w), P(m_),
                                                         P(v_), P(par), eb, None, None))
    elif kernel_class == "adamw":
        n = int(alg_bytes // (7 * 4 + eb)) // 4 * 4
        # real-valued inputs: an all-zero gradient sends the IEEE divisions down their slow path
        w, g_ = torch.randn(n, device=dev), torch.randn(n, device=dev).mul_(1e-3)
        m_, v_ = torch.zeros(n, device=dev), torch.zeros(n, device=dev)
        par = torch.empty(n * eb, dtype=torch.uint8, device=dev)
        cfg = _capi.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
        keep += [w, m_, v_, g_, par]
        fn = lambda: _capi.check(lib.fcdp_adam_step(n, C.byref(cfg), P(w), P(m_), P(v_), P(g_), P(par), eb, None))
    elif kernel_class in ("gather_expand", "shard_copy"):
        chunks = int(alg_bytes // 32)
        lay = dense_layout(chunks)
        x = torch.empty(chunks * 16, dtype=torch.uint8, device=dev)
        y = torch.empty_like(x)
        keep += [x, y]
        fn = lambda: _capi.check(lib.fcdp_expand(lay, (C.c_void_p * 1)(x.data_ptr()), None, P(y), 0, None))
    elif kernel_class == "rs_slice":
        chunks = int(alg_bytes // (16 + 16 * 4 // eb))  # dtype grads in, fp32 shard out
        lay = dense_layout(chunks)
        gbuf = torch.empty(chunks * 16, dtype=torch.uint8, device=dev)
        own = torch.empty(chunks * V, dtype=torch.float32, device=dev)
        wire = torch.empty(chunks * 16, dtype=torch.uint8, device=dev)
        keep += [gbuf, own, wire]
        fn = lambda: _capi.check(lib.fcdp_rs_slice(lay, (C.c_void_p * 1)(gbuf.data_ptr()), 0, 0, 1.0, 1, P(own),
                                                   P(wire), None))
    elif kernel_class == "rs_finalize":
        n = int(alg_bytes // (2 * 4 + eb)) // 4 * 4
        own, out = torch.randn(n, device=dev), torch.empty(n, device=dev)
        wire = torch.zeros(2 * n * eb, dtype=torch.uint8, device=dev)
        keep += [own, out, wire]
        fn = lambda: _capi.check(lib.fcdp_rs_finalize(n, 2, 0, eb, P(own), P(wire), n, 0.5, P(out), None))
    else:
        return None
    ts = []
    for i in range(7):
        flush.fill_(i & 0xFF)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    del keep
    return {"ms_per_launch": ms, "achieved": alg_bytes / (ms / 1e3) / 1e9}


def gpu_capacity_bytes_smi() -> int:
    """This box's GPU memory without creating a CUDA context (nvidia-smi); the
    reference arm builds the same tau-admission programs as the GPU arm."""
    try:
        r = subprocess.run(["nvidia-smi", "--query-gpu=memory.total", "--format=csv,noheader,nounits", "-i", "0"],
                           capture_output=True, text=True, timeout=30)
        return int(float(r.stdout.strip().splitlines()[0])) << 20
    except Exception:
        return 183359 << 20  # B200


def cpu_path_sample(args, mc, N, g, seq, steps, warmup, capacity):
    """The C++ CPU executor (oracle/cpu_executor.cpp) on this host's cores: every
    event of the reference-built program of the bench workload, at full size, all
    N*g simulated ranks (one std::thread each), host DRAM; compute events are a
    synthetic elementwise gradient (no model GEMMs - the reference has none)."""
    import psutil
    from oracle.cpu_step import host_bytes_needed, path_executor
    need = host_bytes_needed(args.preset, N, g)
    avail = psutil.virtual_memory().available
    if need > 0.85 * avail:
        return None, f"needs {need / 1e9:.1f} GB of host memory, {avail / 1e9:.1f} GB available"
    tau = args.tau if args.strategy in ("fcdp", "fcdp-comm") else 0.0
    threads = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    ex = path_executor(args.preset, N, g, args.strategy, tau, capacity if tau > 0 else 0, args.batch, seq,
                       threads=threads)
    setup_s = time.perf_counter() - t0
    for _ in range(max(0, warmup)):
        ex.step()
    secs, st = [], None
    for _ in range(max(1, steps)):
        st = ex.step()
        secs.append(st["seconds"])
    ex.close()
    tokens = N * g * args.batch * seq
    total = sum(secs)
    return {"value": tokens * len(secs) / total, "ms_per_step": 1e3 * total / len(secs), "steps": len(secs),
            "warmup": warmup, "threads": threads, "threads_per_rank": max(1, threads // (N * g)),
            "setup_s": setup_s, "host_bytes": need, "bytes_moved_per_step": st["bytes_moved"],
            "host_GBps": st["bytes_moved"] / (total / len(secs)) / 1e9,
            "nic_bytes_per_node_per_step": st["nic_tx_fwd_ag"] + st["nic_tx_bwd_ag"] + st["nic_tx_rs"],
            "sample": (f"full step of the path, every one of the {st['events']} events of the reference-built "
                       f"{args.strategy} program ({mc.name}, all {len(mc.layer_defs())} layers, full size, "
                       f"{N}x{g} simulated ranks = {N * g} rank threads, {threads} host threads), host DRAM; "
                       f"compute events = synthetic elementwise gradient, no model GEMMs (the reference has "
                       f"no model compute; leaving it out only speeds the CPU up)")}, None


def run_reference(args, world_n):
    """--impl reference: the C++ CPU reference of the path on the host cores
    (rank 0 only; the other ranks exit without work)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2602_06499_b200.driving_model import PRESETS
    mc = PRESETS[args.preset]
    seq = args.seq or mc.seq
    N, g = TOPOLOGY.get(world_n, (1, world_n))
    if args.topology:
        N, g = (int(x) for x in args.topology.lower().split("x"))
    if args.batch <= 0:
        args.batch = 8
    res, why = cpu_path_sample(args, mc, N, g, seq, args.steps, args.warmup, gpu_capacity_bytes_smi())
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return
    value = res["value"]
    cpu = {"value": value, "unit": "tokens/s", "cores": res["threads"], "kind": "port", "sample": res["sample"],
           "executor": "oracle/cpu_executor.cpp (C++; reference control plane oracle/_ref/libshardsim_ref.a)",
           "host_GBps": res["host_GBps"], "bytes_moved_per_step": res["bytes_moved_per_step"],
           "setup_s": res["setup_s"], "control_plane": control_plane_timing(mc, args.strategy, N, g)}
    try:
        from oracle.cpu_step import c1_tiny_timing
        cpu["c1_tiny"] = c1_tiny_timing()
    except Exception as e:  # noqa: BLE001 - a side measurement, never fatal
        cpu["c1_tiny"] = {"error": str(e)[:200]}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world_n,
            "steps": res["steps"], "warmup": res["warmup"], "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16" if mc.dtype_bytes == 2 else "fp32", "data": "synthetic",
            "config": workload_config(args, mc, N, g, world_n, seq), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, mc, N, g, world, seq):
    return {"workload": f"{mc.name} {args.strategy} train step, {N}x{g} emulated nodes x GPUs, "
                        f"inter link {args.inter} (paced NIC emulator)",
            "model": mc.name, "global_batch": args.batch * world, "seq_len": seq,
            "parallelism": f"{args.strategy} dp{world} ({N} emulated nodes x {g} GPUs)",
            "topology": f"{N}x{g}", "inter_link": args.inter, "strategy": args.strategy,
            "fcdp_cache_tau": args.tau if args.strategy in ("fcdp", "fcdp-comm") else None,
            "l2": "inputs larger than L2 (layer params, host cache, optimizer state >> 126 MB)"}


def main():
    args = parse()
    rank, world, local = env_rank()
    import faulthandler
    faulthandler.dump_traceback_later(args.watchdog, exit=True)
    if args.impl == "reference":
        run_reference(args, args.gpus if world == 1 else world)
        return
    import torch
    import torch.distributed as dist
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.driving_model import PRESETS
    from paper_2602_06499_b200.trainer import FcdpTrainer, synthetic_batch

    if world != args.gpus and world > 1:
        args.gpus = world
    ndev = torch.cuda.device_count()
    shared = world > ndev  # more ranks than GPUs (a functional check only: ranks share a GPU's compute)
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if shared else dev  # gloo for the bench's own barrier / reductions then
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if args.topology:
        N, g = (int(x) for x in args.topology.lower().split("x"))
    else:
        N, g = TOPOLOGY.get(world, (1, world))
    assert N * g == world, "topology must cover every rank"
    mc = PRESETS[args.preset]
    seq = args.seq or mc.seq
    topo = S.make_topology(N, g, inter_preset=args.inter)

    def bcast(obj):
        if world == 1:
            return obj
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def pcie_peak() -> dict:
        """Pinned host <-> this GPU copy rate, measured in this run: each rank
        alone in turn (the link's peak: the denominator the engine's copies are
        judged against) and all ranks at once (what a shared host delivers)."""
        n = 256 << 20
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(n, dtype=torch.uint8, device=dev)
        fns = (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True)))

        def rate(fn):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(4):
                fn()
            b.record()
            b.synchronize()
            return 4 * n / (a.elapsed_time(b) / 1e3) / 1e9

        out = {}
        for name, fn in fns:
            fn()
            torch.cuda.synchronize()
            alone = None
            for r in range(world):  # one rank at a time
                barrier()
                if r == rank:
                    alone = rate(fn)
            barrier()
            out[name] = alone
            out[name + "_all_ranks_at_once"] = rate(fn)
        del h, d
        return out

    def zero3_max_batch() -> int:
        """strategy.cpp:116-137 with a measured activation coefficient, and the
        capacity reduced by what this engine really keeps resident beyond the
        reference's persistent estimate (the reference counts optimizer state as
        6 x the grad bytes; the engine also keeps fp32 masters, gathered-layer
        and peer-visible slots), so the chosen batch actually fits."""
        plan = S.StrategyPlan(S.StrategyKind.Zero3)
        shm = bcast(f"fcdp_probe_{uuid.uuid4().hex[:12]}" if rank == 0 else None)
        tr = FcdpTrainer(mc, topo, plan, rank=rank, world_size=world, device=local, shm_name=shm,
                         batch_per_gpu=1, seq_len=seq, nic_pacing=False, timeout_s=args.engine_timeout)
        x, y = synthetic_batch(mc.vocab, 1, seq, 0x5EED, 0, rank, device=dev)
        tr.step(x, y)
        tr.sync()
        torch.cuda.synchronize()
        free, total = torch.cuda.mem_get_info(dev)
        engine_bytes = (total - free) - torch.cuda.memory_reserved(dev)  # outside torch's allocator
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        tr.step(x, y)
        tr.sync()
        torch.cuda.synchronize()
        act = max(torch.cuda.max_memory_allocated(dev) - base, 1)
        model = tr.model
        tr.close()
        del tr
        torch.cuda.empty_cache()
        L = model.num_layers()
        for lyr in model.layers:
            lyr.activation_bytes_per_sample = act // L
        cap = torch.cuda.get_device_properties(dev).total_memory
        ref_persistent = S.memory_footprint(plan, model, topo).gpu_persistent_bytes
        extra = max(0, engine_bytes - ref_persistent)
        b, oom = S.max_feasible_batch(plan, model, topo, max(cap - extra, 1))
        b = int(min(b, 256)) if not oom else 1
        measured_act[0] = int(max_over_ranks(float(act // L)))
        b = int(max_over_ranks(-b) * -1) if world > 1 else b
        if rank == 0:
            print(f"[bench] ZeRO-3 max batch {b}: activation {act / 2**30:.2f} GiB per sample, engine resident "
                  f"{engine_bytes / 2**30:.1f} GiB vs reference persistent {ref_persistent / 2**30:.1f} GiB",
                  file=sys.stderr, flush=True)
        probe_info.update({"zero3_max_batch": b, "activation_bytes_per_sample": act, "capacity_reduction": extra,
                           "engine_resident_bytes": engine_bytes, "reference_persistent_bytes": ref_persistent})
        return b

    measured_act = [None]  # per layer per sample, from the probe (feeds every run's tau projection)
    probe_info = {}

    capacity = torch.cuda.get_device_properties(dev).total_memory

    def measure(strategy: str, steps: int, warmup: int, timing: bool, e2e_steps: int, tau: float = 0.0,
                stats: bool = None):
        plan = S.StrategyPlan(S.StrategyKind.from_string(strategy), tau=tau)
        shm = bcast(f"fcdp_bench_{uuid.uuid4().hex[:12]}" if rank == 0 else None)
        tr = FcdpTrainer(mc, topo, plan, rank=rank, world_size=world, device=local, shm_name=shm,
                         batch_per_gpu=args.batch, seq_len=seq, nic_pacing=not args.no_pacing, lr=1e-4,
                         use_copy_engine=args.copy_engine, timeout_s=args.engine_timeout,
                         gpu_capacity_bytes=(capacity - probe_info.get("capacity_reduction", 0)) if tau > 0 else 0,
                         activation_bytes_per_sample=measured_act[0])
        batches = [synthetic_batch(mc.vocab, args.batch, seq, 0x5EED, i, rank, device=dev)
                   for i in range(warmup + steps)]
        for i in range(warmup):
            tr.step(*batches[i])
        tr.sync()
        torch.cuda.synchronize()
        barrier()
        tr.engine.reset_counters()
        tr.engine.kernel_stats(reset=True)
        # the timed region runs without per-kernel event timing (the kernel
        # statistics come from a separate pass below), so the headline carries
        # no instrumentation and ZeRO-3 / FCDP are timed the same way
        tr.engine.set_timing(False)
        barrier()
        sampler = ClockSampler(min(world, ndev)) if (rank == 0 and timing) else None
        if sampler:
            sampler.start()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        e0, e1 = evs[0], evs[-1]
        from paper_2602_06499_b200._capi import lib as _lib
        _lib().fcdp_model_kernel_launches(1)  # count the driving-model kernels of the timed region
        e0.record(tr.stream)
        for i in range(steps):
            loss = tr.step(*batches[warmup + i])
            evs[i + 1].record(tr.stream)
        tr.sync()
        torch.cuda.synchronize()
        barrier()
        clocks = sampler.stop() if sampler else None
        ms = max_over_ranks(e0.elapsed_time(e1))
        per_step = [round(evs[i].elapsed_time(evs[i + 1]), 3) for i in range(steps)]
        counters = tr.engine.counters()
        numa = tr.engine.numa()
        loss_v = float(loss.item())
        launches = tr.engine.kernel_stats(reset=True)  # launch counts of the timed region
        model_launches = int(_lib().fcdp_model_kernel_launches(1))
        path_launches = sum(launches[k]["launches"] for k in tr.engine.KERNEL_CLASSES)
        gpu_launches = {"total": path_launches + model_launches, "path": path_launches, "model": model_launches}
        kst, kst_steps = None, 0
        if timing if stats is None else stats:
            # kernel statistics pass: CUDA events around every engine launch
            kst_steps = min(steps, 5)
            tr.engine.kernel_stats(reset=True)
            tr.engine.set_timing(True)
            for i in range(kst_steps):
                tr.step(*batches[warmup + i])
            tr.sync()
            torch.cuda.synchronize()
            kst = tr.engine.kernel_stats(reset=True)
            tr.engine.set_timing(False)
            barrier()
        # per-node inter-group bytes per step (sum over the node's ranks), from the NIC counters
        node_tx = {k: sum_over_ranks(counters[k]) / N / steps for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs",
                                                                       "nic_tx_grad_sync")}
        cache = {k: sum_over_ranks(counters[k]) / N / steps for k in ("cache_h2d", "cache_d2h")}
        vol = S.comm_volume(plan, tr.model, topo, warmup + steps)
        e2e = None
        if e2e_steps:
            host = [synthetic_batch(mc.vocab, args.batch, seq, 0x5EED, 10_000 + i, rank, pin=True)
                    for i in range(e2e_steps)]
            tr.sync()
            barrier()
            h2d = sum(x.numel() * x.element_size() + y.numel() * y.element_size() for x, y in host[:1])
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(tr.stream)
            for x, y in host:
                with torch.cuda.stream(tr.stream):
                    xd = x.to(dev, non_blocking=True)
                    yd = y.to(dev, non_blocking=True)
                l = tr.step(xd, yd)
                l.item()  # device -> host read of the step's result
            f1.record(tr.stream)
            tr.sync()
            torch.cuda.synchronize()
            barrier()
            ems = max_over_ranks(f0.elapsed_time(f1))
            e2e = {"value": world * args.batch * seq * e2e_steps / (ems / 1e3), "unit": "tokens/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4, "steps": e2e_steps}
        tr.close()
        del tr
        torch.cuda.empty_cache()
        return {"ms": ms, "per_step": per_step, "counters": counters, "kernels": kst, "kst_steps": kst_steps,
                "gpu_launches": gpu_launches,
                "clocks": clocks, "loss": loss_v, "node_tx": node_tx, "cache": cache, "vol": vol, "e2e": e2e,
                "numa": numa}

    pcie = pcie_peak()
    if args.batch <= 0:
        args.batch = zero3_max_batch()
    if args.strategy not in ("fcdp", "fcdp-comm"):
        args.tau = 0.0
    main_run = measure(args.strategy, args.steps, args.warmup, True, 0 if args.no_e2e else args.steps, args.tau)
    tau_run = None
    if args.tau_variant >= 0 and args.strategy in ("fcdp", "fcdp-comm") and args.tau_variant != args.tau:
        tau_run = measure(args.strategy, args.zero3_steps, 2, False, 0, args.tau_variant, stats=True)
    z3 = None
    if not args.no_zero3 and args.strategy != "zero3":
        z3 = measure("zero3", args.zero3_steps, 2, False, 0)

    zpp = None
    if args.zeropp and args.strategy != "zeropp":
        zpp = measure("zeropp", args.zero3_steps, 2, False, 0)
    mics = None
    if args.mics and args.strategy != "mics":
        mics = measure("mics", args.zero3_steps, 2, False, 0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded: 1 warm-up + 3 timed full steps of the path on the C++ CPU executor
        r, why = cpu_path_sample(args, mc, N, g, seq, 3, 1, capacity)
        if r is None:
            cpu = {"value": None, "unit": "tokens/s", "unavailable": why}
        else:
            cpu = {"value": r["value"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
                   "sample": r["sample"], "ms_per_step": r["ms_per_step"], "host_GBps": r["host_GBps"],
                   "control_plane": control_plane_timing(mc, args.strategy, N, g)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    tokens_per_step = world * args.batch * seq
    ms_step = main_run["ms"] / args.steps
    value = tokens_per_step / (ms_step / 1e3)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    from paper_2602_06499_b200.engine import Engine as _E
    allst = main_run["kernels"]
    ks = max(main_run["kst_steps"], 1)  # steps of the kernel-statistics pass
    kst = {k: v for k, v in allst.items() if k in _E.KERNEL_CLASSES}
    cst = {k: v for k, v in allst.items() if k in _E.COPY_CLASSES}
    dom = max(kst, key=lambda k: kst[k]["ms"]) if any(v["ms"] for v in kst.values()) else "adamw"
    d = kst[dom]
    per_launch_bytes = d["alg_bytes"] / max(d["launches"], 1)
    per_launch_ms = d["ms"] / max(d["timed_launches"], 1)
    nvlink_bound = d.get("link_bytes", 0) > 0 and g > 1
    if nvlink_bound:
        # an intra-node gather / pull-reduce: bounded by NVLink ingress, not HBM
        link_per_launch = d["link_bytes"] / max(d["launches"], 1)
        achieved = link_per_launch / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else None
        pk, why = nvlink_peak()
        peak, unit_peak, src = pk, "GB/s", why + "; achieved = NVLink ingress bytes / launch time"
    else:
        achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9 if per_launch_ms > 0 else None
        peak, unit_peak, src = hbm, "GB/s", "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    roofline = {"bound": "nvlink" if nvlink_bound else "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": unit_peak, "frac": (achieved / peak) if (achieved and peak) else None,
                # the committed ncu capture is the default N=1 GPT-2 run; other configs have other launch sizes
                "traffic": (ncu_traffic("adamw_fused_rs" if (dom == "adamw" and world == 1) else dom)
                            if (not nvlink_bound and world == 1 and args.preset == "gpt2-1.3b") else None),
                "alg_bytes_per_launch": per_launch_bytes,
                "ms_per_launch": per_launch_ms, "peak_source": src,
                "share_of_step": (d["ms"] / ks) / ms_step if ms_step else None,
                # north_star's nominal denominators (B200: ~8 TB/s HBM3e, 900 GB/s NVLink per direction)
                "peak_nominal": 900.0 if nvlink_bound else 8000.0,
                "frac_of_nominal": (achieved / (900.0 if nvlink_bound else 8000.0)) if achieved else None}
    if per_launch_bytes < 64e6:
        # a few MB per launch (PEFT trainable slices): launch latency, not bandwidth, bounds it
        roofline["note"] = f"{per_launch_bytes / 1e6:.1f} MB per launch: launch-latency regime"
    elif dom == "adamw" and world == 1:
        if os.environ.get("FCDP_OPT_STREAM") == "rs":
            roofline["note"] = ("G = 1 fused reduce-scatter + AdamW beside the backward GEMMs (FCDP_OPT_STREAM=rs, one "
                                "CTA per SM): a live launch spans the GEMMs it overlaps; isolated = full grid alone")
        else:
            roofline["note"] = ("G = 1 fused reduce-scatter + AdamW on the compute stream after each layer's backward "
                                "(live = CUDA events around each launch in the step); isolated = the same launch alone")
    elif dom in ("adamw", "rs_slice"):
        # the per-layer update / reduce-scatter runs on its own stream beside the
        # backward GEMMs of the next layers, off the compute stream's critical path;
        # its live duration includes waiting for SMs the GEMM CTAs hold
        roofline["note"] = ("live = CUDA events around each launch while it shares the GPU with the concurrent "
                            "backward GEMMs (off the critical path); isolated = the same launch alone")
    if roofline["bound"] == "hbm":
        iso = isolated_rate(dom, per_launch_bytes, mc.dtype_bytes, dev, fused_adam=(world == 1))
        if iso:
            iso["frac"] = iso["achieved"] / peak if peak else None
            roofline["isolated"] = iso
    gpu_launches = main_run["gpu_launches"]["total"]
    gpu_launches_detail = {k: v for k, v in main_run["gpu_launches"].items() if k != "total"}
    gpu_launches_detail["note"] = ("libfcdp kernels launched in the timed region: path = the engine's "
                                   "(gather / RS / update / copies), model = the driving model's (LayerNorm, "
                                   "bias grads, GELU, cross-entropy, RoPE, SwiGLU, strided copies)")
    ag = {"fcdp_fwd": main_run["node_tx"]["nic_tx_fwd_ag"], "fcdp_bwd": main_run["node_tx"]["nic_tx_bwd_ag"],
          "fcdp_rs": main_run["node_tx"]["nic_tx_rs"],
          "oracle_fcdp_fwd": main_run["vol"].fwd_ag_inter, "oracle_fcdp_bwd": main_run["vol"].bwd_ag_inter}
    if z3:
        ag.update({"zero3_fwd": z3["node_tx"]["nic_tx_fwd_ag"], "zero3_bwd": z3["node_tx"]["nic_tx_bwd_ag"],
                   "oracle_zero3": z3["vol"].fwd_ag_inter + z3["vol"].bwd_ag_inter})
        tot_z = ag["zero3_fwd"] + ag["zero3_bwd"]
        ag["eliminated_frac"] = (1 - (ag["fcdp_fwd"] + ag["fcdp_bwd"]) / tot_z) if tot_z else None
    # Step-level link roofline (N > 1): the NIC bytes a node must move per step at
    # the preset's bandwidth, against the measured step (costmodel.cpp:100-129 shape).
    link_bound = None
    if N > 1:
        nic_b = sum(main_run["node_tx"][k] for k in ("nic_tx_fwd_ag", "nic_tx_bwd_ag", "nic_tx_rs", "nic_tx_grad_sync"))
        bw = topo.inter_node.bandwidth_bytes_per_s
        t_nic = nic_b / bw * 1e3
        link_bound = {"nic_bytes_per_node_per_step": nic_b, "nic_gbs": bw / 1e9, "nic_time_ms": t_nic,
                      "step_ms": ms_step, "frac": t_nic / ms_step if ms_step else None}
    # host-link copies (FCDP-Cache and NIC staging): achieved GB/s of the copies
    # themselves (bytes / their CUDA-event durations) against the PCIe rate
    # measured in this run with every rank copying at once
    def copy_fracs(stats, nsteps):
        out = {}
        for k, v in stats.items():
            if k not in _E.COPY_CLASSES or not v["launches"]:
                continue
            gbs = v["alg_bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None
            peak_c = pcie["d2h"] if k.endswith("d2h") else pcie["h2d"]
            out[k] = {"bytes_per_step": v["alg_bytes"] / nsteps, "copies_per_step": v["launches"] / nsteps,
                      "GBps": gbs, "pcie_peak_gbps": peak_c, "frac": gbs / peak_c if gbs else None}
        return out

    copies = copy_fracs(cst, ks)
    kernels = {k: {"launches_per_step": v["launches"] / ks, "ms_per_step": v["ms"] / ks,
                   "GBps": (v["alg_bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] else None} for k, v in kst.items()}
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if mc.dtype_bytes == 2 else "fp32",
        "data": "synthetic (counter-based token ids, random-init weights of the named architecture)",
        "config": workload_config(args, mc, N, g, world, seq),
        "e2e": main_run["e2e"], "gpu_launches": gpu_launches, "gpu_launches_detail": gpu_launches_detail,
        "roofline": roofline, "link_bound": link_bound,
        "copies": copies, "pcie_peak_gbps": pcie,
        "cpu_baseline": cpu, "clocks": main_run["clocks"],
        "ag_inter_bytes_per_step_per_node": ag,
        "zero3": ({"tokens_per_s": tokens_per_step / (z3["ms"] / z3_steps(args) / 1e3), "ms_per_step": z3["ms"] / z3_steps(args)}
                  if z3 else None),
        "zeropp": ({"tokens_per_s": tokens_per_step / (zpp["ms"] / args.zero3_steps / 1e3),
                    "ms_per_step": zpp["ms"] / args.zero3_steps,
                    "ag_inter_fwd_bwd": [zpp["node_tx"]["nic_tx_fwd_ag"], zpp["node_tx"]["nic_tx_bwd_ag"]]}
                   if zpp else None),
        "mics": ({"tokens_per_s": tokens_per_step / (mics["ms"] / args.zero3_steps / 1e3),
                  "ms_per_step": mics["ms"] / args.zero3_steps,
                  "ag_inter_fwd_bwd": [mics["node_tx"]["nic_tx_fwd_ag"], mics["node_tx"]["nic_tx_bwd_ag"]],
                  "grad_sync_bytes_per_node": mics["node_tx"]["nic_tx_grad_sync"]} if mics else None),
        "cache_bytes_per_step_per_node": main_run["cache"],
        "fcdp_variant": ({"tau": args.tau_variant, "tokens_per_s": tokens_per_step / (tau_run["ms"] / args.zero3_steps / 1e3),
                                "ms_per_step": tau_run["ms"] / args.zero3_steps, "cache": tau_run["cache"],
                                "copies": (copy_fracs(tau_run["kernels"], max(tau_run["kst_steps"], 1))
                                           if tau_run["kernels"] else None),
                                "vs_zero3": ((z3["ms"] / z3_steps(args)) / (tau_run["ms"] / args.zero3_steps)
                                             if z3 else None),
                                "ag_inter_fwd_bwd": [tau_run["node_tx"]["nic_tx_fwd_ag"], tau_run["node_tx"]["nic_tx_bwd_ag"]]}
                               if tau_run else None),
        "host_numa": main_run["numa"], "kernels": kernels,
        "batch_probe": probe_info or None,
        "kernel_stats_pass": {"steps": ks, "note": "per-kernel CUDA-event timing (kernels, roofline, copies) comes "
                                                   "from this many extra steps after the timed region; the timed "
                                                   "region itself runs uninstrumented"},
        "loss": main_run["loss"], "ms_each_step_rank0": main_run["per_step"],
    }
    if shared:  # several ranks per GPU: checks the N-rank flow, not a throughput number
        line["config"]["ranks_per_gpu"] = world / ndev
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def z3_steps(args):
    return args.zero3_steps


if __name__ == "__main__":
    main()
