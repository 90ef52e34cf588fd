"""One rank of an engine parity job (launched by tests/test_engine_gpu.py).

Runs K iterations of a shardsim program on the B200 engine with a synthetic
compute callback whose gradients are an exact function of the gathered layer
and the rank, and dumps everything the CPU oracle needs to re-derive.
"""
import json
import os
import pickle
import sys
os_env_set = __import__('os').environ.setdefault('CUDA_DEVICE_MAX_CONNECTIONS', '32')
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def grad_coeff(rank: int) -> float:
    return (1 + rank) / 8.0


def main():
    cfg = json.loads(sys.argv[1])
    import torch
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.engine import Engine, BWD
    from paper_2602_06499_b200.tensors import device_view
    from oracle import oracle as O
    from tests.engine_oracle import scope_nodes

    rank, world = cfg["rank"], cfg["world"]
    N, g = cfg["N"], cfg["g"]
    ndev = torch.cuda.device_count()
    dev_idx = rank % ndev
    torch.cuda.set_device(dev_idx)
    device = torch.device("cuda", dev_idx)
    eb = cfg["eb"]
    V = 16 // eb
    dtype = torch.bfloat16 if eb == 2 else torch.float32
    masks = [np.array(m, np.uint8) for m in cfg["masks"]]
    layers = []
    for i, (E, m) in enumerate(zip(cfg["params"], masks)):
        frac = float(int(m.sum()) * V) / E
        layers.append(S.LayerSpec(i, E, frac))
    model = S.ModelSpec(layers, eb)
    topo = S.make_topology(N, g, inter_preset=cfg.get("inter", "ib100-rdma-measured"))
    plan = S.StrategyPlan(S.StrategyKind.from_string(cfg["strategy"]), tau=cfg.get("tau", 0.0))
    eng = Engine(model, topo, plan, rank=rank, world_size=world, device=dev_idx, shm_name=cfg["shm"],
                 chunk_masks=masks, nic_pacing=cfg.get("pacing", False),
                 use_copy_engine=cfg.get("use_ce", False), timeout_s=120.0)
    eng.init_params(cfg["seed"], [[(0, E, 0, 0.05)] for E in cfg["params"]])
    eng.set_adam(lr=1e-2, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.01)
    eng.set_keep_grad(True)  # the fused G = 1 path also writes the fp32 gradient shard (read_grad)
    stream = torch.cuda.ExternalStream(eng.compute_stream(), device=device)
    captures = []
    c = grad_coeff(rank)

    def compute(kind, layer, w, gptr, s):
        E = cfg["params"][layer]
        with torch.cuda.stream(stream):
            W = device_view(w, E, dtype, device)
            captures.append((kind, layer, W.clone()))
            if kind == BWD and gptr:
                G = device_view(gptr, E, dtype, device)
                G.copy_((W.float() * c).to(dtype))

    eng.set_compute(compute)
    if cfg.get("trace"):
        eng.set_trace(True)
    if cfg.get("nic_log"):
        eng.set_nic_log(True)
    states = S.init_param_states(model)
    dumps = []
    mut = cfg.get("mutate")
    for it in range(1, cfg["iters"] + 1):
        cap = cfg.get("capacity", 0)
        if mut and mut["kind"] == "capacity_mismatch" and rank == 1:
            cap = mut["capacity"]
        prog = S.build_iteration(plan, model, topo, states, it, gpu_capacity_bytes=cap)
        if mut and it == mut["it"]:
            # SPEC.md:389-409 mutation harness, applied to the EXECUTED program
            evs = prog.events
            last_fwd = max(e.id for e in evs if e.kind == S.EventKind.ComputeFwd)
            if mut["kind"] == "drop_d2h":  # the layer's FCDP-Cache store is lost
                drop = [e.id for e in evs if e.kind == S.EventKind.D2H and e.layer == mut["layer"]]
                prog = prog.without(drop, model.num_layers())
            elif mut["kind"] == "bwd_ag_inter":  # backward reload replaced by an inter-node gather
                h2d = next(e for e in evs if e.kind == S.EventKind.H2D and e.layer == mut["layer"] and e.id > last_fwd)
                intra = next(e for e in evs if e.kind == S.EventKind.AgIntra and e.layer == mut["layer"]
                             and e.id > last_fwd)
                ag = S.Event(h2d.id, S.EventKind.AgInter, h2d.layer, S.ParamSet.All, h2d.bytes_total, h2d.deps)
                prog = prog.without([intra.id], model.num_layers(), replace={h2d.id: ag})
        eng.reset_counters()
        eng.barrier()
        if mut and it == mut["it"]:
            errs = []
            try:
                eng.run_stepwise(prog, states) if cfg.get("stepwise") else eng.run(prog, states)
                eng.sync()
            except Exception as ex:  # noqa: BLE001 - recorded for the test
                errs.append((type(ex).__name__, getattr(ex, "args", [None])[0], str(ex)))
            try:  # the engine must refuse to continue after a failed program
                eng.run(prog, states)
            except Exception as ex:  # noqa: BLE001
                errs.append((type(ex).__name__, getattr(ex, "args", [None])[0], str(ex)))
            with open(os.path.join(cfg["out"], f"rank{rank}.pkl"), "wb") as f:
                pickle.dump({"errors": errs}, f)
            eng.close()
            return
        states = eng.run_stepwise(prog, states) if cfg.get("stepwise") else eng.run(prog, states)
        eng.sync()
        eng.barrier()
        torch.cuda.synchronize()
        d = {"it": it, "captures": [(k, l, t.view(torch.uint8).cpu().numpy() if t.dtype != torch.uint8 else t.cpu().numpy())
                                     for k, l, t in captures],
             "counters": eng.counters(), "host": {}, "grad": {}, "master": {}, "shard_t": {}, "shard_f": {},
             "retained": prog.layer_flags(model.num_layers())}
        if cfg.get("nic_log"):
            d["nic_log"] = eng.nic_log()
        if cfg.get("trace"):
            tr = eng.trace(prog)
            d["trace"] = [(e.id, int(e.kind), e.layer, list(e.deps), b, t) for e, b, t in tr]
        captures.clear()
        for l in range(model.num_layers()):
            geo = O.geom(len(masks[l]), masks[l], scope_nodes(cfg), g)
            j = rank % g
            st, sf = geo.slice_t * 16, geo.slice_f * 16
            d["host"][l] = (eng.read_host_cache(l, False, st), eng.read_host_cache(l, True, sf))
            d["grad"][l] = eng.read_grad(l, geo.shard_t * V)
            d["master"][l] = eng.read_master(l, geo.shard_t * V)
            d["shard_t"][l] = eng.read_shard(l, False, geo.shard_t * 16)
            d["shard_f"][l] = eng.read_shard(l, True, geo.shard_f * 16)
        dumps.append(d)
    with open(os.path.join(cfg["out"], f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(dumps, f)
    eng.barrier()
    eng.close()


if __name__ == "__main__":
    main()
