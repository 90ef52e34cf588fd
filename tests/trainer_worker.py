"""One rank of a training-parity job (launched by tests/test_trainer_gpu.py)."""
import json
import os
import pickle
import sys
os_env_set = __import__('os').environ.setdefault('CUDA_DEVICE_MAX_CONNECTIONS', '32')
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    cfg = json.loads(sys.argv[1])
    import torch
    from paper_2602_06499_b200 import shardsim as S
    from paper_2602_06499_b200.driving_model import PRESETS
    from paper_2602_06499_b200.trainer import FcdpTrainer, synthetic_batch
    rank, N, g = cfg["rank"], cfg["N"], cfg["g"]
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    mc = PRESETS[cfg["preset"]]
    topo = S.make_topology(N, g)
    plan = S.StrategyPlan(S.StrategyKind.from_string(cfg["strategy"]))
    t = FcdpTrainer(mc, topo, plan, rank=rank, world_size=N * g, device=dev, shm_name=cfg["shm"],
                    batch_per_gpu=cfg["batch"], seed=cfg["seed"], nic_pacing=False, lr=cfg["lr"],
                    weight_decay=cfg["wd"])
    from oracle import oracle as O
    t.engine.set_keep_grad(True)  # read_grad after the fused G = 1 update
    V = 16 // mc.dtype_bytes
    geos = [O.geom(d.numel * mc.dtype_bytes // 16, d.chunk_mask(mc.dtype_bytes), N, g) for d in t.defs]
    losses, grads, masters = [], [], []
    for step in range(1, cfg["steps"] + 1):
        x, y = synthetic_batch(mc.vocab, cfg["batch"], mc.seq, cfg["seed"], step, rank, device=t.device)
        loss = t.step(x, y)
        t.sync()
        losses.append(float(loss.item()))
        # this rank's fp32 shard of the reduced gradient of this step and of the
        # updated master weights (global shard j*N + n of each trainable portion)
        grads.append({l: t.engine.read_grad(l, geo.shard_t * V) for l, geo in enumerate(geos) if geo.pt})
        masters.append({l: t.engine.read_master(l, geo.shard_t * V) for l, geo in enumerate(geos) if geo.pt})
    shards = {}
    for l, geo in enumerate(geos):
        shards[l] = (t.engine.read_shard(l, False, geo.shard_t * 16), t.engine.read_shard(l, True, geo.shard_f * 16))
    with open(os.path.join(cfg["out"], f"rank{rank}.pkl"), "wb") as f:
        pickle.dump({"losses": losses, "shards": shards, "grads": grads, "masters": masters}, f)
    t.engine.barrier()
    t.close()


if __name__ == "__main__":
    main()
