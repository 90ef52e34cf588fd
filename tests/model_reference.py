"""Plain single-process torch fp32 CPU training of the driving model (test
infrastructure): the model-math reference that the B200 trainer and the C++
CPU executor are compared against (loss, reduced gradients, updated masters).
The tolerances are stated in tests/test_trainer_gpu.py and DESIGN.md section 5."""
import numpy as np
import torch


def cpu_reference(cfg):
    """Single-process fp32 torch training of the same model on the CPU."""
    from oracle import oracle as O
    from paper_2602_06499_b200.driving_model import PRESETS, layer_forward
    from paper_2602_06499_b200.trainer import synthetic_batch
    mc = PRESETS[cfg["preset"]]
    defs = mc.layer_defs()
    eb = mc.dtype_bytes
    flats = []
    for l, d in enumerate(defs):
        nat = O.init_natural(d.numel, eb, cfg["seed"], l, d.init_ranges())
        w = O.bf16_to_f32(nat) if eb == 2 else nat.astype(np.float32)
        flats.append(torch.from_numpy(w.copy()))
    params = []
    for l, d in enumerate(defs):
        p = {}
        for t in d.tensors:
            v = flats[l][d.offsets[t.name]:d.offsets[t.name] + t.numel].view(t.shape).clone()
            v.requires_grad_(t.trainable)
            p[t.name] = v
        params.append(p)
    opt_state = {}
    world = cfg["N"] * cfg["g"]
    losses, grads, masters = [], [], []
    w0 = [flats[l].clone() for l in range(len(defs))]
    b1, b2, eps, lr, wd = 0.9, 0.95, 1e-8, cfg["lr"], cfg["wd"]
    for step in range(1, cfg["steps"] + 1):
        total = 0.0
        for r in range(world):
            x, y = synthetic_batch(mc.vocab, cfg["batch"], mc.seq, cfg["seed"], step, r)
            h = None
            for l, d in enumerate(defs):
                h = layer_forward(mc, d, params[l], h, x, y)
            (h / world).backward()
            total += float(h)
        losses.append(total / world)
        grads.append([_flat(d, {n: (params[l][n].grad if params[l][n].grad is not None
                                    else torch.zeros_like(params[l][n])) for n in params[l]})
                      for l, d in enumerate(defs)])
        with torch.no_grad():
            for l, d in enumerate(defs):
                for t in d.tensors:
                    if not t.trainable:
                        continue
                    w = params[l][t.name]
                    m, v = opt_state.setdefault((l, t.name), (torch.zeros_like(w), torch.zeros_like(w)))
                    gr = w.grad
                    m.mul_(b1).add_((1 - b1) * gr)
                    v.mul_(b2).add_((1 - b2) * gr * gr)
                    mh = m / (1 - b1 ** step)
                    vh = v / (1 - b2 ** step)
                    w.sub_(lr * (mh / (vh.sqrt() + eps) + wd * w))
                    w.grad = None
        masters.append([_flat(d, params[l]) for l, d in enumerate(defs)])
    return {"losses": losses, "grads": grads, "masters": masters, "w0": [w.numpy() for w in w0]}


def _flat(d, tensors):
    out = np.zeros(d.numel, np.float32)
    for t in d.tensors:
        out[d.offsets[t.name]:d.offsets[t.name] + t.numel] = tensors[t.name].detach().reshape(-1).float().numpy()
    return out


def trainable(d, eb, natural):
    """Mask-order compaction of a natural fp32 layer vector (chunk-granular mask)."""
    V = 16 // eb
    m = d.chunk_mask(eb).astype(bool)
    return natural.reshape(-1, V)[m].reshape(-1)


def gathered(cfg, res, key, step, layer, n):
    """Concatenate the ranks' fp32 shards of a trainable portion in global shard
    order (shard r = j*N + n lives on rank n*g + j) -> the first n elements."""
    N, g = cfg["N"], cfg["g"]
    parts = [res[(r % N) * g + r // N][key][step][layer] for r in range(N * g)]
    return np.concatenate(parts)[:n]


def compare(cfg, res, ref, fp32):
    """res[rank]["grads"|"masters"][step][layer] = that rank's fp32 shard."""
    from paper_2602_06499_b200.driving_model import PRESETS
    mc = PRESETS[cfg["preset"]]
    eb = mc.dtype_bytes
    report = []
    for step in range(cfg["steps"]):
        for l, d in enumerate(mc.layer_defs()):
            gr = trainable(d, eb, ref["grads"][step][l])
            if gr.size == 0:
                continue
            gg = gathered(cfg, res, "grads", step, l, gr.size)
            wr = trainable(d, eb, ref["masters"][step][l])
            wg = gathered(cfg, res, "masters", step, l, wr.size)
            w0 = trainable(d, eb, ref["w0"][l])
            ge = np.abs(gg - gr)
            we = np.abs(wg - wr)
            row = dict(step=step + 1, layer=l, grad_max_err=float(ge.max()), grad_max_ref=float(np.abs(gr).max()),
                       grad_l2_rel=float(np.linalg.norm(ge) / max(np.linalg.norm(gr), 1e-30)),
                       master_max_err=float(we.max()),
                       upd_l2_rel=float(np.linalg.norm(wg - wr) / max(np.linalg.norm(wr - w0), 1e-30)))
            report.append(row)
            if fp32:
                assert ge.max() <= 1e-4 * np.abs(gr).max(), row
                within = we <= 1e-6 + 1e-4 * np.abs(wr)
                assert within.mean() >= 0.999, (row, float(within.mean()))
                assert we.max() <= 2 * cfg["lr"] * (step + 1), row
            else:
                assert row["grad_l2_rel"] <= 5e-2, row
                assert row["upd_l2_rel"] <= 0.25, row
    worst = {k: max(r[k] for r in report) for k in ("grad_l2_rel", "upd_l2_rel")}
    print(f"[parity] {cfg['preset']} {cfg['strategy']} {cfg['N']}x{cfg['g']}: worst grad l2 rel "
          f"{worst['grad_l2_rel']:.3e}, worst update l2 rel {worst['upd_l2_rel']:.3e}")
    return report
