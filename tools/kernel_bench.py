"""Standalone timing of every data-plane kernel at the bench's layer sizes.

    python tools/kernel_bench.py [--out gpurun_out/kernel_bench.json] [--reps 20]

Each kernel is called through the C ABI (include/fcdp.h) on cuda:0 with
inputs larger than L2 (a fresh 1 GiB buffer is written between reps to
flush it), timed with CUDA events on its stream; algorithmic bytes per launch
as in DESIGN.md section 4; fraction of the MEASURED_PEAKS.json HBM copy peak.
Short enough to run under `ncu --set full`.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/kernel_bench.json")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2602_06499_b200 import _capi
    from paper_2602_06499_b200.driving_model import PRESETS
    lib = _capi.lib()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    flush = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    res = {}

    def timeit(name, fn, alg_bytes):
        ts = []
        for i in range(a.reps + 2):
            flush.fill_(i & 0xFF)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(s.elapsed_time(e))
        ms = float(np.median(ts))
        gbs = alg_bytes / (ms / 1e3) / 1e9
        res[name] = {"ms": ms, "alg_bytes": alg_bytes, "GBps": gbs, "frac_of_measured_hbm": gbs / peak}
        print(f"{name:28s} {ms:8.3f} ms  {gbs:8.1f} GB/s  {gbs / peak:6.1%}")

    def layout(mask, eb, N, g):
        out = C.c_void_p()
        m = np.ascontiguousarray(mask, np.uint8)
        _capi.check(lib.fcdp_layout_create(m.size, m.ctypes.data_as(C.POINTER(C.c_uint8)), eb, N, g, C.byref(out)))
        return out

    P = lambda t: C.c_void_p(t.data_ptr())
    # --- GPT-2 1.3B block (dense), g = 1 and a 4-way slice split (all local here)
    E = 50358272
    chunks = E * 2 // 16
    dense = layout(np.ones(chunks, np.uint8), 2, 1, 1)
    X = torch.randint(0, 255, (chunks * 16,), dtype=torch.uint8, device=dev)
    W = torch.empty_like(X)
    timeit("concat_dense_g1", lambda: _capi.check(lib.fcdp_expand(dense, (C.c_void_p * 1)(X.data_ptr()), None, P(W), 0, None)),
           2 * chunks * 16)
    # like-for-like denominator at this launch size: torch's own D2D copy (copy engine / cudaMemcpy)
    timeit("torch_copy_same_size", lambda: W.copy_(X), 2 * chunks * 16)
    d4 = layout(np.ones(chunks, np.uint8), 2, 1, 4)
    per = chunks // 4 * 16
    Xs = [X[i * per:(i + 1) * per] for i in range(4)]
    timeit("concat_dense_g4_local", lambda: _capi.check(lib.fcdp_expand(
        d4, (C.c_void_p * 4)(*[x.data_ptr() for x in Xs]), None, P(W), 0, None)), 2 * chunks * 16)
    # --- Llama-7B + LoRA block: masked expand / partition (PEFT)
    ldef = PRESETS["llama7b-lora16"].layer_defs()[1]
    mask = ldef.chunk_mask(2)
    lc = mask.size
    peft = layout(mask, 2, 1, 1)
    pt = int(mask.sum())
    T = torch.randint(0, 255, (max(pt, 1) * 16,), dtype=torch.uint8, device=dev)
    F = torch.randint(0, 255, ((lc - pt) * 16,), dtype=torch.uint8, device=dev)
    WL = torch.empty(lc * 16, dtype=torch.uint8, device=dev)
    timeit("expand_peft_all_g1", lambda: _capi.check(lib.fcdp_expand(
        peft, (C.c_void_p * 1)(T.data_ptr()), (C.c_void_p * 1)(F.data_ptr()), P(WL), 0, None)), 2 * lc * 16)
    timeit("expand_peft_frozen_g1", lambda: _capi.check(lib.fcdp_expand(
        peft, (C.c_void_p * 1)(T.data_ptr()), (C.c_void_p * 1)(F.data_ptr()), P(WL), 2, None)), 2 * (lc - pt) * 16)
    timeit("partition_peft", lambda: _capi.check(lib.fcdp_partition(peft, P(WL), P(T), P(F), None)), 2 * lc * 16)
    # --- reduce-scatter (dense, N = 1 final: bf16 grads -> scaled fp32 shard)
    G = torch.randn(E, device=dev).to(torch.bfloat16)
    own = torch.empty(E, dtype=torch.float32, device=dev)
    wire = torch.empty(E, dtype=torch.bfloat16, device=dev)
    timeit("rs_dense_g1_final", lambda: _capi.check(lib.fcdp_rs_slice(
        dense, (C.c_void_p * 1)(G.data_ptr()), 0, 0, 1.0, 1, P(own), P(wire), None)), E * 2 + E * 4)
    Gs = [G] + [torch.randn(E, device=dev).to(torch.bfloat16) for _ in range(7)]
    for gg in (2, 4, 8):
        dgb = layout(np.ones(chunks, np.uint8), 2, 1, gg)
        timeit(f"rs_dense_g{gg}_local", lambda: _capi.check(lib.fcdp_rs_slice(
            dgb, (C.c_void_p * gg)(*[x.data_ptr() for x in Gs[:gg]]), 1, 0, 1.0 / gg, 1, P(own), P(wire), None)),
            gg * (E // gg) * 2 + (E // gg) * 4)
    # 2 x 1 (N = 2): own half fp32, the other half to the wire in bf16
    d21 = layout(np.ones(chunks, np.uint8), 2, 2, 1)
    timeit("rs_dense_2x1_wire", lambda: _capi.check(lib.fcdp_rs_slice(
        d21, (C.c_void_p * 1)(G.data_ptr()), 0, 0, 0.5, 0, P(own), P(wire), None)), E * 2 + (E // 2) * 4 + (E // 2) * 2)
    # --- G = 1 fused RS + AdamW of one GPT-2 1.3B block (the engine's one-GPU launch)
    wl, ml, vl = torch.randn(E, device=dev), torch.zeros(E, device=dev), torch.zeros(E, device=dev)
    pl = torch.empty(E, dtype=torch.bfloat16, device=dev)
    cfg1 = _capi.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
    offs, cnts, ptrs = (C.c_int64 * 1)(0), (C.c_int64 * 1)(E), (C.c_void_p * 1)(G.data_ptr())
    timeit("adamw_fused_grad_block", lambda: _capi.check(lib.fcdp_adam_grad_step(
        E, C.byref(cfg1), 1.0, 1, offs, ptrs, cnts, P(wl), P(ml), P(vl), P(pl), 2, None, None)), E * 28)
    wl2 = torch.randn(E, device=dev)
    g32 = torch.randn(E, device=dev)
    timeit("adamw_block", lambda: _capi.check(lib.fcdp_adam_step(E, C.byref(cfg1), P(wl2), P(ml), P(vl), P(g32), P(pl),
                                                                 2, None)), E * 30)
    # --- inter-node finalize, N = 2
    n = E // 2
    timeit("rs_finalize_N2", lambda: _capi.check(lib.fcdp_rs_finalize(n, 2, 0, 2, P(own), P(wire), n, 0.5, P(own), None)),
           n * (4 + 2 + 4))
    # --- AdamW over the whole GPT-2 1.3B trainable arena (the bench's launch, 1x1)
    nA = 1416744960
    w = torch.randn(nA, device=dev)
    m = torch.zeros(nA, device=dev)
    v = torch.zeros(nA, device=dev)
    g = torch.randn(nA, device=dev)
    pp = torch.empty(nA, dtype=torch.bfloat16, device=dev)
    cfg = _capi.AdamConfig(1e-4, 0.9, 0.95, 1e-8, 0.0, 1)
    timeit("adamw_gpt2_1.3b_arena", lambda: _capi.check(lib.fcdp_adam_step(nA, C.byref(cfg), P(w), P(m), P(v), P(g), P(pp), 2, None)),
           nA * 30)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps({"peak_hbm_gbs": peak, "kernels": res}, indent=1))


if __name__ == "__main__":
    main()
