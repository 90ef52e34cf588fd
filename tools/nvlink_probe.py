"""NVLink evidence for the intra-node kernels (run with 2 GPUs: gpurun --gpus 2).

    python tools/nvlink_probe.py [--mb 512] [--out gpurun_out/nvlink_probe.json]

One process, two GPUs, peer access enabled - so the whole run can sit under
ncu (no cross-rank waits to replay):

  * peer copy (copy engine, cudaMemcpyPeer via torch) GPU1 -> GPU0: the
    measured NVLink peak per direction this box gives (the roofline
    denominator bench.py uses instead of a hard-coded figure);
  * the engine's intra-node all-gather kernel (expand_kernel / concat, the
    AgInter / AgIntra unpack) on GPU0 pulling g-1 of g slices from GPU1;
  * the intra-node reduce-scatter kernel (rs_dense_kernel) on GPU0 summing
    g natural gradients of which g-1 live on GPU1.

Achieved NVLink GB/s = bytes that crossed NVLink / CUDA-event time.  Under
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,\\
        nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
the counter bytes per launch can be set against the algorithmic bytes.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=512, help="layer size (MB) per gather / RS launch")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="gpurun_out/nvlink_probe.json")
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2602_06499_b200 import _capi
    lib = _capi.lib()
    assert torch.cuda.device_count() >= 2, "needs 2 GPUs"
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    torch.cuda.set_device(d0)
    _capi.check(lib.fcdp_enable_peer_access(0, 1))
    _capi.check(lib.fcdp_enable_peer_access(1, 0))
    P = lambda t: C.c_void_p(t.data_ptr())
    res = {"gpus": [torch.cuda.get_device_name(0), torch.cuda.get_device_name(1)], "mb": a.mb}

    def timeit(fn, reps=a.reps):
        fn()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record()
        for i in range(reps):
            fn()
            ev[i + 1].record()
        torch.cuda.synchronize()
        return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))

    nbytes = a.mb << 20
    # (1) copy-engine peer read, both directions measured separately
    src1 = torch.zeros(nbytes, dtype=torch.uint8, device=d1)
    torch.cuda.synchronize(d1)
    dst0 = torch.empty(nbytes, dtype=torch.uint8, device=d0)
    ms = timeit(lambda: dst0.copy_(src1, non_blocking=True))
    res["peer_copy_1to0_GBps"] = nbytes / (ms / 1e3) / 1e9
    src0 = torch.empty(nbytes, dtype=torch.uint8, device=d0)
    dst1 = torch.empty(nbytes, dtype=torch.uint8, device=d1)
    with torch.cuda.device(d1):
        ms = timeit(lambda: dst1.copy_(src0, non_blocking=True))
    res["peer_copy_0to1_GBps"] = nbytes / (ms / 1e3) / 1e9

    # (2) the all-gather kernel on GPU0, g slices of which g-1 are on GPU1
    for g in (2, 4, 8):
        chunks = nbytes // 16
        chunks -= chunks % g
        mask = np.ones(chunks, np.uint8)
        lay = C.c_void_p()
        _capi.check(lib.fcdp_layout_create(chunks, mask.ctypes.data_as(C.POINTER(C.c_uint8)), 2, 1, g, C.byref(lay)))
        per = chunks // g * 16
        slices = [torch.empty(per, dtype=torch.uint8, device=d0 if j == 0 else d1) for j in range(g)]
        out = torch.empty(chunks * 16, dtype=torch.uint8, device=d0)
        ts = (C.c_void_p * g)(*[t.data_ptr() for t in slices])
        fn = lambda: _capi.check(lib.fcdp_expand(lay, ts, None, P(out), 0, None))
        ms = timeit(fn)
        remote = per * (g - 1)
        res[f"gather_g{g}"] = {"ms": ms, "nvlink_bytes": remote, "nvlink_GBps": remote / (ms / 1e3) / 1e9,
                               "hbm_bytes": 2 * chunks * 16 - remote}
        # correctness: gathered = concat of the slices
        for j, t in enumerate(slices):
            t.fill_(j + 1)
        torch.cuda.synchronize(d1)
        torch.cuda.synchronize(d0)
        fn()
        torch.cuda.synchronize()
        got = out.view(g, per)[:, ::4096].cpu()
        assert all(int(got[j].min()) == j + 1 == int(got[j].max()) for j in range(g)), "gather mismatch"
        lib.fcdp_layout_destroy(lay)
        del slices, out

    # (3) the intra-node reduce-scatter kernel on GPU0: g bf16 gradients, g-1 remote
    for g in (2, 4):
        chunks = nbytes // 16
        chunks -= chunks % g
        mask = np.ones(chunks, np.uint8)
        lay = C.c_void_p()
        _capi.check(lib.fcdp_layout_create(chunks, mask.ctypes.data_as(C.POINTER(C.c_uint8)), 2, 1, g, C.byref(lay)))
        grads = [torch.randn(chunks * 8, device=d0 if j == 0 else d1).to(torch.bfloat16) for j in range(g)]
        torch.cuda.synchronize(d1)
        gp = (C.c_void_p * g)(*[t.data_ptr() for t in grads])
        slice_chunks = chunks // g
        own = torch.empty(slice_chunks * 8, dtype=torch.float32, device=d0)
        wire = torch.empty(16, dtype=torch.uint8, device=d0)
        fn = lambda: _capi.check(lib.fcdp_rs_slice(lay, gp, 0, 0, 1.0 / g, 1, P(own), P(wire), None))
        ms = timeit(fn)
        remote = slice_chunks * 16 * (g - 1)
        res[f"rs_g{g}"] = {"ms": ms, "nvlink_bytes": remote, "nvlink_GBps": remote / (ms / 1e3) / 1e9,
                           "hbm_bytes": slice_chunks * 16 + slice_chunks * 8 * 4}
        # correctness vs torch on GPU0
        ref = sum(t[:slice_chunks * 8].to(d0).float() for t in grads) * (1.0 / g)
        torch.cuda.synchronize(d1)
        torch.cuda.synchronize(d0)
        fn()
        torch.cuda.synchronize()
        assert torch.allclose(own, ref, rtol=1e-6, atol=1e-6), "rs mismatch"
        lib.fcdp_layout_destroy(lay)
        del grads, own
    res["nvlink_peak_GBps"] = max(res["peer_copy_1to0_GBps"], res["peer_copy_0to1_GBps"])
    for k, v in res.items():
        if isinstance(v, dict) and "nvlink_GBps" in v:
            v["frac_of_peer_copy"] = v["nvlink_GBps"] / res["nvlink_peak_GBps"]
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
