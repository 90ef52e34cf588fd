"""Concurrent pinned-host <-> GPU bandwidth, 1..N GPUs at once (one process per GPU).

    python -m torch.distributed.run --nproc-per-node N tools/pcie_probe.py
Rank 0 prints per-GPU GB/s for D2H, H2D and both directions at once, plus the
NVLink peer copy bandwidth GPU0 <- GPU1 when N >= 2.
"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist


def bw(fn, nbytes, reps=8):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return nbytes * reps / dt / 1e9


def registered(n, kind, tag):
    """Host buffer from a POSIX shm segment or an anonymous mapping, registered
    with cudaHostRegister (what the engine's host-cache tier uses)."""
    import mmap
    if kind == "shm":
        path = f"/dev/shm/pcie_probe_{os.getpid()}_{tag}"
        fd = os.open(path, os.O_CREAT | os.O_RDWR, 0o600)
        os.ftruncate(fd, n)
        m = mmap.mmap(fd, n)
        os.close(fd)
        os.unlink(path)
    else:
        m = mmap.mmap(-1, n)
    t = torch.frombuffer(m, dtype=torch.uint8)
    t.fill_(0)
    err = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), n, 1)
    assert int(err) == 0, err
    registered.keep.append(m)
    return t


registered.keep = []


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "torch"
    dist.init_process_group("gloo")
    r, w = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(r)
    n = 512 << 20
    if src == "torch":
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    else:
        h, h2 = registered(n, src, "a"), registered(n, src, "b")
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    res["d2h"] = bw(lambda: h.copy_(d, non_blocking=True), n)
    res["h2d"] = bw(lambda: d.copy_(h, non_blocking=True), n)

    def both():
        with torch.cuda.stream(s1):
            h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2):
            d2.copy_(h2, non_blocking=True)
    res["bidir_each"] = bw(both, n)
    out = [None] * w
    dist.all_gather_object(out, res)
    if r == 0:
        print(json.dumps({"world": w, "src": src, "per_gpu": out}))
    dist.barrier()


if __name__ == "__main__":
    main()
