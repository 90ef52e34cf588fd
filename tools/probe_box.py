"""Probe the GPU box: host cores, RAM, /dev/shm, PCIe H2D/D2H pinned bandwidth, P2P access."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["meminfo"] = [l.strip() for l in f.readlines()[:5]]
out["shm"] = subprocess.run(["df", "-h", "/dev/shm"], capture_output=True, text=True).stdout
out["ulimit_l"] = subprocess.run(["bash", "-c", "ulimit -l"], capture_output=True, text=True).stdout.strip()
out["ngpu"] = torch.cuda.device_count()
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
n = torch.cuda.device_count()
out["p2p"] = [[torch.cuda.can_device_access_peer(i, j) if i != j else True for j in range(n)] for i in range(n)]
def bw(nbytes, dev, h2d):
    torch.cuda.set_device(dev)
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for _ in range(3):
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
    e.record(); torch.cuda.synchronize()
    return nbytes * 5 / (s.elapsed_time(e) / 1e3) / 1e9
out["h2d_gbs_1gpu"] = bw(1 << 30, 0, True)
out["d2h_gbs_1gpu"] = bw(1 << 30, 0, False)
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
