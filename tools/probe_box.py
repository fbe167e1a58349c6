"""One-off probe of the GPU box: host RAM/cores, PCIe link, pinned copy bandwidth."""
import os, subprocess, time, json
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = sh("head -3 /proc/meminfo")
out["lscpu"] = sh("lscpu | head -20")
out["numa"] = sh("numactl -H 2>/dev/null || ls /sys/devices/system/node")
out["smi"] = sh("nvidia-smi -q | grep -i -A3 -E 'PCIe Generation|Link Width|Bus Id' | head -40")
out["topo"] = sh("nvidia-smi topo -m")
out["ulimit_l"] = sh("ulimit -l")
dev = torch.device("cuda")
res = {}
for mb in (1, 16, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for direction in ("h2d", "d2h"):
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        s.record()
        for _ in range(reps):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e.record(); torch.cuda.synchronize()
        res[f"{direction}_{mb}MB_GBs"] = n * reps / (s.elapsed_time(e) * 1e-3) / 1e9
# bidirectional
n = 1024 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
res["bidir_total_GBs"] = 2 * 5 * n / dt / 1e9
# pinned alloc time for 16 GiB
t = time.perf_counter()
big = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True)
res["pin_16GiB_s"] = time.perf_counter() - t
out["copy"] = res
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps(res, indent=1))
print(out["meminfo"], out["nproc"])
