# One-off probe of the GPU box: host cores/RAM, pinned host-link bandwidth per direction.
import os, subprocess, time, json, torch
out = {}
out["nproc"] = os.cpu_count()
out["lscpu"] = subprocess.run("lscpu | grep -E 'Model name|Socket|NUMA node\\(s\\)|Thread'", shell=True, capture_output=True, text=True).stdout
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
out["smi"] = subprocess.run("nvidia-smi; nvidia-smi topo -m", shell=True, capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
res = {}
for mb in (1, 16, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(s):
            for _ in range(3): fn()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            reps = max(3, 2048 // mb)
            e0.record(s)
            for _ in range(reps): fn()
            e1.record(s)
        e1.synchronize()
        res[f"{name}_{mb}MiB_GBps"] = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
# bidirectional
n = 1024 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(4):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
res["bidir_total_GBps"] = 2 * 4 * n / dt / 1e9
out["hostlink"] = res
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
