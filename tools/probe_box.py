"""Probe the GPU box: host cores, GPU, pinned H2D bandwidth (the migration roofline denominator)."""
import json, os, subprocess, time
import torch

out = {"nproc": os.cpu_count()}
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500]
except Exception as e:  # noqa
    out["lscpu"] = str(e)
out["meminfo"] = open("/proc/meminfo").read()[:200]
out["smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout[:3000]
dev = torch.device("cuda:0")
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device=dev)
best = 0.0
for i in range(10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h, non_blocking=True); e.record(); torch.cuda.synchronize()
    best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
out["h2d_pinned_gbs_best_of_10_1GiB"] = best
best = 0.0
for i in range(10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); h.copy_(d, non_blocking=True); e.record(); torch.cuda.synchronize()
    best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
out["d2h_pinned_gbs_best_of_10_1GiB"] = best
props = torch.cuda.get_device_properties(0)
out["sm_count"] = props.multi_processor_count
out["total_mem"] = props.total_memory
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "smi", "meminfo")}))
