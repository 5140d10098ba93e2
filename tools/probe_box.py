"""One-off box probe: host RAM/cores, device memory, cuBLAS FP64 DGEMM rate (context)."""
import os, subprocess, time, json
import torch
out = {}
out["nproc_affinity"] = len(os.sched_getaffinity(0))
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["cpu_model"] = [l for l in open("/proc/cpuinfo").read().splitlines() if l.startswith("model name")][:1]
p = torch.cuda.get_device_properties(0)
out["sm_count"] = p.multi_processor_count
out["total_mem"] = p.total_memory
free, total = torch.cuda.mem_get_info()
out["mem_free"] = free
out["ngpu"] = torch.cuda.device_count()
res = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    res[n] = 2 * n**3 / best / 1e12
# HPL-shaped: m x n x 512
m = 32768
A = torch.randn(m, 512, dtype=torch.float64, device="cuda")
B = torch.randn(512, m, dtype=torch.float64, device="cuda")
C = torch.randn(m, m, dtype=torch.float64, device="cuda")
for _ in range(3): C.addmm_(A, B, alpha=-1)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); C.addmm_(A, B, alpha=-1); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
res["hpl_32768x32768x512"] = 2 * m * m * 512 / best / 1e12
out["cublas_dgemm_tflops"] = res
print(json.dumps(out, indent=1))
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit", "--format=csv"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
