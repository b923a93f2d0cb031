"""Host placement vs H2D bandwidth probe (NVML CPU affinity, pinned copies)."""
import os, time, torch, numpy as np
import pynvml as N
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
ncpu = os.cpu_count()
words = (ncpu + 63) // 64
aff = N.nvmlDeviceGetCpuAffinity(h, words)
cpus = [w * 64 + b for w, m in enumerate(aff) for b in range(64) if (m >> b) & 1]
print("cpus", ncpu, "gpu-local", len(cpus), cpus[:4], "...", "current", len(os.sched_getaffinity(0)))
try:
    print("numa nodes:", open('/sys/devices/system/node/online').read().strip())
except Exception as e: print(e)
def bw():
    x = torch.empty(4_200_000 // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(x, device='cuda')
    for _ in range(5): d.copy_(x, non_blocking=True); torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 4.2e6 / np.median(ts) / 1e9
for i in range(3):
    print("H2D GB/s default affinity", round(bw(), 1))
os.sched_setaffinity(0, cpus)
for i in range(3):
    print("H2D GB/s gpu-local affinity", round(bw(), 1))
x = torch.empty(4_200_000 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device='cuda')
for n in (1, 2, 5, 20, 100):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): d.copy_(x, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / n
    print(f"back-to-back x{n}: {4.2e6 / dt / 1e9:.1f} GB/s")
