"""Host topology probe: GPU-local CPU set (NVML), process affinity, and H2D bandwidth of
pinned buffers allocated with/without binding to the GPU-local cores."""
import os, sys, time, subprocess
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
ncpu = os.cpu_count()
words = (ncpu + 63) // 64
mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
local = [w * 64 + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1]
print("cpus", ncpu, "affinity", len(os.sched_getaffinity(0)), "gpu-local", len(local), local[:4], "...", local[-4:])
try:
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
except Exception as e:
    print(e)
try:
    print(open("/sys/devices/system/node/online").read())
except Exception as e:
    print(e)
