#!/bin/bash
# e2e distribution without and with binding to the GPU-local cores
python tools/numa_probe.py
python tools/e2e_dist.py
LOCAL=$(python -c "
import os, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
m = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count()+63)//64)
print(','.join(str(w*64+b) for w, x in enumerate(m) for b in range(64) if (x>>b)&1))")
echo "local=$LOCAL"
taskset -c $LOCAL python tools/e2e_dist.py
taskset -c $LOCAL python tools/e2e_dist.py
python tools/e2e_dist.py
