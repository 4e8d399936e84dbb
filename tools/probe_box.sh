#!/bin/bash
# Probe the GPU box host: cores, memory, NUMA, CPU ISA, PCIe H2D bandwidth.
set -x
nproc; free -g; lscpu; numactl -H 2>/dev/null || true
nvidia-smi; nvidia-smi topo -m
cat /proc/meminfo | head -5
ulimit -l
python - <<'PY'
import torch, time, os
print("cuda", torch.cuda.is_available(), torch.cuda.get_device_name(0))
for mb in (64, 352, 1024):
    n = mb*1024*1024
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print("H2D", mb, "MB", 5*n/(e0.elapsed_time(e1)/1e3)/1e9, "GB/s")
# pin a large buffer
t=time.time()
try:
    big = torch.empty(64*1024**3, dtype=torch.uint8).pin_memory()
    print("pinned 64GiB ok", time.time()-t)
    del big
except Exception as e:
    print("pin 64GiB failed", e)
# host dram bandwidth rough
import numpy as np
a = np.ones(512*1024*1024//8)
t=time.time(); 
for _ in range(3): s=a.sum()
print("numpy sum 1thread GB/s", 3*a.nbytes/(time.time()-t)/1e9)
torch.set_num_threads(os.cpu_count())
x = torch.ones(2*1024**3//2, dtype=torch.bfloat16)
t=time.time()
for _ in range(3): s=x.sum()
print("torch sum all threads GB/s", 3*x.nbytes/(time.time()-t)/1e9, torch.get_num_threads())
PY
