set -x
nproc; lscpu | head -30; free -g; nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -iA3 -E "PCIe Generation|Link Width" | head -20
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for sz in [1<<20, 8<<20, 64<<20, 256<<20, 1<<30]:
    h = torch.empty(sz, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(sz, dtype=torch.uint8, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    n=10
    for _ in range(n): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)/n
    print(f"H2D {sz>>20} MiB: {sz/ms/1e6:.1f} GB/s")
    s.record()
    for _ in range(n): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    ms=s.elapsed_time(e)/n
    print(f"D2H {sz>>20} MiB: {sz/ms/1e6:.1f} GB/s")
import numpy as np, os
print("cpu_count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
a=np.ones((4096,14336)); x=np.ones((1,4096))
for _ in range(3): x@a
t=time.perf_counter(); 
for _ in range(10): x@a
print("numpy fp64 gemv 4096x14336 ms", (time.perf_counter()-t)/10*1e3)
import threadpoolctl; print(threadpoolctl.threadpool_info())
PY
cat /proc/meminfo | head -5
