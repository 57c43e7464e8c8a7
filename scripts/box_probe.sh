#!/bin/bash
# One-off probe of the GPU box: cores, memory, GPU properties, pinned H2D bandwidth, ncu access.
out=gpurun_out/probe; mkdir -p $out
nproc > $out/nproc.txt; free -g > $out/free.txt; lscpu > $out/lscpu.txt
nvidia-smi > $out/smi.txt; nvidia-smi -q > $out/smi_q.txt; nvidia-smi topo -m > $out/topo.txt 2>&1
python - > $out/props.txt 2>&1 <<'PY'
import torch, time, os
p = torch.cuda.get_device_properties(0)
print(p)
print("sms", p.multi_processor_count, "l2", getattr(p, "L2_cache_size", None), "mem", p.total_memory)
print("affinity", len(os.sched_getaffinity(0)))
for mb in (64, 256, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize(); t = s.elapsed_time(e) / 10
    print(f"h2d {mb} MiB: {n/t/1e6:.1f} GB/s")
    s.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize(); t = s.elapsed_time(e) / 10
    print(f"d2h {mb} MiB: {n/t/1e6:.1f} GB/s")
PY
cat > /tmp/k.py <<'PY'
import torch
x = torch.ones(1<<20, device="cuda"); y = x * 2; torch.cuda.synchronize(); print(y.sum().item())
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --csv python /tmp/k.py > $out/ncu_test.txt 2>&1
echo done
