#!/bin/bash
# NUMA placement of the GPU box vs pinned H2D bandwidth.
out=gpurun_out/numa; mkdir -p $out
lscpu > $out/lscpu.txt; nvidia-smi topo -m > $out/topo.txt 2>&1; (numactl --hardware || true) > $out/numactl.txt 2>&1
cat /sys/class/pci_bus/*/device/numa_node 2>/dev/null | sort | uniq -c > $out/pci_numa.txt
python - > $out/affinity.txt 2>&1 <<'PY'
import os
print("allowed", sorted(os.sched_getaffinity(0)))
try:
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, 8)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    print("gpu0 local cpus", cpus[:8], "...", len(cpus))
    try:
        print("gpu0 numa", pynvml.nvmlDeviceGetNumaNodeId(h))
    except Exception as e:
        print("numa id n/a", e)
except Exception as e:
    print("nvml", e)
PY
cat > /tmp/h2d.py <<'PY'
import torch, os, sys
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(2): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): d.copy_(h, non_blocking=True)
e.record(); torch.cuda.synchronize(); t = s.elapsed_time(e) / 5
print(sys.argv[1], f"h2d 1 GiB: {n/t/1e6:.1f} GB/s", "cpus", len(os.sched_getaffinity(0)))
PY
python /tmp/h2d.py all >> $out/h2d.txt 2>&1
for node in $(ls -d /sys/devices/system/node/node* 2>/dev/null | sed 's/.*node//'); do
  cpus=$(cat /sys/devices/system/node/node$node/cpulist)
  taskset -c $cpus python /tmp/h2d.py node$node >> $out/h2d.txt 2>&1
  (numactl --cpunodebind=$node --membind=$node python /tmp/h2d.py numactl$node >> $out/h2d.txt 2>&1) || true
done
echo done
