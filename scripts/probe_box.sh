#!/bin/bash
# One-shot host/topology dump of the GPU box.
out=gpurun_out/probe_box.txt
{
echo "== nvidia-smi -L"; nvidia-smi -L
echo "== CUDA_VISIBLE_DEVICES=$CUDA_VISIBLE_DEVICES NVIDIA_VISIBLE_DEVICES=$NVIDIA_VISIBLE_DEVICES"
echo "== topo"; nvidia-smi topo -m
echo "== nvlink"; nvidia-smi nvlink -s 2>&1 | head -40
echo "== pcie"; nvidia-smi -q | grep -A12 -i "GPU Link Info" | head -40
echo "== lscpu"; lscpu
echo "== nproc"; nproc
echo "== free"; free -g
echo "== numa nodes"; ls /sys/devices/system/node/ 2>&1; cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep MemTotal
echo "== gpu numa"; for b in $(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader); do bb=$(echo $b | tr 'A-F' 'a-f' | sed 's/^0000//'); f=$(ls -d /sys/bus/pci/devices/*${bb#0000} 2>/dev/null | head -1); echo "$b $f numa=$(cat $f/numa_node 2>/dev/null)"; done
echo "== ulimit -l"; ulimit -l
echo "== torch"
python - <<'PY'
import torch, time
print("count", torch.cuda.device_count())
for i in range(torch.cuda.device_count()):
    p = torch.cuda.get_device_properties(i); print(i, p.name, p.multi_processor_count, p.total_memory)
n = torch.cuda.device_count()
for i in range(n):
    print([torch.cuda.can_device_access_peer(i,j) if i!=j else None for j in range(n)])
torch.cuda.set_device(0)
B = 1<<30
h = torch.empty(B, dtype=torch.uint8).pin_memory()
d = torch.empty(B, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for name, f in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    best = 1e9
    with torch.cuda.stream(s):
        for r in range(6):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(name, "GB/s", B/best/1e6)
# host memcpy bandwidth
import numpy as np
a = np.ones(B, dtype=np.uint8); b = np.empty_like(a)
t=time.time(); np.copyto(b,a); print("host memcpy 1thr GB/s", B/(time.time()-t)/1e9)
PY
} > $out 2>&1
cat $out | tail -80
