set -x
nproc; lscpu | head -30; free -g; cat /proc/meminfo | head -5
nvidia-smi; nvidia-smi topo -m; nvidia-smi -q | grep -i -A3 "PCI" | head -40
ulimit -l
numactl -H 2>/dev/null || true
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for sz in [64<<20, 256<<20, 1<<30]:
    h = torch.empty(sz, dtype=torch.uint8).pin_memory()
    d = torch.empty(sz, dtype=torch.uint8, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("H2D", sz, sz*10/(s.elapsed_time(e)/1e3)/1e9, "GB/s")
    s.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("D2H", sz, sz*10/(s.elapsed_time(e)/1e3)/1e9, "GB/s")
# pin large
t=time.time()
try:
    big = torch.empty(40<<30, dtype=torch.uint8).pin_memory()
    print("pinned 40GiB in", time.time()-t)
except Exception as ex:
    print("pin fail", ex)
PY
