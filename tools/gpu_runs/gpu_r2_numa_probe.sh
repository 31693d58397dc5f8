lscpu | grep -i "numa\|socket\|model name\|^CPU(s)"; nvidia-smi topo -m 2>&1 | head -12; cat /sys/fs/cgroup/cpuset.cpus.effective 2>/dev/null; nproc
bdf=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//'); echo "bdf $bdf"; cat /sys/bus/pci/devices/${bdf}/numa_node 2>/dev/null; cat /sys/bus/pci/devices/${bdf}/local_cpulist 2>/dev/null
python - <<'PY'
import os, time, torch
print("affinity", sorted(os.sched_getaffinity(0)))
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
def bw(cpus):
    os.sched_setaffinity(0, cpus)
    h = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
    h.copy_(x); torch.cuda.synchronize()
    best = 0
    for _ in range(5):
        t0 = time.perf_counter(); h.copy_(x, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t0
        best = max(best, (1 << 30) / dt / 1e9)
    return best
all_cpus = sorted(os.sched_getaffinity(0))
for c in all_cpus:
    print("alloc on cpu", c, "D2H GB/s", round(bw({c}), 1), flush=True)
PY
