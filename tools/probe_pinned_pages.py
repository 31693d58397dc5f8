"""Does the D2H rate into pinned memory depend on how (and when) the pinned buffer was allocated?  cudaHostAlloc at
process start, cudaHostAlloc after the process has churned through host memory, and an mmap + MADV_HUGEPAGE +
cudaHostRegister buffer.  usage: probe_pinned_pages.py"""
import ctypes, mmap, os, time
import numpy as np, torch
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), "| defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
def meminfo(keys=("MemFree", "AnonHugePages", "HugePages_Total")):
    d = dict(l.split(":") for l in open("/proc/meminfo"))
    return {k: d[k].strip() for k in keys}
print(meminfo())
SIZE = 1 << 31
x = torch.empty(SIZE, dtype=torch.uint8, device="cuda")
def rate(h):
    h.copy_(x); torch.cuda.synchronize()
    best = 0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
        best = max(best, SIZE / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best
a = torch.empty(SIZE, dtype=torch.uint8).pin_memory()
print("cudaHostAlloc at start:            ", round(rate(a), 2), "GB/s", meminfo(("AnonHugePages",)))
del a
# churn: touch a lot of host memory in small pieces, free every other piece (fragmentation), keep the rest alive
keep = []
for i in range(4096):
    b = np.ones(4 << 20, np.uint8)           # 16 GiB in 4 MiB pieces
    if i & 1:
        keep.append(b)
b = torch.empty(SIZE, dtype=torch.uint8).pin_memory()
print("cudaHostAlloc after 16 GiB churn:  ", round(rate(b), 2), "GB/s", meminfo(("AnonHugePages",)))
del b
libc = ctypes.CDLL("libc.so.6", use_errno=True)
m = mmap.mmap(-1, SIZE + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
al = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
rc = libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(SIZE), 14)    # MADV_HUGEPAGE
arr = np.frombuffer(m, np.uint8, SIZE, al - addr)
arr[::4096] = 1
t = torch.from_numpy(arr)
r = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), SIZE, 0)
print("mmap + MADV_HUGEPAGE + register:   ", round(rate(t), 2), "GB/s", "madvise rc", rc, "register rc", r, meminfo(("AnonHugePages",)))
