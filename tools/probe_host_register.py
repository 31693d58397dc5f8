"""How fast is cudaHostRegister on a caller's ordinary numpy array (numpy madvises large allocations for transparent
huge pages)?  If pinning in place outruns the link, a pageable destination could take the D2H copies directly.
usage: probe_host_register.py"""
import time
import numpy as np, torch
rt = torch.cuda.cudart()
torch.zeros(1, device="cuda")
SIZE = 1 << 31
for touched in (True, False):
    for chunk_mib in (2048, 256, 64, 16):
        a = np.empty(SIZE, np.uint8)
        if touched:
            a[::4096] = 1
        c = chunk_mib << 20
        t0 = time.perf_counter()
        for o in range(0, SIZE, c):
            r = rt.cudaHostRegister(a.ctypes.data + o, c, 0)
            assert int(r) == 0, r
        t1 = time.perf_counter()
        for o in range(0, SIZE, c):
            rt.cudaHostUnregister(a.ctypes.data + o)
        t2 = time.perf_counter()
        print(f"{'touched  ' if touched else 'untouched'} 2 GiB, chunks of {chunk_mib:4d} MiB: register {1e3 * (t1 - t0):7.1f} ms ({SIZE / (t1 - t0) / 1e9:6.1f} GB/s)"
              f"  unregister {1e3 * (t2 - t1):6.1f} ms", flush=True)
        del a
