"""Device-to-pinned-host copy rate by chunk size: 2 GiB moved as back-to-back cudaMemcpyAsync calls of one size on one
stream (what a staging pipeline's copy stream does), and the same with a concurrent kernel stream writing the
source buffers.  usage: probe_d2h_chunks.py"""
import time, torch
total = 1 << 31
x = torch.empty(total, dtype=torch.uint8, device="cuda")
h = torch.empty(total, dtype=torch.uint8).pin_memory()
s = torch.cuda.Stream()
for mib in (2, 4, 8, 16, 32, 64, 128, 256, 512, 2048):
    c = mib << 20
    best = 0
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for o in range(0, total, c):
                h[o:o + c].copy_(x[o:o + c], non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize()
        best = max(best, total / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(f"chunk {mib:5d} MiB: {best:6.2f} GB/s  ({total // c} copies)", flush=True)
