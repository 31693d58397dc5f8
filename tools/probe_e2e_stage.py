#!/usr/bin/env python
"""Host-buffer (e2e) throughput vs staging tile size: pinned key/IV in, pinned keystream out, through the C ABI."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1909_04750_b200 as pkg
KEY = bytes.fromhex("123456789abcdef01234")
def run(layout, n, tc, stage_mb):
    gen = pkg.MickeyGenerator(0)
    gen.set_stage_bytes(stage_mb << 20)
    keys = torch.from_numpy(np.tile(np.frombuffer(KEY, np.uint8), (n, 1))).pin_memory()
    ivs_np = np.zeros((n, 10), np.uint8); ivs_np[:, 2:] = np.arange(n, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(n, 8)
    ivs = torch.from_numpy(ivs_np).pin_memory()
    host = (torch.empty((tc, n // 32), dtype=torch.int32) if layout == "col" else torch.empty((n, tc // 8), dtype=torch.uint8)).pin_memory()
    def one():
        gen.init_material(keys, ivs, 80)
        (gen.generate_colmajor if layout == "col" else gen.generate_rowmajor)(tc, host)
    for _ in range(2): one()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3): one()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
    print(f"{layout} n=2^{n.bit_length()-1} T={tc} stage={stage_mb} MiB: {dt*1e3:.2f} ms/step {n*tc/dt/1e12:.4f} Tb/s  D2H {host.numel()*host.element_size()/dt/1e9:.1f} GB/s", flush=True)
    gen.close()
for mb in (0, 16, 32, 64, 128, 256):
    run("col", 1 << 20, 16384, mb)
for mb in (0, 16, 32, 64, 128, 256):
    run("row", 1 << 20, 16384, mb)
for mb in (0, 32, 64, 128):
    run("row", 1 << 24, 1024, mb)
