#!/usr/bin/env python
"""One keystream launch for ncu: probe_one.py <col|row> [log2 instances] [clocks] [block] [chunk]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1909_04750_b200 as pkg

layout = sys.argv[1] if len(sys.argv) > 1 else "col"
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 20
T = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
block = int(sys.argv[4]) if len(sys.argv) > 4 else 0
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 0
n = 1 << lg
gen = pkg.MickeyGenerator(0)
gen.set_stream(torch.cuda.current_stream().cuda_stream)
gen.set_block_threads(block)
gen.set_chunk_clocks(chunk)
gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, n)
if layout == "col":
    out = torch.empty((T, n // 32), dtype=torch.int32, device="cuda")
    for _ in range(2):
        gen.generate_colmajor(T, out)
else:
    out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        gen.generate_rowmajor(T, out)
torch.cuda.synchronize()
print(layout, n, T, gen.last_plan(), "ms", gen.last_kernel_ms, "Tb/s", n * T / gen.last_kernel_ms / 1e9)
