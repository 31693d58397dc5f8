#!/usr/bin/env python
"""Row-major keystream: staging tile in shared memory (7 worker warps per SM) vs tensor memory (8)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1909_04750_b200 as pkg
for lg, T in ((22, 16384), (24, 8192), (24, 65536 // 4)):
    n = 1 << lg
    out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
    for mode in (1, 2, 0, 1, 2, 0):
        gen = pkg.MickeyGenerator(0)
        gen.set_row_staging(mode)
        gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, n)
        ms = []
        for _ in range(3):
            gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
        print("staging", mode, "n 2^%d T %d plan" % (lg, T), gen.last_plan(), "ms", [round(m, 3) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 4), flush=True)
        gen.close()
    del out
