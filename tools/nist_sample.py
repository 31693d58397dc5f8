#!/usr/bin/env python
"""GPU side of the NIST quality check: generate 2^16 counter-IV
instances x 1 Mbit row-major on the B200, keep every 256th row (256 streams x 1 Mbit = 32 MB)
under gpurun_out/ for tools/nist_check.py, which runs the REFERENCE's stats.run_suite on them."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1909_04750_b200 as pkg

N, T = 1 << 16, 1_000_000
key = bytes.fromhex("123456789abcdef01234")
gen = pkg.MickeyGenerator(0)
gen.init_counter(key, 0, N)
rows = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
gen.generate_rowmajor(T, rows)
torch.cuda.synchronize()
print("kernel ms", gen.last_kernel_ms, "Tb/s", N * T / gen.last_kernel_ms / 1e9, "plan", gen.last_plan())
sel = rows[::256].cpu().numpy()
np.save("gpurun_out/nist_rows_256x1Mbit.npy", sel)
print("saved", sel.shape, "checksum", hex(gen.checksum()))
