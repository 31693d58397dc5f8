#!/usr/bin/env python
"""One Grain v1 keystream launch for ncu: probe_grain.py <col|row> [log2 instances] [clocks]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1909_04750_b200 import grain

layout = sys.argv[1] if len(sys.argv) > 1 else "col"
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 22
T = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
n = 1 << lg
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
gen = grain.GrainGenerator(0)
gen.init_material(keys, ivs)
out = torch.empty((T, n // 32), dtype=torch.int32, device="cuda") if layout == "col" else torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
for _ in range(2):
    gen.generate_colmajor(T, out) if layout == "col" else gen.generate_rowmajor(T, out)
torch.cuda.synchronize()
print("grain", layout, n, T, gen.last_plan(), "ms", gen.last_kernel_ms, "Tb/s", n * T / gen.last_kernel_ms / 1e9)
