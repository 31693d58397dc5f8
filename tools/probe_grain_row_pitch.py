"""Grain v1 row-major at 2^22 instances x 65536 bits with padded row pitches: does the power-of-two pitch (8 KiB
rows) cost DRAM efficiency?  usage: probe_grain_row_pitch.py"""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
gen = grain.GrainGenerator(0)
for pad in (0, 32, 64, 128, 256, 512, 1024, 4096):
    out = torch.empty((n, T // 8 + pad), dtype=torch.uint8, device="cuda")
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
    print("pitch", T // 8 + pad, [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
    del out
