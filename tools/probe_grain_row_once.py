"""One Grain v1 row-major launch at 2^22 instances x 65536 bits (for ncu captures and A/B runs).
usage: probe_grain_row_once.py [row_staging] [chunk] [reps]"""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
staging = int(sys.argv[1]) if len(sys.argv) > 1 else 0
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
gen = grain.GrainGenerator(0)
gen.set_row_staging(staging); gen.set_chunk_clocks(chunk)
gen.init_material(keys, ivs)
ms = []
for _ in range(reps):
    gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
print("grain row staging", staging, "plan", gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
