#!/bin/bash
mkdir -p gpurun_out


timeout 300 python - <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
for mode in (1, 2, 1, 2):
    gen = grain.GrainGenerator(0)
    gen.set_row_staging(mode) if hasattr(gen, "set_row_staging") else None
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
    print("grain row staging", mode, gen.last_plan(), [round(m, 3) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
PY
