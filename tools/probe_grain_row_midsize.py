# Grain v1 row-major at mid-size batches (fewer chains than 16 per SM, where the planner picks four lone warps per SM):
# worker warps per SM x instances, 65536 clocks.
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
T = 65536
rng = np.random.default_rng(1)
for logn in (19, 20, 21):
    n = 1 << logn
    keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
    ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
    out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
    for block in (0, 128, 160, 192, 224):
        gen = grain.GrainGenerator(0)
        gen.set_block_threads(block)
        gen.init_material(keys, ivs)
        ms = []
        for _ in range(3):
            gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
        print("grain row n=2^%d chains %d block" % (logn, n // 1024), block, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
    del out
