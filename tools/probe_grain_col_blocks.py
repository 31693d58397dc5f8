"""Grain v1 column-major by worker warps per SM: the lone-warp ceiling of the clock loop without any drain."""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((T, n // 32), dtype=torch.int32, device="cuda")
for block in (128, 160, 192, 224, 256):
    gen = grain.GrainGenerator(0)
    gen.set_block_threads(block); gen.set_chunk_clocks(4096)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_colmajor(T, out); ms.append(gen.last_kernel_ms)
    print("grain col warps/SM", block // 32, gen.last_plan(), "ms", round(min(ms), 2), "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
    gen.close()
