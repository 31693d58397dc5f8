# Grain v1 row-major: chunk length x worker warps per SM (the library named by MK2_LIB, default build otherwise).
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
for block in (192, 224):
    for chunk in (2048, 4096, 8192, 16384, 32768):
        gen = grain.GrainGenerator(0)
        gen.set_block_threads(block); gen.set_chunk_clocks(chunk)
        gen.init_material(keys, ivs)
        ms = []
        for _ in range(3):
            gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
        print("grain row block", block, "chunk", chunk, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
