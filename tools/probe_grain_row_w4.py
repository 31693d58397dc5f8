# Grain v1 row-major, worker warps per SM x chunk with the CURRENT store policy (one 256-bit evict_last store per
# row sector).  The store-pattern probe (profiles/r02_probe_store_pattern.txt) says four warps per SM with the keep
# hint can retire 32-byte runs at 1.9-2.0 TB/s; the round-1 geometry probe predates the hint.
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
for block, chunk in ((0, 0), (128, 4096), (128, 16384), (128, 65536), (160, 16384), (192, 16384), (224, 16384), (224, 65536), (0, 0)):
    gen = grain.GrainGenerator(0)
    gen.set_block_threads(block); gen.set_chunk_clocks(chunk)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
    print("grain row block", block, "chunk", chunk, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3), flush=True)
