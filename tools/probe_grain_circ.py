# Grain v1 column-major: circular-buffer clocking (no realignment moves; mk2_set_row_staging(ctx, 4)) against the
# sliding window, eight warps per SM and four (lone warps).
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 8192
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
col = torch.empty((T, n // 32), dtype=torch.int32, device="cuda")
ref = None
for staging, block in ((0, 0), (4, 0), (0, 128), (4, 128), (4, 0), (0, 0)):
    gen = grain.GrainGenerator(0)
    gen.set_row_staging(staging); gen.set_block_threads(block)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_colmajor(T, col); ms.append(gen.last_kernel_ms)
    torch.cuda.synchronize()
    h = (int(col.view(torch.int64)[::4099].sum().item()), gen.checksum())
    if ref is None: ref = h
    print("grain col staging", staging, "block", block, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3),
          "same words" if h == ref else "DIFFERENT", flush=True)
