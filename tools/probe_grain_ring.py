# Grain v1 row-major: the lone-warp ring kernel (mk2_set_row_staging(ctx, 4)) against the default, by chunk length;
# Grain column-major with four warps per SM for the lone-warp efficiency of the bare cipher loop.
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
ref = None
for staging, chunk in ((0, 0), (4, 4096), (4, 16384), (4, 65536), (4, 0), (0, 0)):
    gen = grain.GrainGenerator(0)
    gen.set_row_staging(staging); gen.set_chunk_clocks(chunk)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
    torch.cuda.synchronize()
    h = int(out.view(torch.int64)[::4099].sum().item())
    if ref is None: ref = h
    print("grain row staging", staging, "chunk", chunk, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3),
          "same bytes" if h == ref else "DIFFERENT BYTES", flush=True)
del out
col = torch.empty((T // 8, n // 32), dtype=torch.int32, device="cuda")
for block in (0, 128):
    gen = grain.GrainGenerator(0)
    gen.set_block_threads(block)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_colmajor(T // 8, col); ms.append(gen.last_kernel_ms)
    print("grain col block", block, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * (T // 8) / min(ms) / 1e9, 3), flush=True)
