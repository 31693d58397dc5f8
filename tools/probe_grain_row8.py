# Grain v1 row-major: the eight-warp kernel (mk2_set_row_staging(ctx, 5): 28 groups of the tile in shared memory, 4 in
# tensor memory) against the seven-warp default, by chunk length.
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1909_04750_b200 import grain
n, T = 1 << 22, 65536
rng = np.random.default_rng(1)
keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
ref = None
for staging, chunk in ((0, 0), (5, 4096), (5, 8192), (5, 16384), (5, 32768), (5, 0), (0, 0)):
    gen = grain.GrainGenerator(0)
    gen.set_row_staging(staging); gen.set_chunk_clocks(chunk)
    gen.init_material(keys, ivs)
    ms = []
    for _ in range(3):
        gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
    torch.cuda.synchronize()
    h = (int(out.view(torch.int64)[::4099].sum().item()), gen.checksum())
    if ref is None: ref = h
    print("grain row staging", staging, "chunk", chunk, gen.last_plan(), [round(m, 2) for m in ms], "Tb/s", round(n * T / min(ms) / 1e9, 3),
          "same bytes" if h == ref else "DIFFERENT BYTES", flush=True)
