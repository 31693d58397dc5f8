"""One-shot bulk call at keystream-dominated shapes: fused kernel vs block pipeline vs init + generate."""
import sys; sys.path.insert(0, ".")
import torch
import paper_1909_04750_b200 as pkg
for lg, T in ((24, 8192), (22, 65536), (24, 65536)):
    N = 1 << lg
    g = torch.Generator(device="cuda").manual_seed(1)
    dk = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    di = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
    with pkg.MickeyGenerator(0) as gen:
        for fused in (True, False):
            gen.set_bulk_fused(fused)
            ms = []
            for _ in range(2):
                _, cs = gen.bulk_rowmajor(dk, di, 80, T, out); ms.append(gen.last_kernel_ms)
            print(lg, T, "bulk fused" if fused else "bulk blocks", round(min(ms), 2), "Tb/s", round(N * T / min(ms) / 1e9, 4), flush=True)
        ms = []
        for _ in range(2):
            gen.init_material(dk, di, 80); m = gen.last_kernel_ms
            gen.generate_rowmajor(T, out); ms.append(m + gen.last_kernel_ms)
        print(lg, T, "init + generate", round(min(ms), 2), "Tb/s", round(N * T / min(ms) / 1e9, 4), flush=True)
    del out, dk, di
    torch.cuda.empty_cache()
