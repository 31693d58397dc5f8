"""Where the fused bulk kernel spends its time: the same batch at T = 8, 1024, 2048 (marginal cost of 1024 keystream
clocks) against the three-kernel path.  usage: probe_fused_split.py [log2 N]"""
import sys; sys.path.insert(0, ".")
import torch
import paper_1909_04750_b200 as pkg
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
N = 1 << lg
g = torch.Generator(device="cuda").manual_seed(1)
dk = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
di = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
with pkg.MickeyGenerator(0) as gen:
    for T in (8, 1024, 2048):
        out = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
        for fused in (True, False):
            gen.set_bulk_fused(fused)
            ms = []
            for _ in range(3):
                gen.bulk_rowmajor(dk, di, 80, T, out); ms.append(gen.last_kernel_ms)
            print("T", T, "fused" if fused else "blocks", round(min(ms), 3), flush=True)
        ms = []; mi = []
        for _ in range(3):
            gen.init_material(dk, di, 80); a = gen.last_kernel_ms
            gen.generate_rowmajor(T, out); ms.append(a + gen.last_kernel_ms); mi.append(a)
        print("T", T, "init+generate", round(min(ms), 3), "init", round(min(mi), 3), flush=True)
        del out
