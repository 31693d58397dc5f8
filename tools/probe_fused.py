"""Fused one-kernel bulk_rowmajor (csrc/mk2_fused.cuh) against the oracle and the three-kernel path, then timing
at BASELINE config 5 (2^26 key/IV pairs x 1024 bits).  usage: probe_fused.py [parity|time|all]"""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1909_04750_b200 as pkg
from oracle import mickey_oracle as orc
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("parity", "all"):
    for N, T, ivb, pad in ((1024, 1024, 80, 0), (32 * 70 + 11, 1000, 80, 0), (5, 8, 0, 0), (4099, 264, 32, 3), (1 << 15, 4096 + 520, 80, 0),
                           (2 * 8 * 148 * 1024 + 4096 + 7, 128, 16, 0), (1 << 16, 256, 0, 16)):
        rng = np.random.default_rng(N + T)
        keys = rng.integers(0, 256, (N, 10), dtype=np.uint8); ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
        dk, di = torch.from_numpy(keys).cuda(), torch.from_numpy(ivs).cuda()
        sample = np.unique(np.concatenate([np.arange(min(N, 96)), np.arange(max(0, N - 96), N), rng.integers(0, N, 64)]))
        want = orc.bulk_rowmajor(keys[sample], ivs[sample], ivb, T)
        with pkg.MickeyGenerator(0) as gen:
            a = torch.zeros((N, T // 8 + pad), dtype=torch.uint8, device="cuda")
            _, ca = gen.bulk_rowmajor(dk, di, ivb, T, a)
            fused_launches = gen.last_kernel_launches
            resumable = N <= 2 * 8 * 148 * 1024
            if resumable:
                more = gen.generate_rowmajor(64)
                cs_resumed = gen.checksum()
            gen.set_bulk_fused(False)
            b = torch.zeros((N, T // 8 + pad), dtype=torch.uint8, device="cuda")
            _, cb = gen.bulk_rowmajor(dk, di, ivb, T, b)
            if resumable:
                more_b = gen.generate_rowmajor(64)
                assert np.array_equal(more, more_b) and cs_resumed == gen.checksum(), "resume differs"
        torch.cuda.synchronize()
        ok = bool((a == b).all().item()) and ca == cb and np.array_equal(a.cpu().numpy()[sample][:, : T // 8], want)
        print(N, T, ivb, pad, "fused launches", fused_launches, "same as 3-kernel path + oracle sample:", ok, hex(ca), flush=True)
        assert ok
if what in ("time", "all"):
    N, T = 1 << 26, 1024
    g = torch.Generator(device="cuda").manual_seed(1)
    dk = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    di = torch.randint(0, 256, (N, 10), dtype=torch.uint8, device="cuda", generator=g)
    out = torch.empty((N, T // 8), dtype=torch.uint8, device="cuda")
    with pkg.MickeyGenerator(0) as gen:
        for fused in (True, False, True, False):
            gen.set_bulk_fused(fused)
            ms = []
            for _ in range(4):
                _, cs = gen.bulk_rowmajor(dk, di, 80, T, out); ms.append(gen.last_kernel_ms)
            print("bulk fused" if fused else "bulk blocks", [round(m, 2) for m in ms], "Tb/s", round(N * T / min(ms) / 1e9, 4), hex(cs), flush=True)
        ms = []
        for _ in range(4):
            gen.init_material(dk, di, 80); m = gen.last_kernel_ms
            gen.generate_rowmajor(T, out); ms.append(m + gen.last_kernel_ms)
        print("init + generate", [round(m, 2) for m in ms], "Tb/s", round(N * T / min(ms) / 1e9, 4), hex(gen.checksum()), flush=True)
