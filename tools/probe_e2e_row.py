"""Pinned host buffers, row-major: one-shot mk2_bulk_rowmajor (upload | init + keystream | download of instance blocks)
at config 3's and config 5's shapes, 2 GiB of rows per call.  Experiment knobs: MK2_ROW_WORKERS (worker warps per SM of
a tile's chain block), MK2_ROW_TILE_FACTOR (tile bytes = factor x 32 MiB).  usage: probe_e2e_row.py"""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1909_04750_b200 as pkg
for lg, T in ((20, 16384), (24, 1024), (22, 4096)):
    n = 1 << lg
    rng = np.random.default_rng(1)
    keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).pin_memory()
    ivs = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).pin_memory()
    host = torch.empty((n, T // 8), dtype=torch.uint8).pin_memory()
    with pkg.MickeyGenerator(0) as gen:
        gen.bulk_rowmajor(keys, ivs, 80, T, host)
        v = []
        for _ in range(5):
            t0 = time.perf_counter(); gen.bulk_rowmajor(keys, ivs, 80, T, host); v.append(time.perf_counter() - t0)
    dt = min(v)
    print(f"n=2^{lg} T={T}: {dt * 1e3:7.2f} ms  {n * T / dt / 1e12:.4f} Tb/s  D2H {n * T / 8 / dt / 1e9:5.1f} GB/s", flush=True)
