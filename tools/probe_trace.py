#!/usr/bin/env python
"""Trace the persistent scheduler: per-job timeline analysis."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1909_04750_b200 as pkg

T = 32768
def run(label, G, chunk, block=256, max_ctas=0, dump=None):
    gen = pkg.MickeyGenerator(0)
    gen.set_block_threads(block); gen.set_chunk_clocks(chunk); gen.set_max_ctas(max_ctas)
    n = G * 32
    gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, n)
    out = torch.empty((T, G), dtype=torch.int32, device="cuda")
    gen.generate_colmajor(T, out.data_ptr())
    ms_untraced = gen.last_kernel_ms
    gen.set_trace(1 << 17)
    gen.generate_colmajor(T, out.data_ptr())
    ms = gen.last_kernel_ms
    tr = gen.read_trace()
    t0 = tr["t_pop"].min()
    dur = (tr["t_end"] - tr["t_start"]) / 1e6
    wait = (tr["t_start"] - tr["t_pop"]) / 1e6
    span = (tr["t_end"].max() - t0) / 1e6
    jobs_per_warp = np.bincount(tr["warp"])
    used = (jobs_per_warp > 0).sum()
    print(f"{label}: G={G} chunk={chunk} block={block} ctas={max_ctas or 'all'} kernel {ms_untraced:.2f}/{ms:.2f} ms jobs {len(tr)} "
          f"job ms mean {dur.mean():.3f} min {dur.min():.3f} max {dur.max():.3f} | wait mean {wait.mean():.3f} max {wait.max():.3f} "
          f"| jobs/warp {jobs_per_warp[jobs_per_warp>0].min()}..{jobs_per_warp.max()} warps {used} "
          f"| ideal-at-99% {n*T*327/32/18.5e12*1e3/0.99:.2f} ms", flush=True)
    if dump:
        np.save(dump, tr)
    gen.close(); del out

run("exact", 37888, 1 << 30)
run("exact", 37888, 4096)
for chunk in (8192, 4096, 2048, 1024, 512):
    run("C2", 32768, chunk)
run("C2-b128", 32768, 4096, block=128)
run("C2-b128-148", 32768, 4096, block=128, max_ctas=148)
run("C2-b128-148", 32768, 1024, block=128, max_ctas=148)
run("C3", 1 << 19, 4096)
