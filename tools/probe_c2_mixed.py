#!/usr/bin/env python
"""Config-2 geometry (1024 chains, 592 sub-partitions): the automatic plan (one worker warp per sub-partition,
few long chunks) against plans with MORE workers than chains (7 or 8 warps per SM, short chunks): chains then
migrate between shared and lone sub-partitions and every sub-partition keeps at least one busy warp."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1909_04750_b200 as pkg
from paper_1909_04750_b200 import _native
T = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
G = 32768
gen = pkg.MickeyGenerator(0)
gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, G * 32)
peak, _ = gen.lop3_peak()
lib = _native.lib()
per_clock = lib.mk2_lop3_per_block(0) / lib.mk2_rblock(0)
out = torch.empty((T, G), dtype=torch.int32, device="cuda")
ideal = G * T * per_clock / peak * 1e3
for block, chunk in ((0, 0), (160, 4096), (160, 16384), (160, 32768), (192, 4096), (192, 8192), (192, 16384), (192, 32768), (224, 4096), (224, 16384), (0, 0)):
    gen.set_block_threads(block); gen.set_chunk_clocks(chunk)
    ms = []
    for _ in range(3):
        gen.generate_colmajor(T, out.data_ptr()); ms.append(gen.last_kernel_ms)
    print(f"block={block} chunk={chunk} plan={gen.last_plan()} ms={[round(m, 2) for m in ms]} frac={ideal / min(ms):.4f}", flush=True)
