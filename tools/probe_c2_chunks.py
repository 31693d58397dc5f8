#!/usr/bin/env python
"""Full-size config 2 (2^20 instances x 10^6 clocks, column-major): chunk-count sweep of the FIFO scheduler."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1909_04750_b200 as pkg
from paper_1909_04750_b200 import _native

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
G = 32768
gen = pkg.MickeyGenerator(0)
gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, G * 32)
peak, _ = gen.lop3_peak()
lib = _native.lib()
per_clock = lib.mk2_lop3_per_block(0) / lib.mk2_rblock(0)
out = torch.empty((T, G), dtype=torch.int32, device="cuda")
ideal = G * T * per_clock / peak * 1e3
print(f"T={T} ideal at 100% of the LOP3 peak ({per_clock:.1f} LOP3/clock): {ideal:.2f} ms")
ks = [int(a) for a in sys.argv[2:]] or [0, 37, 74, 111, 148, 185, 222, 296]
for k in ks:
    chunk = 0 if k == 0 else -(-T // k)
    gen.set_block_threads(0 if k == 0 else 128)
    gen.set_chunk_clocks(chunk)
    ms = []
    for _ in range(3):
        gen.generate_colmajor(T, out.data_ptr())
        ms.append(gen.last_kernel_ms)
    print(f"k={k} chunk={chunk} plan={gen.last_plan()} ms={[round(m, 2) for m in ms]} frac={ideal / min(ms):.4f}", flush=True)
