#!/usr/bin/env python
"""A/B: traced vs untraced, power-of-two vs padded output stride, C2 geometry."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1909_04750_b200 as pkg
T = 65536
G = 32768
gen = pkg.MickeyGenerator(0)
gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, G * 32)
peak, _ = gen.lop3_peak()
ideal = G * 32 * T * 327 / 32 / peak * 1e3
print("ideal ms at 100% of LOP3 peak:", round(ideal, 2))
out = torch.empty((T, G + 64), dtype=torch.int32, device="cuda")
def t(label, stride, trace, block=128, chunk=4096, reps=3):
    gen.set_block_threads(block); gen.set_chunk_clocks(chunk)
    gen.set_trace(1 << 17 if trace else 0)
    ms = []
    for _ in range(reps):
        gen.generate_colmajor(T, out.data_ptr(), stride_words=stride)
        ms.append(round(gen.last_kernel_ms, 2))
        if trace: gen.read_trace()
    print(f"{label}: stride={stride} trace={trace} block={block} chunk={chunk} plan={gen.last_plan()} ms={ms} frac={ideal/min(ms):.3f}", flush=True)
for rep in range(2):
    t("A", G, False); t("B", G, True); t("C", G + 32, False); t("D", G + 32, True); t("E", G + 64, False)
t("auto", G, False, block=0, chunk=0)
t("auto-pad", G + 32, False, block=0, chunk=0)
for chunk in (1772, 1024, 2048, 3072, 5462, 8192):
    t("sweep", G + 32, False, chunk=chunk, reps=2)
t("b256", G + 32, False, block=256, chunk=1024, reps=2)
