#!/usr/bin/env python
"""Measured figures for the SURVEY 8(f) rows that bench.py (the MICKEY headline) does not cover:
Grain v1 keystream (column- and row-major) and GPU seed derivation.  Same hygiene as bench.py:
3 warm-up launches, CUDA-event times of the launches themselves, outputs >> L2, LOP3 peak measured
live.  Prints one JSON line per measurement."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_1909_04750_b200 as pkg
from paper_1909_04750_b200 import grain

GRAIN_ALU_PER_CLOCK = 37.4  # SASS: 598 LOP3 and nothing else on the ALU pipe per 16 clocks (profiles/r01b_sass_loop_stats.txt)


def best_ms(fn, gen, warm=3, reps=5):
    for _ in range(warm):
        fn()
    ms = []
    for _ in range(reps):
        fn()
        ms.append(gen.last_kernel_ms)
    return min(ms), float(np.median(ms))


def main():
    rng = np.random.default_rng(1)
    n, T = 1 << 22, 65536
    keys = torch.from_numpy(rng.integers(0, 256, (n, 10), dtype=np.uint8)).cuda()
    ivs = torch.from_numpy(rng.integers(0, 256, (n, 8), dtype=np.uint8)).cuda()
    with grain.GrainGenerator(0) as gen:
        peak, _ = gen.lop3_peak()
        init_best, _ = best_ms(lambda: gen.init_material(keys, ivs), gen)
        for layout in ("colmajor", "rowmajor"):
            out = (torch.empty((T, n // 32), dtype=torch.int32, device="cuda") if layout == "colmajor"
                   else torch.empty((n, T // 8), dtype=torch.uint8, device="cuda"))
            fn = (lambda: gen.generate_colmajor(T, out)) if layout == "colmajor" else (lambda: gen.generate_rowmajor(T, out))
            b, med = best_ms(fn, gen)
            print(json.dumps({"what": f"grain v1 keystream, {layout}", "instances": n, "clocks": T, "plan": gen.last_plan(),
                              "ms_best": b, "ms_median": med, "tbps": n * T / med / 1e9, "store_gbs": n * T / 8 / med / 1e6,
                              "alu_ops_per_clock": GRAIN_ALU_PER_CLOCK,
                              "frac_of_lop3_peak": n * T * GRAIN_ALU_PER_CLOCK / 32 / (med * 1e-3) / peak,
                              "lop3_peak_tlaneops": peak / 1e12}))
            del out
        print(json.dumps({"what": "grain v1 init (key/IV transpose + 160 clocks)", "instances": n, "ms_best": init_best,
                          "inits_per_s": n / (init_best * 1e-3)}))
    seed = bytes(range(32))
    for lg in (20, 26):
        m = 1 << lg
        dk = torch.empty((m, 10), dtype=torch.uint8, device="cuda")
        di = torch.empty((m, 10), dtype=torch.uint8, device="cuda")
        with pkg.MickeyGenerator(0) as gen:
            b, med = best_ms(lambda: gen.derive_material(seed, 0, m, dk, di), gen)
            print(json.dumps({"what": "seed derivation (2 AES-128 blocks per lane)", "lanes": m, "ms_median": med,
                              "lanes_per_s": m / (med * 1e-3), "aes_blocks_per_s": 2 * m / (med * 1e-3)}))
            b2, med2 = best_ms(lambda: gen.init_seed(seed, 0, m), gen)
            print(json.dumps({"what": "mk2_init_from_seed (derive + pack + MICKEY init)", "lanes": m, "ms_median": med2}))
        del dk, di


if __name__ == "__main__":
    main()
