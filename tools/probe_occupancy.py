#!/usr/bin/env python
"""GPU probe: keystream-loop throughput vs CTA size / grid size (wave quantisation),
against the live LOP3 peak.  Prints one JSON line per configuration."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_1909_04750_b200 as pkg

KEY = bytes.fromhex("123456789abcdef01234")
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
gen = pkg.MickeyGenerator(0)
gen.set_stream(torch.cuda.current_stream().cuda_stream)
peak, ms = gen.lop3_peak()
sms = torch.cuda.get_device_properties(0).multi_processor_count
print(json.dumps({"lop3_peak_Tlaneops": peak / 1e12, "probe_ms": ms, "sms": sms,
                  "implied_lanes_per_clk_per_sm_at_1965MHz": peak / sms / 1.965e9}))
configs = []
for block, chunk in ((0, 0), (256, 1 << 30), (128, 4096), (256, 4096)):
    configs.append((block, chunk, sms * 8 * 32, "8 warps/SM exactly"))
    configs.append((block, chunk, 32768, "C2 geometry (2^20 instances)"))
    configs.append((block, chunk, 1 << 19, "C3 geometry (2^24 instances)"))
    configs.append((block, chunk, 50000, "odd: 1.6M instances"))
for layout in ("col", "row"):
    for block, chunk, G, label in configs:
        n = G * 32
        gen.set_block_threads(block)
        gen.set_chunk_clocks(chunk)
        gen.init_counter(KEY, 0, n)
        if layout == "col":
            out = torch.empty((T, G), dtype=torch.int32, device="cuda")
            fn = lambda: gen.generate_colmajor(T, out)
        else:
            out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
            fn = lambda: gen.generate_rowmajor(T, out)
        fn()
        best = 1e9
        for _ in range(3):
            fn()
            best = min(best, gen.last_kernel_ms)
        ops = n * T * 327 / 32
        print(json.dumps({"layout": layout, "block": block, "chunk": chunk, "plan": gen.last_plan(), "G": G, "label": label, "T": T, "ms": round(best, 3),
                          "Tbps": round(n * T / best / 1e9, 4), "lop3_frac": round(ops / (best * 1e-3) / peak, 4)}))
        del out
gen.close()
