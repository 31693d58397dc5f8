#!/usr/bin/env python
"""LOP3-rate efficiency of the column-major loop with one / two worker warps per sub-partition (no hand-offs)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1909_04750_b200 as pkg
from paper_1909_04750_b200 import _native
lib = _native.lib()
per_clock = lib.mk2_lop3_per_block(0) / lib.mk2_rblock(0)
T = 65536
gen = pkg.MickeyGenerator(0)
peak, _ = gen.lop3_peak()
for warps_per_sm in (4, 8):
    G = 148 * warps_per_sm * 32
    gen.init_counter(bytes(10), 0, G * 32)
    out = torch.empty((T, G), dtype=torch.int32, device="cuda")
    gen.set_block_threads(32 * warps_per_sm); gen.set_chunk_clocks(1 << 30)
    ms = []
    for _ in range(4):
        gen.generate_colmajor(T, out.data_ptr()); ms.append(gen.last_kernel_ms)
    print(f"{warps_per_sm} warps/SM unchunked: ms {min(ms):.3f} frac(executed) {G * T * per_clock / (min(ms) * 1e-3) / peak:.4f}")
    for chunk in (16384, 4096):
        gen.set_chunk_clocks(chunk)
        ms = []
        for _ in range(3):
            gen.generate_colmajor(T, out.data_ptr()); ms.append(gen.last_kernel_ms)
        n_handoffs = T // chunk
        print(f"   chunk {chunk}: ms {min(ms):.3f}  -> {(min(ms) - 0) :.3f}; hand-offs per chain {n_handoffs}")
    del out
# trace of the C2 geometry at T = 262144, automatic plan
G = 32768; T = 262144
gen.init_counter(bytes(10), 0, G * 32)
out = torch.empty((T, G), dtype=torch.int32, device="cuda")
gen.set_block_threads(0); gen.set_chunk_clocks(0)
gen.generate_colmajor(T, out.data_ptr())
gen.set_trace(1 << 17)
gen.generate_colmajor(T, out.data_ptr())
tr = gen.read_trace()
print("C2 T=262144 plan", gen.last_plan(), "kernel ms", gen.last_kernel_ms, "jobs", len(tr))
t0 = tr["t_pop"].min()
dur = (tr["t_end"] - tr["t_start"]) / 1e6
wait = (tr["t_start"] - tr["t_pop"]) / 1e6
print("job ms: mean %.3f min %.3f max %.3f | pop->start ms: mean %.4f median %.4f max %.3f" % (dur.mean(), dur.min(), dur.max(), wait.mean(), np.median(wait), wait.max()))
# per worker: busy time vs span
span = (tr["t_end"].max() - t0) / 1e6
busy = np.zeros(tr["warp"].max() + 1)
np.add.at(busy, tr["warp"], dur)
nj = np.bincount(tr["warp"])
print("span ms %.3f | per-worker busy ms: mean %.3f min %.3f max %.3f | jobs per worker %d..%d" % (span, busy[nj > 0].mean(), busy[nj > 0].min(), busy[nj > 0].max(), nj[nj > 0].min(), nj.max()))
# gaps between consecutive jobs of a worker (end -> next start)
gaps = []
for w in np.unique(tr["warp"]):
    rows = tr[tr["warp"] == w]
    rows = rows[np.argsort(rows["t_start"])]
    gaps.extend(((rows["t_start"][1:] - rows["t_end"][:-1]) / 1e3).tolist())
gaps = np.array(gaps)
print("end->next start gap us: mean %.2f median %.2f p90 %.2f max %.2f" % (gaps.mean(), np.median(gaps), np.percentile(gaps, 90), gaps.max()))
last_end = np.zeros(tr["warp"].max() + 1); np.maximum.at(last_end, tr["warp"], (tr["t_end"] - t0) / 1e6)
print("tail: worker last-end ms: min %.3f mean %.3f max %.3f" % (last_end[nj > 0].min(), last_end[nj > 0].mean(), last_end[nj > 0].max()))
per_clock_ns = dur * 1e6 / (T / (T // gen.last_plan()[1] + (1 if T % gen.last_plan()[1] else 0)))
