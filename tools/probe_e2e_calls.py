"""Host-buffer column-major calls into pinned memory: fixed cost per call and per-byte rate (t = a + b * bytes), by
staging tile size.  usage: probe_e2e_calls.py"""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1909_04750_b200 as pkg
n = 1 << 20; G = n // 32
KEY = bytes.fromhex("123456789abcdef01234")
host = torch.empty((16384, G), dtype=torch.int32).pin_memory()
for stage_mib in (0, 8, 16, 64):
    with pkg.MickeyGenerator(0) as gen:
        if stage_mib:
            gen.set_stage_bytes(stage_mib << 20)
        gen.init_counter(KEY, 0, n)
        res = {}
        for tc in (1024, 4096, 16384):
            gen.generate_colmajor(tc, host[:tc])
            v = []
            for _ in range(6):
                t0 = time.perf_counter(); gen.generate_colmajor(tc, host[:tc]); v.append(time.perf_counter() - t0)
            res[tc] = min(v)
        b = (res[16384] - res[4096]) / ((16384 - 4096) * G * 4)
        a = res[4096] - b * 4096 * G * 4
        print(f"stage {stage_mib or 32:3d} MiB: " + "  ".join(f"T={tc}: {res[tc] * 1e3:7.3f} ms ({tc * G * 4 / res[tc] / 1e9:5.1f} GB/s)" for tc in res)
              + f"  | fixed {a * 1e6:6.0f} us per call, streaming rate {1 / b / 1e9:5.2f} GB/s", flush=True)
