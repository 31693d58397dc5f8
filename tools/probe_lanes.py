"""Copy-lane experiment (run under gpurun): pageable 2 GiB outputs, sub-chunk size x store flavour x lane count."""
import json, os, subprocess, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
CODE = r'''
import sys, time, json
import numpy as np
sys.path.insert(0, %r)
import paper_1909_04750_b200 as pkg
N, T = 1 << 20, 16384
key = bytes.fromhex("123456789abcdef01234")
res = {}
with pkg.MickeyGenerator(0) as gen:
    gen.init_counter(key, 0, N)
    page = np.empty((T, N // 32), np.uint32); page[:] = 0
    rows = np.empty((N, T // 8), np.uint8); rows[:] = 0
    for th in (4, 8, 12, 16):
        gen.set_host_threads(th)
        v = []
        for _ in range(4):
            t0 = time.perf_counter(); gen.generate_colmajor(T, page); v.append(time.perf_counter() - t0)
        res["col_%%d" %% th] = round(N * T / 8 / min(v[1:]) / 1e9, 1)
        v = []
        for _ in range(3):
            t0 = time.perf_counter(); gen.generate_rowmajor(T, rows); v.append(time.perf_counter() - t0)
        res["row_%%d" %% th] = round(N * T / 8 / min(v[1:]) / 1e9, 1)
print(json.dumps(res))
''' % str(ROOT)
out = {}
for lane_bytes in (1 << 20, 2 << 20, 8 << 20):
    for nt in (0, 1):
        env = dict(os.environ, MK2_LANE_BYTES=str(lane_bytes), MK2_LANE_NT=str(nt))
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        out[f"lane_bytes={lane_bytes >> 20}MiB nt={nt}"] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
print(json.dumps(out, indent=1))
