#!/usr/bin/env python
"""NIST SP 800-22 subset on GPU-generated keystream, using the
REFERENCE's own suite (pkg/src/slicerng/stats.py:525-567, run as-is, read-only).

Runs in the build container only (the reference does not travel):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/nist_check.py \
        gpurun_out/nist_rows_256x1Mbit.npy profiles/r01_nist_suite_gpu_keystream.txt
Input: uint8 [streams][125000] rows written by tools/nist_sample.py on the B200
(rows 0, 256, 512, ... of a 2^16-instance x 1 Mbit row-major run, counter-IV material).
Also cross-checks the first and last sampled rows against the oracle, so the rows
judged here are known to be the reference's keystream bit for bit.
"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from slicerng import stats  # the reference

from oracle import mickey_oracle as orc

src, dst = sys.argv[1], sys.argv[2]
nstreams = int(sys.argv[3]) if len(sys.argv) > 3 else 100
rows = np.load(src)
key = bytes.fromhex("123456789abcdef01234")
for i in (0, len(rows) - 1):
    keys, ivs = orc.counter_material(key, 256 * i, 1)
    assert rows[i].tobytes() == orc.bulk_rowmajor(keys, ivs, 80, 1_000_000)[0].tobytes(), f"row {i} differs from the oracle"
streams = [stats.BitStream.from_bytes(r.tobytes()) for r in rows[:nstreams]]
t0 = time.time()
res = stats.run_suite(streams, alpha=0.01, workers=8)
dt = time.time() - t0
lines = [f"# NIST SP 800-22 subset (reference slicerng.stats.run_suite, alpha=0.01) on {len(streams)} GPU-generated",
         "# MICKEY 2.0 streams x 1 Mbit (tools/nist_sample.py on B200: 2^16 counter-IV instances, row-major, every 256th row)",
         f"# suite passed: {res.passed}   ({dt:.0f} s on the build container's CPU)",
         f"{'test':28s} {'proportion':>10s} {'min ok':>8s} {'uniformity p':>13s} {'pass':>5s}"]
for row in res.rows:
    lines.append(f"{row.name:28s} {row.proportion:10.4f} {row.proportion_interval[0]:8.4f} {row.uniformity_p:13.4f} {str(row.passed):>5s}")
lines.append(f"# delegated to the official sts battery (not in the reference's subset): {', '.join(res.delegated)}")
Path(dst).write_text("\n".join(lines) + "\n")
print("\n".join(lines))
