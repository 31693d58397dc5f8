#!/usr/bin/env python
"""Fixture for the NIST quality chain (TEST INFRASTRUCTURE ONLY).

    python oracle/gen_nist_rows.py      -> tests/golden/nist_rows_sha256.json

The rows judged by the reference's NIST SP 800-22 subset (stats.run_suite, pkg/src/slicerng/stats.py:525-567)
are 100 MICKEY 2.0 streams of 1 Mbit: instances 0, 256, 512, ... of the counter-IV set of SURVEY.md 8(d)
(key 123456789abcdef01234, IV = 80-bit big-endian instance index), MSB-first bytes.  This script writes their
SHA-256 digests, computed with the oracle (itself pinned to the reference by tests/test_oracle.py), so that
    tests/test_nist_quality.py   (CPU)  oracle rows == fixture, reference suite passes on those rows
    tests/test_gpu_parity.py     (GPU)  GPU rows    == fixture
close the chain  GPU == oracle == rows judged  without the reference having to travel to the GPU box.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import mickey_oracle as orc  # noqa: E402

KEY = bytes.fromhex("123456789abcdef01234")
NROWS, STEP, NBITS = 100, 256, 1_000_000


def rows() -> np.ndarray:
    keys = np.tile(np.frombuffer(KEY, np.uint8), (NROWS, 1))
    ivs = np.zeros((NROWS, 10), np.uint8)
    ivs[:, 2:] = (np.arange(NROWS, dtype=np.uint64) * np.uint64(STEP)).astype(">u8").view(np.uint8).reshape(NROWS, 8)
    # every row is its own instance: the oracle batches 64 consecutive rows per engine, lanes are independent
    return orc.bulk_rowmajor(keys, ivs, 80, NBITS)


def main():
    r = rows()
    out = {"key": KEY.hex(), "rows": NROWS, "instance_step": STEP, "nbits": NBITS,
           "sha256": [hashlib.sha256(x.tobytes()).hexdigest() for x in r]}
    (ROOT / "tests" / "golden" / "nist_rows_sha256.json").write_text(json.dumps(out, indent=0) + "\n")
    print("wrote", len(out["sha256"]), "digests; row 0 starts", r[0, :16].tobytes().hex())


if __name__ == "__main__":
    main()
