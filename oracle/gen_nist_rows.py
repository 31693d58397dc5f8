#!/usr/bin/env python
"""Fixture for the NIST quality chain (TEST INFRASTRUCTURE ONLY).

    python oracle/gen_nist_rows.py      -> tests/golden/nist_rows_sha256.json

The rows judged are the reference's own acceptance streams (criterion 4, pkg/tests/test_acceptance.py:188-223 =
cli._suite_streams, cli.py:212-231): 100 MICKEY 2.0 streams of 1 Mbit from the master seed 0x11..11, 64-lane batches
keyed by seed[0] ^ batch, seed-derived key/IV per lane, MSB-first bytes.  This script writes their SHA-256 digests,
computed with the oracle (oracle.suite_streams; pinned to the reference by tests/test_oracle.py, which checks the
first three of these very streams at full length against digests made by the reference itself), so that
    tests/test_nist_quality.py   (CPU)  oracle rows == fixture, the reference's NIST subset passes on those rows
    tests/test_gpu_parity.py     (GPU)  cli.suite_streams on the B200 == fixture
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

SEED = bytes.fromhex("11" * 32)
NROWS, NBITS = 100, 1_000_000


def rows() -> np.ndarray:
    return orc.suite_streams(SEED, NROWS, NBITS)


def main():
    r = rows()
    out = {"seed": SEED.hex(), "rows": NROWS, "nbits": NBITS,
           "sha256": [hashlib.sha256(x.tobytes()).hexdigest() for x in r]}
    (ROOT / "tests" / "golden" / "nist_rows_sha256.json").write_text(json.dumps(out, indent=0) + "\n")
    print("wrote", len(out["sha256"]), "digests; row 0 starts", r[0, :16].tobytes().hex())


if __name__ == "__main__":
    main()
