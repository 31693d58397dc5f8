#!/usr/bin/env python
"""Fixture: SHA-256 of the streams the reference's `slicerng test` generates (TEST INFRASTRUCTURE ONLY).

    python oracle/gen_suite_streams.py      -> tests/golden/suite_streams_sha256.json   (needs /root/reference)

Runs the reference's own cli._suite_streams (pkg/src/slicerng/cli.py:212-231: 64-lane batches, batch seed =
master seed with its first byte XORed with the batch index, seedgen.derive_lane_material, mickey_sliced_words,
MSB-first packing) for a few (seed, streams, stream_bits) sets and records one digest per stream.  The GPU test
test_suite_streams_match_the_reference_cli compares `paper_1909_04750_b200.cli.suite_streams` with it; the
oracle restates the same construction in tests/test_oracle.py.
"""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mk2_numba_cache")
Path(os.environ["NUMBA_CACHE_DIR"]).mkdir(parents=True, exist_ok=True)
sys.path.insert(0, "/root/reference/pkg/src")
from slicerng import cli as rcli  # noqa: E402  (the reference)

CASES = [("11" * 32, 100, 4096), ("11" * 32, 3, 1_000_000), ("00" * 31 + "5a", 130, 1000), ("a7" + "00" * 31, 64, 77)]


def main():
    out = {"source": "slicerng.cli._suite_streams (reference)", "cases": []}
    for seed, streams, bits in CASES:
        args = argparse.Namespace(files=[], algo="mickey", seed=seed, streams=streams, stream_bits=bits)
        got = rcli._suite_streams(args)
        assert len(got) == streams and all(s.n == bits for s in got)
        out["cases"].append({"seed": seed, "streams": streams, "stream_bits": bits,
                             "first16": bytes(got[0].data[:16]).hex(),
                             "sha256": [hashlib.sha256(bytes(s.data)).hexdigest() for s in got]})
    (ROOT / "tests" / "golden" / "suite_streams_sha256.json").write_text(json.dumps(out) + "\n")
    print("wrote", sum(len(c["sha256"]) for c in out["cases"]), "digests")


if __name__ == "__main__":
    main()
