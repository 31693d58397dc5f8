#!/usr/bin/env python
"""Small end-to-end run of every kernel for compute-sanitizer (memcheck / racecheck / initcheck)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1909_04750_b200 as pkg
from oracle import mickey_oracle as orc

rng = np.random.default_rng(0)
N, T = 32 * 40 + 5, 392
keys = rng.integers(0, 256, (N, 10), dtype=np.uint8)
ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
nbits = rng.integers(0, 81, N, dtype=np.uint8)
with pkg.MickeyGenerator(0) as gen:
    gen.set_chunk_clocks(128)
    col = gen.init_material(keys, ivs, 80).generate_colmajor(T)
    row = gen.init_material(keys, ivs, 80).generate_rowmajor(T)
    colr = gen.init_ragged(keys, ivs, nbits).generate_colmajor(T)
    gen.init_counter(bytes(range(10)), 64, N)
    gen.generate_rowmajor(T)
    gen.clock(True, None, 3)
    gen.checksum()
    bulk, bsum = gen.bulk_rowmajor(keys, ivs, 80, T)
    gen.set_row_staging(1)
    row_smem = gen.init_material(keys, ivs, 80).generate_rowmajor(T)
    gen.set_row_staging(0)
    k2, i2 = gen.derive_material(bytes(range(32)), 5, 777)
    gen.init_seed(bytes(range(32)), 5, 777).generate_colmajor(64)
assert np.array_equal(col, orc.bulk_colmajor(keys, ivs, 80, T))
assert np.array_equal(row, orc.bulk_rowmajor(keys, ivs, 80, T))
assert np.array_equal(bulk, row) and np.array_equal(row_smem, row)
assert np.array_equal(colr, orc.bulk_colmajor(keys, ivs, nbits, T))
wk, wi = orc.derive_material(bytes(range(32)), 5, 777)
assert np.array_equal(k2, wk) and np.array_equal(i2, wi)
print("sanitize run ok")
