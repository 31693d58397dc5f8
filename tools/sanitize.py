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
    # round 2: ragged fast path (complete groups, 16-byte aligned) with unused lanes, LSB row order in both
    # MICKEY row kernels, derivation tag 2
    nb2 = nbits.copy()
    nb2[3] = nb2[77] = 0xFF
    colr2 = gen.init_ragged(keys[:1280], ivs[:1280], nb2[:1280]).generate_colmajor(96)
    lsb_t = gen.init_material(keys, ivs, 80).generate_rowmajor(T, bit_order="lsb")
    gen.set_row_staging(1)
    lsb_s = gen.init_material(keys, ivs, 80).generate_rowmajor(T, bit_order="lsb")
    gen.set_row_staging(0)
    kg, ig = gen.derive_material(bytes(range(32)), 0, 100, algo_tag=2)
    k2, i2 = gen.derive_material(bytes(range(32)), 5, 777)
    gen.init_seed(bytes(range(32)), 5, 777).generate_colmajor(64)
assert np.array_equal(col, orc.bulk_colmajor(keys, ivs, 80, T))
assert np.array_equal(row, orc.bulk_rowmajor(keys, ivs, 80, T))
assert np.array_equal(bulk, row) and np.array_equal(row_smem, row)
assert np.array_equal(colr, orc.bulk_colmajor(keys, ivs, nbits, T))
wk, wi = orc.derive_material(bytes(range(32)), 5, 777)
assert np.array_equal(k2, wk) and np.array_equal(i2, wi)
assert np.array_equal(lsb_t, lsb_s) and np.array_equal(lsb_t, np.packbits(np.unpackbits(row, axis=1), axis=1, bitorder="little"))
want2 = orc.bulk_colmajor(keys[:1280], ivs[:1280], np.where(nb2[:1280] == 0xFF, 0, nb2[:1280]).astype(np.uint8), 96)
lanes = np.ones(1280, bool); lanes[[3, 77]] = False
bits = lambda a: ((a[:, np.arange(1280) // 32] >> (np.arange(1280) % 32).astype(np.uint32)) & 1)[:, lanes]
assert np.array_equal(bits(colr2), bits(want2))
# pageable host outputs through the copy lanes (>= 64 MiB) and the opt-in Grain kernel with tensor-memory tiles
N2, T2 = (1 << 17) + 64, 4096
k3 = rng.integers(0, 256, (N2, 10), dtype=np.uint8)
i3 = rng.integers(0, 256, (N2, 10), dtype=np.uint8)
with pkg.MickeyGenerator(0) as gen:
    gen.set_stage_bytes(8 << 20)
    out = np.empty((T2, (N2 + 31) // 32), np.uint32)
    gen.init_material(k3, i3, 80).generate_colmajor(T2, out)
    rows = np.empty((N2, T2 // 8), np.uint8)
    gen.bulk_rowmajor(k3, i3, 80, T2, rows)
assert np.array_equal(out, orc.bulk_colmajor(k3, i3, 80, T2)) and np.array_equal(rows, orc.bulk_rowmajor(k3, i3, 80, T2))
from paper_1909_04750_b200 import grain
gk = rng.integers(0, 256, (N, 10), dtype=np.uint8)
gi = rng.integers(0, 256, (N, 8), dtype=np.uint8)
with grain.GrainGenerator(0) as gg:
    gg.set_row_staging(2)
    grow = gg.init_material(gk, gi).generate_rowmajor(1024 + 136)
assert np.array_equal(grow, orc.grain_bulk_rowmajor(gk, gi, 1024 + 136))
# Grain: default kernels (top-of-window realignment) in both layouts with a tail, and the mode-4 kernels (lone-warp
# ring kernel with three tiles per chunk + a one-tile chunk; circular-buffer column-major kernel)
with grain.GrainGenerator(0) as gg:
    gcol = gg.init_material(gk, gi).generate_colmajor(200)
    grow2 = gg.init_material(gk, gi).generate_rowmajor(392)
    gg.set_row_staging(4)
    gg.set_chunk_clocks(768)
    ring = gg.init_material(gk[:1280], gi[:1280]).generate_rowmajor(1024)
    circ = gg.init_material(gk, gi).generate_colmajor(208)
assert np.array_equal(gcol, orc.grain_bulk_colmajor(gk, gi, 200)) and np.array_equal(grow2, orc.grain_bulk_rowmajor(gk, gi, 392))
assert np.array_equal(ring, orc.grain_bulk_rowmajor(gk[:1280], gi[:1280], 1024))
assert np.array_equal(circ, orc.grain_bulk_colmajor(gk, gi, 208))
print("sanitize run ok")
