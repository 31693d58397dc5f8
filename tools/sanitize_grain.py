#!/usr/bin/env python
"""compute-sanitizer run of the Grain kernels of the second half of round 2 (tools/sanitize.py has the rest and takes
memcheck longer than one sitting): default kernels with top-of-window realignment and in-register transposes (full
tiles, a partial tile, partial groups, unaligned rows), the lone-warp ring kernel and the circular-buffer kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1909_04750_b200 import grain
from oracle import mickey_oracle as orc

rng = np.random.default_rng(0)
N = 32 * 40 + 5
gk = rng.integers(0, 256, (N, 10), dtype=np.uint8)
gi = rng.integers(0, 256, (N, 8), dtype=np.uint8)
with grain.GrainGenerator(0) as gg:
    gcol = gg.init_material(gk, gi).generate_colmajor(200)
    grow = gg.init_material(gk, gi).generate_rowmajor(512 + 136)
    glsb = gg.init_material(gk[:1280], gi[:1280]).generate_rowmajor(512, bit_order="lsb")
    gg.set_row_staging(4)
    gg.set_chunk_clocks(768)
    ring = gg.init_material(gk[:1280], gi[:1280]).generate_rowmajor(1024)
    circ = gg.init_material(gk, gi).generate_colmajor(208)
with grain.GrainGenerator(0) as gg:   # eight-warp kernel: whole chains, three tiles in two chunks
    gg.set_row_staging(5)
    gg.set_chunk_clocks(512)
    row8 = gg.init_material(gk[:1024], gi[:1024]).generate_rowmajor(768)
assert np.array_equal(row8, orc.grain_bulk_rowmajor(gk[:1024], gi[:1024], 768))
assert np.array_equal(gcol, orc.grain_bulk_colmajor(gk, gi, 200))
assert np.array_equal(grow, orc.grain_bulk_rowmajor(gk, gi, 512 + 136))
assert np.array_equal(glsb, orc.grain_bulk_rowmajor(gk[:1280], gi[:1280], 512, "lsb"))
assert np.array_equal(ring, orc.grain_bulk_rowmajor(gk[:1280], gi[:1280], 1024))
assert np.array_equal(circ, orc.grain_bulk_colmajor(gk, gi, 208))
print("grain sanitize run ok")
