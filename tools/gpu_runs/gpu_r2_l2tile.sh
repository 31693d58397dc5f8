#!/bin/bash
# Grain row-major with the staging tile in L2-resident scratch (mk2_set_row_staging 3): parity spot check, then A/B
mkdir -p gpurun_out
python - <<'PY' 2>&1 | tail -5
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1909_04750_b200 import grain
from oracle import mickey_oracle as orc
for N, T, chunk in ((2048, 1536, 0), (1000, 520, 0), (4096 + 17, 2048 + 64, 512), (70000, 1024, 0)):
    rng = np.random.default_rng(N + T)
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8); ivs = rng.integers(0, 256, (N, 8), dtype=np.uint8)
    want = orc.grain_bulk_rowmajor(keys, ivs, T)
    with grain.GrainGenerator(0) as gen:
        gen.set_row_staging(3); gen.set_chunk_clocks(chunk)
        got = gen.init_material(keys, ivs).generate_rowmajor(T)
        lsb = gen.init_material(keys, ivs).generate_rowmajor(T, bit_order="lsb")
    print(N, T, chunk, "parity", np.array_equal(got, want), np.array_equal(lsb, orc.grain_bulk_rowmajor(keys, ivs, T, "lsb")), flush=True)
PY
for rep in 1 2; do
for st in 0 3; do python tools/probe_grain_row_once.py $st 0 3 2>&1 | tail -1; done
for lib in variants/libmk2_st0out2.so variants/libmk2_st1out0.so variants/libmk2_st0out0.so variants/libmk2_st1out1.so; do
  echo "lib=$lib"; MK2_LIB=$lib python tools/probe_grain_row_once.py 3 0 3 2>&1 | tail -1
done; done
for ch in 4096 65536; do python tools/probe_grain_row_once.py 3 $ch 3 2>&1 | tail -1; done
