#!/bin/bash
# A/B the column-major loop unroll factor (build-time knob MK2_COL_UNROLL) on C2 and full-occupancy geometry
for lib in "" variants/libmk2_u2.so variants/libmk2_u4.so; do
  echo "== lib=${lib:-default(unroll 1)}"
  for cfg in "20 262144 0 0" "20 262144 128 8192" "20 262144 256 1073741824"; do set -- $cfg
    MK2_LIB=$lib python tools/probe_one.py col $1 $2 $3 $4 2>&1 | tail -1
  done
  MK2_LIB=$lib python - <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_1909_04750_b200 as pkg
gen = pkg.MickeyGenerator(0); G = 148 * 8 * 32; T = 65536
gen.init_counter(bytes(10), 0, G * 32); out = torch.empty((T, G), dtype=torch.int32, device="cuda")
peak, _ = gen.lop3_peak()
for blk, chunk in ((256, 1 << 30), (128, 4096)):
    gen.set_block_threads(blk); gen.set_chunk_clocks(chunk)
    best = 1e9
    for _ in range(4):
        gen.generate_colmajor(T, out.data_ptr()); best = min(best, gen.last_kernel_ms)
    print("exact geometry", blk, chunk, "ms", round(best, 3), "frac", round(G * 32 * T * 327 / 32 / (best * 1e-3) / peak, 4))
PY
done
