#!/bin/bash
# A/B the clock_block length (build-time knob MK2_RBLOCK; variants/libmk2_k<K>.so) on C2 geometry,
# full-occupancy column-major, row-major and the init kernel.
for lib in "" "$@"; do
  echo "== lib=${lib:-default}"
  MK2_LIB=$lib python tools/probe_one.py col 20 262144 0 0 2>&1 | tail -1
  MK2_LIB=$lib python tools/probe_one.py row 22 16384 0 0 2>&1 | tail -1
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
    print("exact geometry", blk, chunk, "ms", round(best, 3), "frac(327)", round(G * 32 * T * 327 / 32 / (best * 1e-3) / peak, 4))
# init-dominated: 2^24 fresh key/IV pairs (device-resident material)
n = 1 << 24
keys = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device="cuda"); ivs = torch.randint(0, 256, (n, 10), dtype=torch.uint8, device="cuda")
gen2 = pkg.MickeyGenerator(0); gen2.set_stream(torch.cuda.current_stream().cuda_stream)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    ev[0].record(); gen2.init_material(keys, ivs, 80); ev[1].record(); torch.cuda.synchronize()
print("init 2^24 x (80+80+100 clocks) ms", round(ev[0].elapsed_time(ev[1]), 3))
PY
done
