"""Warp-per-group small-batch kernels (csrc/mk2_coop.cuh) against the thread-per-group throughput kernels: same
words, device time of init + T keystream clocks, by batch size.  usage: probe_small_batch.py [T]"""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1909_04750_b200 as pkg
from oracle import mickey_oracle as orc
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(7)
for N in (1, 32, 64, 1000, 4096, 16384, 32768, 65536, 131072, 262144):
    keys = rng.integers(0, 256, (N, 10), dtype=np.uint8); ivs = rng.integers(0, 256, (N, 10), dtype=np.uint8)
    res = {}
    with pkg.MickeyGenerator(0) as gen:
        for mode in (True, False):
            gen.set_small_batch(mode)
            best = 1e9
            for _ in range(3):
                gen.init_material(keys, ivs, 80); a = gen.last_kernel_ms
                col = gen.generate_colmajor(T); best = min(best, a + gen.last_kernel_ms)
            more = gen.generate_colmajor(37)               # resume, odd count
            res[mode] = (best, col.copy(), more.copy(), gen.checksum(), gen.last_plan())
    same = np.array_equal(res[True][1], res[False][1]) and np.array_equal(res[True][2], res[False][2]) and res[True][3] == res[False][3]
    ok = same
    if N <= 4096:
        ok = ok and np.array_equal(res[True][1], orc.bulk_colmajor(keys, ivs, 80, T))
    print(f"N={N:7d} T={T}: warp-per-group {res[True][0]:8.3f} ms {res[True][4]}  thread-per-group {res[False][0]:8.3f} ms {res[False][4]}  "
          f"speed-up {res[False][0] / res[True][0]:5.2f}  identical+oracle {ok}", flush=True)
    assert ok
