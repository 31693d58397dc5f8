"""One small-batch column-major launch for ncu: probe_small_once.py [instances] [clocks]"""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1909_04750_b200 as pkg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
T = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
rng = np.random.default_rng(1)
keys = rng.integers(0, 256, (n, 10), dtype=np.uint8); ivs = rng.integers(0, 256, (n, 10), dtype=np.uint8)
with pkg.MickeyGenerator(0) as gen:
    gen.init_material(keys, ivs, 80)
    for _ in range(2):
        gen.generate_colmajor(T)
    print(n, T, gen.last_plan(), "ms", gen.last_kernel_ms, "ns per clock", gen.last_kernel_ms * 1e6 / T)
