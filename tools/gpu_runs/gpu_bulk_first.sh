#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_bulk.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bulk.log; tail -15 gpurun_out/pytest_bulk.log
timeout 600 python - <<'PY'
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch, paper_1909_04750_b200 as pkg
KEY = bytes.fromhex("123456789abcdef01234")
for n, tc in ((1 << 24, 1024), (1 << 20, 16384), (1 << 22, 4096)):
    keys = torch.from_numpy(np.tile(np.frombuffer(KEY, np.uint8), (n, 1))).pin_memory()
    ivs_np = np.zeros((n, 10), np.uint8); ivs_np[:, 2:] = np.arange(n, dtype=np.uint64).astype(">u8").view(np.uint8).reshape(n, 8)
    ivs = torch.from_numpy(ivs_np).pin_memory()
    host = torch.empty((n, tc // 8), dtype=torch.uint8).pin_memory()
    gen = pkg.MickeyGenerator(0)
    def two():
        gen.init_material(keys, ivs, 80); gen.generate_rowmajor(tc, host)
    def one():
        gen.bulk_rowmajor(keys, ivs, 80, tc, host)
    for name, fn in (("init+generate", two), ("bulk", one), ("init+generate", two), ("bulk", one)):
        fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3): fn()
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
        print(f"n=2^{n.bit_length()-1} T={tc} {name}: {dt*1e3:.2f} ms/step {n*tc/dt/1e12:.4f} Tb/s", flush=True)
    gen.close()
PY
