#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "tensor_memory" > gpurun_out/pytest_tmem.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tmem.log; tail -15 gpurun_out/pytest_tmem.log
timeout 300 python - <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_1909_04750_b200 as pkg
for lg, T in ((22, 16384), (24, 8192)):
    n = 1 << lg
    out = torch.empty((n, T // 8), dtype=torch.uint8, device="cuda")
    for mode in (1, 2, 1, 2):
        gen = pkg.MickeyGenerator(0)
        gen.set_row_staging(mode)
        gen.init_counter(bytes.fromhex("123456789abcdef01234"), 0, n)
        ms = []
        for _ in range(3):
            gen.generate_rowmajor(T, out); ms.append(gen.last_kernel_ms)
        print("staging", mode, "n 2^%d T %d plan" % (lg, T), gen.last_plan(), "ms", round(min(ms), 3), "Tb/s", round(n * T / min(ms) / 1e9, 4), flush=True)
        gen.close()
PY
