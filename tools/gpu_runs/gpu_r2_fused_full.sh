#!/bin/bash
# fused bulk kernel: full GPU test suite + default bench line (c5 now the one-shot call) + sanitizer on the new test
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log; tail -4 gpurun_out/r02_pytest_gpu.log
(time timeout 1500 python bench.py --steps 5 --warmup 3) > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench_default.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02_bench_default.json"))
print("c2", round(d["value"], 4), "frac", round(d["roofline"]["frac"], 4), "traffic/alg", d["roofline"].get("traffic_over_algorithmic"))
for k, v in d["extra_workloads"].items():
    print(k, round(v["value"], 4), "frac", round(v["roofline"]["frac"], 4), "whole step", round(v["step_split"]["whole_step_lop3_frac"], 4),
          "traffic/alg", v["roofline"].get("traffic_over_algorithmic"), v["roofline"].get("traffic_live_unavailable"))
print(json.dumps(d["extra_workloads"]["c5"]["step_split"])[:900])
PY
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "fused_kernel and not 2428935" > gpurun_out/r02_sanitizer_fused.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/r02_sanitizer_fused.log
