#!/bin/bash
# Round-2 final validation on the B200, in the order the driver uses: smoke, GPU tests, both bench arms; then the
# builder-run extras (Grain, seed derivation) and the host-buffer probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/r02_smoke.log; tail -2 gpurun_out/r02_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log; tail -3 gpurun_out/r02_pytest_gpu.log
(time timeout 900 python bench.py --impl reference --steps 5 --warmup 1) > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "ref rc=$?"; tail -3 gpurun_out/r02_bench_reference_arm.err
(time timeout 1500 python bench.py --steps 5 --warmup 3) > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench_default.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02_bench_default.json"))
r = json.load(open("gpurun_out/r02_bench_reference_arm.json"))
print("c2", round(d["value"], 4), "frac", round(d["roofline"]["frac"], 4), "clocks", d["clocks"])
for k, v in d["extra_workloads"].items():
    print(k, round(v["value"], 4), "frac", round(v["roofline"]["frac"], 4), "whole step", round(v["step_split"]["whole_step_lop3_frac"], 4))
p = d["e2e_pageable"]
print("e2e", round(d["e2e"]["value"], 4), "GB/s", round(d["e2e"]["d2h_gb_s"], 1), "| pageable", round(p["value"], 4), "ratio", round(p["pageable_over_pinned"], 3),
      "fresh", round(p["fresh_over_pinned"], 3))
print("latency overhead us", round(d["small_call_latency"]["overhead_over_kernel_time_us"], 1), "ragged/uniform", round(d["ragged_init"]["ragged_over_uniform"], 3))
print("reference arm", r["value"], r["cpu_baseline"]["kind"], r["cpu_baseline"]["cores"], "-> e2e ratio", round(d["e2e"]["value"] / r["value"], 1), "kernel ratio", round(d["value"] / r["value"], 1))
PY
timeout 600 python tools/bench_extras.py > gpurun_out/r02_bench_extras_grain_seedgen.jsonl 2>&1; cut -c1-220 gpurun_out/r02_bench_extras_grain_seedgen.jsonl | head -4
