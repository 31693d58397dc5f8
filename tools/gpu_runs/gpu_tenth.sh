#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for tool in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log; tail -4 gpurun_out/sanitizer_$tool.log
done
timeout 1200 ncu --set full --clock-control none -k regex:gen_colmajor -s 1 -c 1 -f -o gpurun_out/prof_col_full python tools/probe_one.py col 20 1000000 > gpurun_out/ncu_col_full.log 2>&1; tail -2 gpurun_out/ncu_col_full.log
