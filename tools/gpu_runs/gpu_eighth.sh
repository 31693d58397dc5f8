#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log
for cfg in "24 65536 0 0" "24 65536 256 0" "24 65536 128 0" "20 65536 0 0" "20 65536 192 0" "26 1024 0 0"; do set -- $cfg; timeout 300 python tools/probe_one.py row $1 $2 $3 $4 2>&1 | tail -1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor -s 1 -c 1 -f -o gpurun_out/prof_row3 python tools/probe_one.py row 24 8192 > gpurun_out/ncu_row3.log 2>&1; tail -2 gpurun_out/ncu_row3.log
