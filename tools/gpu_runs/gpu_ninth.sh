#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -4 gpurun_out/pytest_gpu.log
for cfg in "24 65536 0 0" "24 65536 256 0" "20 65536 0 0" "26 1024 0 0"; do set -- $cfg; timeout 300 python tools/probe_one.py row $1 $2 $3 $4 2>&1 | tail -1; done
timeout 600 python tools/nist_sample.py 2>&1 | tail -3
