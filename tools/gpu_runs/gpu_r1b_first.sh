#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 tools/probe_rblock.sh variants/libmk2_k1.so variants/libmk2_k5.so > gpurun_out/probe_rblock.txt 2>&1; cat gpurun_out/probe_rblock.txt
