#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python tools/probe_occupancy.py 65536 > gpurun_out/probe4.log 2>&1; cat gpurun_out/probe4.log
timeout 900 python bench.py --steps 2 --warmup 3 --clocks 200000 --cpu-seconds 5 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err; tail -2 gpurun_out/bench_short.json | cut -c1-1500; tail -5 gpurun_out/bench_short.err
