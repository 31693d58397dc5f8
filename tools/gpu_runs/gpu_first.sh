#!/bin/bash
# First GPU visit: parity tests, smoke, occupancy probe, short + full bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/gpu.csv 2>&1
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/host.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -3 gpurun_out/smoke.log
timeout 600 python tools/probe_occupancy.py 32768 > gpurun_out/probe.log 2>&1; tail -30 gpurun_out/probe.log
timeout 600 python bench.py --steps 2 --warmup 3 --clocks 100000 --cpu-seconds 5 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err; tail -2 gpurun_out/bench_short.json; tail -5 gpurun_out/bench_short.err
