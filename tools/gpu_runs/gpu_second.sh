#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
timeout 900 python tools/probe_occupancy.py 32768 > gpurun_out/probe2.log 2>&1; cat gpurun_out/probe2.log
# ncu: full capture of one launch of each keystream kernel (C2 geometry, 8192 clocks)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_colmajor -s 1 -c 1 -f -o gpurun_out/prof_col python tools/probe_one.py col 20 8192 > gpurun_out/ncu_col.log 2>&1; tail -3 gpurun_out/ncu_col.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor -s 1 -c 1 -f -o gpurun_out/prof_row python tools/probe_one.py row 20 8192 > gpurun_out/ncu_row.log 2>&1; tail -3 gpurun_out/ncu_row.log
timeout 900 python bench.py --steps 2 --warmup 3 --clocks 200000 --cpu-seconds 5 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err; tail -2 gpurun_out/bench_short.json; tail -5 gpurun_out/bench_short.err
