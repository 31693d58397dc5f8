#!/bin/bash
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gen_colmajor -s 1 -c 1 -f -o gpurun_out/prof_col_full python tools/probe_one.py col 20 1000000 > gpurun_out/ncu_col_full.log 2>&1; tail -2 gpurun_out/ncu_col_full.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_full.csv python bench.py --steps 2 --warmup 1 --no-curand --no-cpu-baseline > gpurun_out/launches_c2_full.log 2>&1; tail -1 gpurun_out/launches_c2_full.log | cut -c1-200
