#!/bin/bash
# Round-1 evidence run: full bench (C2), launch list, ncu --set full of both keystream kernels + init kernel.
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?"; cut -c1-2500 gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cut -c1-600 gpurun_out/bench_ref.json
# launch list of the bench command (short clocks so ncu's serialisation stays cheap)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --clocks 65536 --no-e2e --no-curand --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_c2.csv | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_colmajor -s 1 -c 1 -f -o gpurun_out/prof_col python tools/probe_one.py col 20 65536 > gpurun_out/ncu_col.log 2>&1; tail -2 gpurun_out/ncu_col.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor -s 1 -c 1 -f -o gpurun_out/prof_row python tools/probe_one.py row 24 8192 > gpurun_out/ncu_row.log 2>&1; tail -2 gpurun_out/ncu_row.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:init_kernel -c 1 -f -o gpurun_out/prof_init python tools/probe_one.py row 24 1024 > gpurun_out/ncu_init.log 2>&1; tail -2 gpurun_out/ncu_init.log
timeout 900 ncu --set full --clock-control none -k regex:lop3_peak -s 1 -c 1 -f -o gpurun_out/prof_peak python tools/probe_occupancy.py 256 > gpurun_out/ncu_peak.log 2>&1; tail -2 gpurun_out/ncu_peak.log
