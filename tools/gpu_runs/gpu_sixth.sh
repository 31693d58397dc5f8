#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --workload c3 --steps 2 --warmup 3 --no-curand --cpu-seconds 4 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"; cut -c1-1800 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 1500 python bench.py --workload c5 --steps 3 --warmup 3 --no-curand --cpu-seconds 4 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"; cut -c1-1800 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --clocks 100000 --no-curand --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "torchrun rc=$?"; cut -c1-400 gpurun_out/bench_torchrun1.json; tail -3 gpurun_out/bench_torchrun1.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor -s 1 -c 1 -f -o gpurun_out/prof_row2 python tools/probe_one.py row 24 8192 > gpurun_out/ncu_row2.log 2>&1; tail -2 gpurun_out/ncu_row2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:init_kernel -c 1 -f -o gpurun_out/prof_init2 python tools/probe_one.py row 24 1024 > gpurun_out/ncu_init2.log 2>&1; tail -2 gpurun_out/ncu_init2.log
