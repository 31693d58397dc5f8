#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -6 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --workload c5 --steps 3 --warmup 3 --no-curand --cpu-seconds 4 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"; cut -c1-2400 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 1500 python bench.py --workload c3 --steps 2 --warmup 3 --no-curand --cpu-seconds 4 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['value'], d['roofline']['frac'], d['e2e'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --clocks 100000 --no-curand --no-cpu-baseline > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "torchrun rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_torchrun1.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'], d['e2e'])"
