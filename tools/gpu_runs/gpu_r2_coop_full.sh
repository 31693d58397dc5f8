#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log; tail -5 gpurun_out/r02_pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "small_batch and not 65536" > gpurun_out/r02_sanitizer_coop.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r02_sanitizer_coop.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "small_batch and not 65536 and not 5000" > gpurun_out/r02_racecheck_coop.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r02_racecheck_coop.log
python bench.py --steps 1 --warmup 3 --extras none --no-e2e --no-curand --no-cpu-baseline --no-ncu-traffic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['small_call_latency'], indent=1))"
