#!/bin/bash
# live ncu traffic in the bench line; NCCL calls at world size 1 under torchrun; the staging-3 parity test
mkdir -p gpurun_out
(time python bench.py --steps 2 --warmup 3 --no-e2e --no-curand --no-cpu-baseline --no-latency) > gpurun_out/r02_bench_traffic_live.json 2> gpurun_out/r02_bench_traffic_live.err; echo "bench rc=$?"; tail -4 gpurun_out/r02_bench_traffic_live.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02_bench_traffic_live.json"))
for name, r in [("c2", d["roofline"])] + [(k, v["roofline"]) for k, v in d.get("extra_workloads", {}).items()]:
    print(name, r["traffic"], r.get("traffic_over_algorithmic"), r["traffic_model"], r.get("traffic_live_unavailable"), r["traffic_source"][:60])
PY
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 --extras none --no-e2e --no-curand --no-cpu-baseline --no-latency > gpurun_out/r02_bench_torchrun_1gpu.json 2> gpurun_out/r02_bench_torchrun.err; echo "torchrun rc=$?"; tail -3 gpurun_out/r02_bench_torchrun.err
python -c "
import json; d=json.load(open('gpurun_out/r02_bench_torchrun_1gpu.json')); print(d['value'], d['checksum_check'], d['ranks'])"
timeout 600 python -m pytest tests -m gpu -q -k "512_clock or two_ranks or multi_rank" 2>&1 | tail -3
