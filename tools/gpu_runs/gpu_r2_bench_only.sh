mkdir -p gpurun_out
(time timeout 1500 python bench.py --steps 5 --warmup 3) > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"; tail -3 gpurun_out/r02_bench_default.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02_bench_default.json"))
print("c2", round(d["value"], 4), "frac", round(d["roofline"]["frac"], 4), "traffic/alg", d["roofline"].get("traffic_over_algorithmic"))
for k, v in d["extra_workloads"].items():
    print(k, round(v["value"], 4), "frac", round(v["roofline"]["frac"], 4), "whole step", round(v["step_split"]["whole_step_lop3_frac"], 4),
          "traffic/alg", v["roofline"].get("traffic_over_algorithmic"), v["roofline"].get("traffic_live_unavailable"))
print(json.dumps(d["extra_workloads"]["c5"]["step_split"])[:900])
p = d["e2e_pageable"]; print("e2e", d["e2e"]["value"], "pageable ratio", p["pageable_over_pinned"], "fresh", p["fresh_over_pinned"])
PY
