#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 tools/probe_rblock.sh > gpurun_out/probe_rblock3.txt 2>&1; cat gpurun_out/probe_rblock3.txt
timeout 600 python tools/probe_solo.py 2>&1 | head -8
timeout 1500 python bench.py --no-curand --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 1500 python bench.py --workload c3 --no-curand --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --workload c5 --no-curand --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json
for w in ("c2", "c3", "c5"):
    try:
        d = json.load(open(f"gpurun_out/bench_{w}.json"))
        r = d.get("roofline", {})
        print(w, "value", round(d["value"], 4), "ms/step", round(d["ms_per_step"], 2), "frac", round(r.get("frac", 0), 4),
              "frac327", round(r["at_survey_count"]["frac"], 4), "share", round(r.get("kernel_share_of_step", 0), 3),
              "e2e", round(d["e2e"]["value"], 4), "clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
    except Exception as e:
        print(w, "ERR", e)
PY
