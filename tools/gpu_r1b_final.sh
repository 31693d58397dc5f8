#!/bin/bash
# Round-1 (second half) final validation: smoke, GPU tests, the three bench workloads, reference arm, extras.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 1500 python bench.py --workload c3 --no-curand --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 1500 python bench.py --workload c5 --no-curand --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
python - <<'PY'
import json
for w in ("ref", "c2", "c3", "c5"):
    try:
        d = json.load(open(f"gpurun_out/bench_{w}.json"))
        r = d.get("roofline", {})
        print(w, "value", round(d["value"], 4), "ms/step", round(d["ms_per_step"], 2), "frac", round(r.get("frac", 0), 4),
              "frac327", round(r.get("at_survey_count", {}).get("frac", 0), 4), "share", round(r.get("kernel_share_of_step", 0), 3),
              "e2e", round(d["e2e"]["value"], 4), "clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
    except Exception as e:
        print(w, "ERR", e)
PY
timeout 600 python tools/bench_extras.py > gpurun_out/bench_extras.jsonl 2>&1; cut -c1-200 gpurun_out/bench_extras.jsonl | head -4
