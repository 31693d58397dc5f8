#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
for tool in memcheck racecheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python tools/sanitize.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log; tail -3 gpurun_out/sanitizer_$tool.log
done
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
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_rowmajor -s 1 -c 1 -f -o gpurun_out/prof_row python tools/probe_one.py row 24 8192 > gpurun_out/ncu_row.log 2>&1; tail -1 gpurun_out/ncu_row.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_colmajor -s 1 -c 1 -f -o gpurun_out/prof_col python tools/probe_one.py col 20 65536 > gpurun_out/ncu_col.log 2>&1; tail -1 gpurun_out/ncu_col.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:init_kernel -s 1 -c 1 -f -o gpurun_out/prof_init python tools/probe_one.py col 24 64 > gpurun_out/ncu_init.log 2>&1; tail -1 gpurun_out/ncu_init.log
