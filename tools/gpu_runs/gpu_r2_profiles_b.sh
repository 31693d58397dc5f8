#!/bin/bash
# Round 2, second half: ncu launch list of the default bench command (c5 is now the fused one-shot kernel), ncu --set full
# capture of the fused kernel at config 5's full size, summaries only.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_ncu_launches_bench_default.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-curand --no-cpu-baseline --no-latency --no-ncu-traffic > /tmp/ncu_bench.json 2> /tmp/ncu_bench.err; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:bulk_rowmajor_kernel --launch-skip 3 --launch-count 1 -f -o /tmp/r02b_c5 \
    python bench.py --workload c5 --extras none --steps 1 --warmup 3 --no-e2e --no-curand --no-cpu-baseline --no-latency --no-ncu-traffic > /dev/null 2> /tmp/ncu_c5.err; echo "ncu c5 rc=$?"; tail -2 /tmp/ncu_c5.err
python tools/ncu_summary.py /tmp/r02b_c5.ncu-rep gpurun_out/r02b_ncu_fused_bulk_c5_full.txt "fused::bulk_rowmajor_kernel, BASELINE config 5 at full size (2^26 key/IV pairs x 1024 bits): records -> input words (tensor memory) -> load + pre-clocks -> keystream -> rows in one launch" | tail -45
ncu -i /tmp/r02b_c5.ncu-rep --page source --csv > /tmp/src.csv 2>/dev/null; python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/src.csv")))
print("source page rows", len(rows)); print(rows[0][:12] if rows else None)
PY
