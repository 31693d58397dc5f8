#!/bin/bash
# five back-to-back runs of the default bench line on the final build: spread of the three workloads and the host-buffer legs
mkdir -p gpurun_out
out=gpurun_out/r02b_bench_repeatability.txt
echo "# five back-to-back runs of \`python bench.py --steps 5 --warmup 3 --no-curand --no-cpu-baseline\` on the final round-2 build" > $out
for i in 1 2 3 4 5; do
  python bench.py --steps 5 --warmup 3 --no-curand --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
e=d['extra_workloads']; p=d['e2e_pageable']
print('run $i: c2 %.4f Tb/s (frac %.4f)  c3 %.4f (%.4f)  c5 %.4f (%.4f, traffic %.3fx)  e2e %.4f  pageable/pinned %.3f  fresh/pinned %.3f  small call %.0f us  clocks %s MHz %s' % (
  d['value'], d['roofline']['frac'], e['c3']['value'], e['c3']['roofline']['frac'], e['c5']['value'], e['c5']['roofline']['frac'],
  e['c5']['roofline'].get('traffic_over_algorithmic') or 0, d['e2e']['value'], p['pageable_over_pinned'], p['fresh_over_pinned'],
  d['small_call_latency']['idle_context_reused_us']['best'], d['clocks']['sm_mhz'], d['clocks']['reasons']))" | tee -a $out
done
