#!/bin/bash
# e2e_pageable of the bench line by the number of copy lanes a contiguous tile uses (MK2_LANE_WIDE), two runs each.
mkdir -p gpurun_out
for rep in 1 2; do for w in 8 12 16; do
  MK2_LANE_WIDE=$w python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-curand --no-latency --no-ncu-traffic --extras none 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); p=d['e2e_pageable']
print('MK2_LANE_WIDE=$w', 'pageable GB/s', round(p['d2h_gb_s'],1), 'ratio', round(p['pageable_over_pinned'],3), 'fresh', round(p['fresh_over_pinned'],3), 'pinned e2e GB/s', round(d['e2e']['d2h_gb_s'],1))"
done; done
