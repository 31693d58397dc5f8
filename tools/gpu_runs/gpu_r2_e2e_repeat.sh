for i in 1 2 3; do
python bench.py --steps 3 --warmup 3 --extras none --no-curand --no-cpu-baseline --no-latency --no-ncu-traffic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['e2e_pageable']; print('no extras: e2e %.4f (%.1f GB/s) pinned_same %.1f ms pageable %.3f fresh %.3f' % (d['e2e']['value'], d['e2e']['d2h_gb_s'], p['pinned_same_sample']['ms_per_step'], p['pageable_over_pinned'], p['fresh_over_pinned']))"
python bench.py --steps 3 --warmup 3 --no-curand --no-cpu-baseline --no-latency --no-ncu-traffic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['e2e_pageable']; print('with extras: e2e %.4f (%.1f GB/s) pinned_same %.1f ms pageable %.3f fresh %.3f' % (d['e2e']['value'], d['e2e']['d2h_gb_s'], p['pinned_same_sample']['ms_per_step'], p['pageable_over_pinned'], p['fresh_over_pinned']))"
done
