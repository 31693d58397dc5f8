python tools/probe_e2e_full.py 2 | tail -2
python bench.py --steps 3 --warmup 3 --extras none --no-curand --no-cpu-baseline --no-latency --no-ncu-traffic 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench e2e %.4f (%.1f GB/s) ms/step %.1f' % (d['e2e']['value'], d['e2e']['d2h_gb_s'], d['e2e']['ms_per_step']))"
python tools/probe_e2e_full.py 2 | tail -2
