python tools/dbg_p24.py 2>&1 | grep -E "mismatches"
for w in 5 4 2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_w$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})"
done
