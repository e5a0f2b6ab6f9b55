# A/B of env knobs on bench stages: AB="NAME=v1 NAME=v2 ..." (one bench per setting)
python tools/dbg_p24.py 2>&1 | grep -E "mismatches"
for kv in ${AB:-X=0}; do
  for w in ${BW:-5 4}; do
    env $kv timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_w$w.json 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('$kv', 'w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
