#!/bin/bash
# A/B of env settings on bench stages: AB="K=V K=V ..." (one bench per setting), BW workloads
for kv in ${AB:-X=0}; do
  for w in ${BW:-4}; do
    env $kv timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
    python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$kv w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
