#!/bin/bash
for d in ${DBGS:-0 3 7 11 15}; do
  SFC_OM_DEBUG=$d timeout 300 python bench.py --workload ${W:-4} --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('dbg $d', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
done
