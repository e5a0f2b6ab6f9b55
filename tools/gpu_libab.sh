#!/bin/bash
# A/B of library builds on bench stages: LIBS="name ..." (paper_2407_02913_b200/libsfc_<name>.so), BW workloads
for l in ${LIBS:-b200}; do
  for w in ${BW:-4}; do
    SFC_B200_LIB=$PWD/paper_2407_02913_b200/libsfc_$l.so timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 ${BARGS} > gpurun_out/b.json 2>gpurun_out/b.err
    python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print('$l w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
