#!/bin/bash
# Sparse plane 2 iteration: targeted parity first, the GPU suite, then A/B benches (dense vs sparse).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p24 or mma or config5 or config2" 2>&1 | tail -8
if [ -z "$NOSUITE" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/gpu_tests.log 2>&1
  tail -15 gpurun_out/gpu_tests.log | grep -E "FAILED|passed|failed|Error|error" | tail -8
fi
for kv in SFC_P2_DENSE=1 SFC_P2_DENSE=0; do
  for w in ${BW:-4 5 3}; do
    env $kv timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_${kv}_w$w.json 2>gpurun_out/bench_${kv}_w$w.err
    python -c "
import json; d=json.loads(open('gpurun_out/bench_${kv}_w$w.json').read().strip().splitlines()[-1]); print('$kv', 'w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
  done
done
