#!/bin/bash
# out_mma iteration: targeted parity, benches, instruction counts of the output kernel on VGG layer 1
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "p24 or mma or config5 or config2 or requant or stack" 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_stacks.py -q -x -k "cfg4_layer1 or cfg4_layer8 or cfg3_layer0 or cfg3_layer12" 2>&1 | tail -3
for w in ${BW:-4 5 3}; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/bench_w$w.json 2>gpurun_out/bench_w$w.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" 2>&1 | tail -1
done
if [ -n "$PROF" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_out_mma|k_gemm|k_act_row" -s 3 -c 3 python tools/prof_once.py --workload 4 --layer 1 --iters 2 --i8 2>&1 | grep -E "k_out_mma|k_gemm|k_act_row|duration|inst_executed|issue_active"
fi
