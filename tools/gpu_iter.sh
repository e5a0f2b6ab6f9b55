#!/bin/bash
# One build-measure iteration on the GPU box: targeted tests first, then the full GPU suite,
# then benches of the given workloads.
mkdir -p gpurun_out
if [ -n "$QUICK" ]; then
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "$QUICK" 2>&1 | tail -15
fi
if [ -z "$NOSUITE" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/gpu_tests.log 2>&1
  tail -15 gpurun_out/gpu_tests.log | grep -E "FAILED|passed|failed|Error|error" | tail -8
fi
for w in ${WORKLOADS:-4 5 2}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_w$w.json 2>gpurun_out/bench_w$w.err
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/bench_w$w.json").read().strip().splitlines()[-1])
    print("bench w$w", round(d["value"], 2), d["unit"], "ms/step", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 2), "stages", {k: round(v, 4) for k, v in d.get("stage_ms_per_step", {}).items()})
except Exception as e:
    print("bench w$w failed", e); print(open("gpurun_out/bench_w$w.err").read()[-2000:])
PY
done
if [ -n "$PERLAYER" ]; then timeout 300 python tools/per_layer.py --workload $PERLAYER --reps 3 2>&1 | tail -16; fi
