#!/bin/bash
# One GPU iteration: gpu tests (log kept), timelines and benches for workloads 2 and 5.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/gpu_tests.log 2>&1
grep -E "FAILED|passed|failed|error" gpurun_out/gpu_tests.log | tail -5
for w in ${WORKLOADS:-2 5}; do
  python tools/timeline.py --workload $w --reps 1 2>&1 | tail -3
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_w$w.json 2>gpurun_out/bench_w$w.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/bench_w$w.json").read().strip().splitlines()[-1])
print("bench w$w", round(d["value"], 2), d["unit"], "ms/step", round(d["ms_per_step"], 4), "e2e", round(d["e2e"]["value"], 2))
PY
done
