#!/bin/bash
# Round-2 GPU iteration: gpu tests, default bench (config 4), config 5 / 2 benches, reference arm.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; lscpu | grep "Model name" >> gpurun_out/smi.txt
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -rf -x --durations=25 > gpurun_out/gpu_tests.log 2>&1
tail -40 gpurun_out/gpu_tests.log | grep -E "FAILED|passed|failed|error|s call" | tail -30
for w in ${WORKLOADS:-4 5 2}; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_w$w.json 2>gpurun_out/bench_w$w.err
  tail -c 1500 gpurun_out/bench_w$w.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
tail -c 800 gpurun_out/bench_ref.json
