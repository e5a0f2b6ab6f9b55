#!/bin/bash
# Round-2 profile capture (one GPU): default bench line, its ncu launch list, per-layer DRAM
# traffic of one config-4 forward, and --set full counters of the stage kernels of VGG-16
# layer 1 (kept-V schedule) and config 5 (recompute schedule).  Summaries: tools/summarize_r02.py
set -u
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_default.json 2> gpurun_out/prof/bench_default.err
tail -c 400 gpurun_out/prof/bench_default.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/prof/launches_w4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof/ncu_launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/prof/layers_w4.csv python tools/layer_launches.py --workload 4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/prof/layers_w5.csv python tools/layer_launches.py --workload 5 > /dev/null 2>&1
for spec in "4 1 --i8 3" "5 0 _ 4" "4 8 --i8 4"; do
  set -- $spec
  ex=$3; [ "$ex" = "_" ] && ex=""
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_act|k_quant|k_gemm|k_out" -s $4 -c $4 \
      -o gpurun_out/prof/full_w$1_l$2 python tools/prof_once.py --workload $1 --layer $2 --iters 1 $ex \
      > gpurun_out/prof/full_w$1_l$2.log 2>&1
  ncu -i gpurun_out/prof/full_w$1_l$2.ncu-rep --page raw --csv > gpurun_out/prof/full_w$1_l$2.raw.csv 2>/dev/null
  rm -f gpurun_out/prof/full_w$1_l$2.ncu-rep
done
ls -la gpurun_out/prof; du -sh gpurun_out/prof
