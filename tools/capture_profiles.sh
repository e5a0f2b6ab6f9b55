#!/bin/bash
# Round profile capture (run under gpurun, one GPU): plain bench first, then the ncu launch
# list of the same default bench command, then one `--set full` capture per workload and
# variant of the four per-call kernels (second forward of tools/prof_once.py).
set -u
mkdir -p gpurun_out/prof
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_plain.json 2> gpurun_out/prof/bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/prof/launches_w2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launches.log 2>&1
for w in 2 5; do
  # stage kernels per forward matched by the regex: kept-V schedule (w2) 3, recompute (w5) 4
  n=$([ $w = 5 ] && echo 4 || echo 3)
  for v in sfc4-4x4-3x3 sfc6-6x6-3x3 sfc6-7x7-3x3; do
    python tools/prof_once.py --workload $w --variant $v --iters 2 > /dev/null 2>&1 || continue
    ncu --set full --import-source on --clock-control none -k regex:"k_act|k_quant|k_gemm|k_output" -s $n -c $n \
        -o gpurun_out/prof/full_w${w}_${v} python tools/prof_once.py --workload $w --variant $v --iters 2 \
        > gpurun_out/prof/ncu_full_w${w}_${v}.log 2>&1
  done
done
ls gpurun_out/prof | wc -l
# shrink for the 64 MiB copy-back: raw metric pages as CSV, keep one report for source views
for r in gpurun_out/prof/full_*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  case "$r" in *w2_sfc6-6x6-3x3*) ;; *) rm -f "$r" ;; esac
done
du -sh gpurun_out/prof
