#!/bin/bash
# ncu --set full + source/SASS page of chosen kernels of one layer: W, L, KRES, EXTRA
mkdir -p gpurun_out/prof
for kre in ${KRES:-k_out_mma}; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s ${SKIP:-1} -c 1 \
      -o gpurun_out/prof/src_$kre python tools/prof_once.py --workload $W --layer $L --iters 2 $EXTRA > gpurun_out/prof/src_$kre.log 2>&1
  echo "---- $kre"
  python tools/ncu_summary.py gpurun_out/prof/src_$kre.ncu-rep 2>&1 | grep -E "duration|dram__bytes|issue_active|warps_active|tensor|inst_executed|long_score|barrier_per|short_score|wait_per|mio_thr|lg_thr|sleeping|math_pipe|membar|dispatch|no_inst|branch|tex_thr|selected|not_sel"
  python tools/ncu_hot.py gpurun_out/prof/src_$kre.ncu-rep "$kre" 60 > gpurun_out/prof/hot_$kre.txt 2>&1
  ncu -i gpurun_out/prof/src_$kre.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/sass_$kre.csv 2>/dev/null
  ls -la gpurun_out/prof/src_$kre.ncu-rep
done
