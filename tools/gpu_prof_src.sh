# ncu --set full + source page of each per-call kernel of one layer (second forward):
# W (workload), L (layer), EXTRA (prof_once flags), KRES (kernel regexes)
mkdir -p gpurun_out/prof
for kre in ${KRES:-k_act_row k_gemm k_out_mma}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s ${SKIP:-1} -c 1 \
      -o gpurun_out/prof/src_$kre python tools/prof_once.py --workload $W --layer $L --iters 2 $EXTRA > gpurun_out/prof/src_$kre.log 2>&1
  echo "---- $kre"
  python tools/ncu_summary.py gpurun_out/prof/src_$kre.ncu-rep 2>&1 | grep -E "duration|dram__bytes|issue_active|warps_active|tensor|inst_executed|long_score|barrier_per|short_score|wait_per|mio_thr|lg_thr|sleeping"
  ncu -i gpurun_out/prof/src_$kre.ncu-rep --page source --csv > gpurun_out/prof/src_$kre.csv 2>/dev/null
  rm -f gpurun_out/prof/src_$kre.ncu-rep
done
