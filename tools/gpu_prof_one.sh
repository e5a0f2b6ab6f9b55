# ncu --set full of one kernel (regex $KRE) in tools/prof_once.py --workload $W --layer $L [$EXTRA]
mkdir -p gpurun_out/prof
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$KRE" -s ${SKIP:-1} -c 1 \
    -o gpurun_out/prof/one python tools/prof_once.py --workload $W --layer $L --iters 2 $EXTRA > gpurun_out/prof/one.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/one.ncu-rep 2>&1 | grep -E "^----|duration|dram__bytes|issue_active|warps_active|tensor|inst_executed|long_score|barrier_per|short_score|wait_per|math_pipe|sleeping"
ncu -i gpurun_out/prof/one.ncu-rep --page source --csv > gpurun_out/prof/one_src.csv 2>/dev/null
ncu -i gpurun_out/prof/one.ncu-rep --page raw --csv > gpurun_out/prof/one_raw.csv 2>/dev/null
rm -f gpurun_out/prof/one.ncu-rep
