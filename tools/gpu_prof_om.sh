mkdir -p gpurun_out/prof
python tools/dbg_p24.py 2>&1 | grep -E "mismatches"
for w in ${BW:-5 4}; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_w$w.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_w$w.json').read().strip().splitlines()[-1]); print('w$w', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})"
done
for spec in ${SPECS:-"5 0" "4 1"}; do
  set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_out_mma|k_gemm" -s 2 -c 2 \
      -o gpurun_out/prof/om_w$1_l$2 python tools/prof_once.py --workload $1 --layer $2 --iters 2 $([ $1 = 4 ] && echo --i8) > gpurun_out/prof/om_w$1_l$2.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/om_w$1_l$2.ncu-rep 2>&1 | grep -E "^----|duration|dram__bytes|issue_active|warps_active|tensor|inst_executed|lts__t_bytes|long_score|barrier_per|short_score|wait_per|mio_thr|lg_thr|math_pipe|sleeping|membar"
  ncu -i gpurun_out/prof/om_w$1_l$2.ncu-rep --page source --csv --kernel-name regex:k_out_mma > gpurun_out/prof/om_src_w$1.csv 2>/dev/null
  rm -f gpurun_out/prof/om_w$1_l$2.ncu-rep
done
ls -la gpurun_out/prof
