# ncu --set full of the per-call kernels of VGG-16 layers (config 4), second forward.
mkdir -p gpurun_out/prof
for l in ${LAYERS:-1 0 8}; do
  python tools/prof_once.py --workload 4 --layer $l --i8 --iters 1 > /dev/null 2>&1 || { echo "layer $l failed"; continue; }
  n=3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_act|k_quant|k_gemm|k_output" -s $n -c $n \
      -o gpurun_out/prof/full_w4_l$l python tools/prof_once.py --workload 4 --layer $l --i8 --iters 1 \
      > gpurun_out/prof/ncu_full_w4_l$l.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof/full_w4_l$l.ncu-rep > gpurun_out/prof/full_w4_l$l.txt 2>&1
  cat gpurun_out/prof/full_w4_l$l.txt
done
du -sh gpurun_out/prof
