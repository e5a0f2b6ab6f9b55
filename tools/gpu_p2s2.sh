#!/bin/bash
mkdir -p gpurun_out
python tools/p2_flags.py --workload 4 2>&1 | tail -14
python tools/p2_flags.py --workload 5 --batch 64 2>&1 | tail -2
for kv in SFC_P2_DENSE=1 SFC_P2_DENSE=0; do echo $kv; env $kv python tools/per_layer.py --workload 4 --reps 5 2>&1 | tail -15; done
