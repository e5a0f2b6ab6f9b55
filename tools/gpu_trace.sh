#!/bin/bash
# per-role clock trace of k_out_mma (OM_TRACE build): one forward of VGG-16 layer L
for d in ${DBGS:-0}; do
echo "== SFC_OM_DEBUG=$d"
SFC_OM_DEBUG=$d SFC_B200_LIB=$PWD/paper_2407_02913_b200/libsfc_tr.so python tools/prof_once.py --workload ${W:-4} --layer ${L:-1} --iters 1 --i8 2>&1 | grep -E "^u[ 0-9]" | tail -20
done
