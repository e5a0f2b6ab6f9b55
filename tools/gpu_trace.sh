#!/bin/bash
# per-role clock traces (OM_TRACE / GM_TRACE build libsfc_tr.so): one forward of workload W layer L;
# PAT selects the lines (u = output transform, g = GEMM)
for d in ${DBGS:-0}; do
echo "== SFC_OM_DEBUG=$d"
SFC_OM_DEBUG=$d SFC_B200_LIB=$PWD/paper_2407_02913_b200/libsfc_tr.so python tools/prof_once.py --workload ${W:-4} --layer ${L:-1} --iters 1 ${EXTRA:---i8} 2>&1 | grep -E "^[${PAT:-u}][ 0-9]" | tail -20
done
