#!/bin/bash
# Full ncu captures (under gpurun) of the C3 GAT kernels: the row statistics
# (GAT statistics launch, then the standalone edge softmax) and the fused
# aggregate, driven by tools/ncu_ops.py C3.
# Usage: bash tools/gpu_full3.sh TAG
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:row_stats_warp -c 2 -o $OUT/prof_rowstats_C3_$TAG -f python tools/ncu_ops.py C3 > $OUT/ncu_rowstats_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:WeightAlphaHM -c 1 -o $OUT/prof_gat_C3_$TAG -f python tools/ncu_ops.py C3 > $OUT/ncu_gat_$TAG.log 2>&1
echo done
