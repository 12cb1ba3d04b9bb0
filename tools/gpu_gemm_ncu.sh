#!/bin/bash
# ncu --set full capture of the tcgen05 GEMM on the C4 layer-1 shape (one launch)
OUT=gpurun_out; TAG=${1:-gemm}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:linear_tc_kernel -s 3 -c 1 \
  -o $OUT/prof_$TAG -f python tools/linear_probe.py > $OUT/ncu_$TAG.log 2>&1
ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
ncu -i $OUT/prof_$TAG.ncu-rep --page details --csv > $OUT/details_$TAG.csv 2>/dev/null
