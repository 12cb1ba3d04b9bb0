#!/bin/bash
# ncu of the fused GAT kernel (C3) and of the SpMM at slab 64 (C4)
OUT=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:WeightGat -s 3 -c 1 -o $OUT/prof_gat_$1 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_gat_$1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:engine_kernel -s 5 -c 1 -o $OUT/prof_spmm64_$1 -f \
  python bench.py --steps 1 --warmup 5 --no-gat --no-cpu-baseline --no-e2e --slab-cols 64 > $OUT/ncu_spmm64_$1.log 2>&1
