#!/bin/bash
# Round profile set (under gpurun): bench line, ncu launch list of the bench,
# ncu --set full of the C4 SpMM, the C3 GAT aggregate and the C3 statistics kernel.
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:engine_kernel<.int.4, .int.32, gsp::WeightVal, gsp::RedSum, gsp::XF32" -s 5 -c 1 \
    -o $OUT/prof_spmm_$TAG -f python bench.py --steps 1 --warmup 5 --no-gat --no-cpu-baseline --no-e2e > $OUT/ncu_full_spmm_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:GatT<.bool.1>" \
    -s 3 -c 1 -o $OUT/prof_gat_$TAG -f python tools/gat_probe.py C3 > $OUT/ncu_full_gat_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:row_stats_warp<.int.8, .bool.1, .bool.0>" -s 3 -c 1 -o $OUT/prof_stats_$TAG -f \
    python tools/gat_probe.py C3 > $OUT/ncu_full_stats_$TAG.log 2>&1
echo done
