#!/bin/bash
# One GPU session: tests, bench, ncu launch list and a full capture of the SpMM kernel.
# Usage (from repo root, under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py ${BENCH_ARGS} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 5 -c 1 \
    -o $OUT/prof_spmm_$TAG -f python bench.py --steps 1 --warmup 5 --no-gat --no-cpu-baseline --no-e2e > $OUT/ncu_full_$TAG.log 2>&1
echo done
