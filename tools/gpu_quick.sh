#!/bin/bash
# Quick GPU check: gpu tests, bench (default args), optional extra command.
# Usage (under gpurun): bash tools/gpu_quick.sh TAG [extra command...]
TAG=${1:-q}; shift
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py ${BENCH_ARGS} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
if [ $# -gt 0 ]; then timeout 900 bash -c "$*" > $OUT/extra_$TAG.log 2>&1; fi
tail -n 2 $OUT/pytest_gpu_$TAG.log
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print(d['ms_per_step'], d.get('e2e',{}).get('ms_per_step'), d['secondary']['C3_gat']['aggregate_ms'])"
