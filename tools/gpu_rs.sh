#!/bin/bash
# Row-statistics iteration (under gpurun): GAT / softmax parity tests, C3
# timings, per-launch ncu metrics and a full capture of the three C3 launches.
TAG=${1:-rs}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "gat or softmax or stat or alpha or backward or infer" > $OUT/pytest_$TAG.log 2>&1
tail -2 $OUT/pytest_$TAG.log
python tools/variant_probe.py C3 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_stats_warp -c 3 -o $OUT/prof_rs_$TAG -f \
    python tools/ncu_ops.py C3 > $OUT/ncu_rs_$TAG.log 2>&1
echo done
