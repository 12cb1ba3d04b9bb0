#!/bin/bash
# Time every variants/libgsp_*.so on the C4 SpMM at several slab widths.
OUT=gpurun_out
mkdir -p $OUT
for lib in variants/libgsp_*.so; do
  tag=$(basename $lib .so)
  GSP_LIB=$PWD/$lib timeout 300 python bench.py --config ${CONFIG:-C4} --steps 10 --warmup 3 --no-gat --no-cpu-baseline --no-e2e \
     --sweep ${SWEEP:-32,64,128} > $OUT/sweep_${CONFIG:-C4}_${tag}.json 2> $OUT/sweep_${CONFIG:-C4}_${tag}.err
  python -c "import json,sys; d=json.load(open('$OUT/sweep_${CONFIG:-C4}_${tag}.json')); print('$tag', {k:round(v['ms'],3) for k,v in d['sweep_slab_cols'].items()})" 2>&1
done
