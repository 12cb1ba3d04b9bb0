#!/bin/bash
# Time the fused GAT aggregate (C3) for every variants/libgsp_*.so
for lib in variants/libgsp_*.so; do
  tag=$(basename $lib .so)
  GSP_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gat_${tag}.json 2> gpurun_out/gat_${tag}.err
  python -c "import json; d=json.load(open('gpurun_out/gat_${tag}.json')); print('$tag', round(d['secondary']['C3_gat']['aggregate_ms'],3), 'spmm', round(d['ms_per_step'],3), 'l2peak', round(d['roofline_l2']['peak']))" 2>&1 | tail -1
done
