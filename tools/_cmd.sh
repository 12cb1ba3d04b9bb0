python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2k.log 2>&1
SKIP_BENCH=1 SKIP_LAUNCH=1 OPS="C3" bash tools/gpu_measure.sh r2k
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ncu|C3-flickr-gat8x64|a5-a7_gat_fused/" -o gpurun_out/prof_gat_r2k -f python tools/ncu_ops.py C3 > gpurun_out/ncu_gat_r2k.log 2>&1
