python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2f.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "softmax or gat or validate or GAT or sddmm" > gpurun_out/pytest_r2f.log 2>&1; echo "exit $?" >> gpurun_out/pytest_r2f.log
python tools/gat_probe.py C3 > gpurun_out/gat_probe_r2f.json 2>&1
LDS=604,608,616,624,632,640,672,704,768,1024 SLABS=0 timeout 900 python tools/ld_probe.py C4 > gpurun_out/ld_probe_r2f_c4.txt 2>&1
LDS=300,304,320,352,384,512 SLABS=0 timeout 900 python tools/ld_probe.py C5 > gpurun_out/ld_probe_r2f_c5.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ncu|C3-flickr-gat8x64|a5-a7_gat_fused/" -o gpurun_out/prof_gat_r2f -f python tools/ncu_ops.py C3 > gpurun_out/ncu_gat_r2f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "ncu|C3-flickr-gat8x64|a6_edge_softmax/" -o gpurun_out/prof_softmax_r2f -f python tools/ncu_ops.py C3 > gpurun_out/ncu_softmax_r2f.log 2>&1
