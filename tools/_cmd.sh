python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2e.log 2>&1
timeout 900 python tools/ld_probe.py C4 C5 > gpurun_out/ld_probe_r2e.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:row_stats_warp<8, true, false>" -s 2 -c 1 -o gpurun_out/prof_stats_r2e -f python tools/gat_probe.py C3 > gpurun_out/ncu_stats_r2e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:row_stats_warp<8, false, true>" -s 1 -c 1 -o gpurun_out/prof_softmax_r2e -f python tools/gat_probe.py C3 > gpurun_out/ncu_softmax_r2e.log 2>&1
