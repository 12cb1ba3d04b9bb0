python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2i.log 2>&1
bash tools/sanitize.sh > gpurun_out/sanitize_r2i.txt 2>&1
SKIP_LAUNCH=1 bash tools/gpu_measure.sh r2i
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2i.csv python bench.py --steps 3 --warmup 3 --no-rows --no-secondary --no-e2e > gpurun_out/ncu_launch_bench_r2i.log 2>&1
