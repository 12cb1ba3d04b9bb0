#!/bin/bash
# One measurement session (under gpurun): build, bench line, per-(config, op)
# ncu metrics, the ncu launch list of the bench, and a full capture of the top kernel.
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nproc > $OUT/nproc_$TAG.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/nproc_$TAG.txt; free -g >> $OUT/nproc_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} --report $OUT/report_$TAG.jsonl > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
fi
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sector_hit_rate.pct
if [ -z "$SKIP_ROWS" ]; then
  timeout 1200 ncu --nvtx --print-nvtx-rename kernel --clock-control none --cache-control all --metrics $M --csv \
      --log-file $OUT/ncu_ops_$TAG.csv python tools/ncu_ops.py ${OPS} > $OUT/ncu_ops_$TAG.log 2>&1
  python tools/ncu_rows.py $OUT/ncu_ops_$TAG.csv $OUT/${TAG}_ncu_rows.json > $OUT/ncu_rows_$TAG.txt 2>&1
fi
if [ -z "$SKIP_LAUNCH" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
      python bench.py --steps 3 --warmup 3 --no-rows --no-secondary --no-e2e > $OUT/ncu_launch_bench_$TAG.log 2>&1
fi
if [ -n "$FULL_KERNEL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$FULL_KERNEL" -s ${FULL_SKIP:-5} -c 1 -o $OUT/prof_${FULL_NAME:-top}_$TAG -f \
      python bench.py --steps 1 --warmup 5 --no-rows --no-secondary --no-e2e > $OUT/ncu_full_$TAG.log 2>&1
fi
echo done
