#!/bin/bash
# initcheck and racecheck on the default build; racecheck on the per-row-wait variant
# (variants/libgsp_rowwait.so, built with -DGSP_WINDOW_PER_ROW_WAIT)
OUT=gpurun_out
PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_initcheck.log 2>&1
echo "initcheck exit=$? $(grep -E 'ERROR SUMMARY' $OUT/sanitize_initcheck.log | tr '\n' ' ')"
PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_racecheck.log 2>&1
echo "racecheck exit=$? $(grep -E 'RACECHECK SUMMARY' $OUT/sanitize_racecheck.log | tr '\n' ' ')"
if [ -f variants/libgsp_rowwait.so ]; then
GSP_LIB=$PWD/variants/libgsp_rowwait.so PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_racecheck_rowwait.log 2>&1
echo "racecheck(per-row window waits) exit=$? $(grep -E 'RACECHECK SUMMARY' $OUT/sanitize_racecheck_rowwait.log | tr '\n' ' ')"
fi
