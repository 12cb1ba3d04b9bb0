#!/bin/bash
# initcheck on the default build; racecheck on the default and the debug-window-barrier builds
OUT=gpurun_out
PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_initcheck.log 2>&1
echo "initcheck exit=$? $(grep -E 'ERROR SUMMARY' $OUT/sanitize_initcheck.log | tr '\n' ' ')"
PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_racecheck.log 2>&1
echo "racecheck exit=$? $(grep -E 'RACECHECK SUMMARY' $OUT/sanitize_racecheck.log | tr '\n' ' ')"
GSP_LIB=$PWD/variants/libgsp_dbgwin.so PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_smoke.py > $OUT/sanitize_racecheck_dbg.log 2>&1
echo "racecheck(debug window barrier) exit=$? $(grep -E 'RACECHECK SUMMARY' $OUT/sanitize_racecheck_dbg.log | tr '\n' ' ')"
