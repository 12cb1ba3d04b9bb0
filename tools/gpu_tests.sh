#!/bin/bash
# GPU test pass (under gpurun): build, -m gpu tests, smoke.
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> $OUT/smoke_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
