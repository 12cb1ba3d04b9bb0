#!/bin/bash
# Round-2 closing measurement (under gpurun): -m gpu tests + smoke, the bench
# line with report rows, per-(config, op) ncu rows, the bench launch list, full
# captures of the C4 SpMM, the C3 row statistics and GAT aggregate and the C4
# layer-1 GEMM, and the compute-sanitizer pass.
TAG=${1:-r2i}
OUT=gpurun_out
mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
FULL_KERNEL=engine_kernel FULL_NAME=spmm_C4 bash tools/gpu_measure.sh $TAG
bash tools/gpu_full3.sh $TAG
bash tools/gpu_gemm_ncu.sh gemm_$TAG
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset)
echo done
