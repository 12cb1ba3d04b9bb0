#!/bin/bash
# Build tuning variants of libgsp (same sources, different compile-time knobs)
# into variants/ (git-ignored; shipped to the GPU box by gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
rm -f variants/*.so
build() { python paper_2103_00959_b200/_build.py --force --out=variants/libgsp_$1.so ${@:2} > /dev/null; }
build base
build stat_w4 -DGSP_STAT_WARPS=4 -DGSP_STAT_MINB=8
build gatpre_b4 -DGSP_GATPRE_MIN_BLOCKS=4
build l2hint -DGSP_L2HINT=1
build csr_normal -DGSP_CSR_EVICT_NORMAL
ls variants
