#!/bin/bash
# Build tuning variants of libgsp (same sources, different compile-time knobs).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
rm -f variants/*.so
build() { python paper_2103_00959_b200/_build.py --force --out=variants/libgsp_$1.so ${@:2} > /dev/null & }
build base -DGSP_MIN_BLOCKS=4 -DGSP_UNROLL=8
build pipe4 -DGSP_MIN_BLOCKS=4 -DGSP_UNROLL=4 -DGSP_PIPE=1
build pipe8 -DGSP_MIN_BLOCKS=3 -DGSP_UNROLL=8 -DGSP_PIPE=1
build pipe2 -DGSP_MIN_BLOCKS=4 -DGSP_UNROLL=2 -DGSP_PIPE=1
wait
ls variants
