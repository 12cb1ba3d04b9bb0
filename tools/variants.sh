#!/bin/bash
# Build tuning variants of libgsp (same sources, different compile-time knobs).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
build() { python paper_2103_00959_b200/_build.py --force --out=variants/libgsp_$1.so ${@:2} > /dev/null & }
build mb5u4 -DGSP_MIN_BLOCKS=5 -DGSP_UNROLL=4
build mb3u8 -DGSP_MIN_BLOCKS=3 -DGSP_UNROLL=8
build mb4u8 -DGSP_MIN_BLOCKS=4 -DGSP_UNROLL=8
build mb4u4 -DGSP_MIN_BLOCKS=4 -DGSP_UNROLL=4
wait
ls -la variants
