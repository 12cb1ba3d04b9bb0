#!/bin/bash
# Build tuning variants of libgsp (same sources, different compile-time knobs).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
rm -f variants/*.so
build() { python paper_2103_00959_b200/_build.py --force --out=variants/libgsp_$1.so ${@:2} > /dev/null & }
build gat_b4 -DGSP_GAT_MIN_BLOCKS=4
build gat_b3 -DGSP_GAT_MIN_BLOCKS=3
wait
ls variants
