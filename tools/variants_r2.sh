#!/bin/bash
# Round-2 tuning variants of libgsp (same sources, different compile-time
# knobs) into variants/ (git-ignored; shipped to the GPU box by gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
rm -f variants/*.so
build() { python paper_2103_00959_b200/_build.py --force --out=variants/libgsp_$1.so ${@:2} > /dev/null; }
for v in "$@"; do
  case $v in
    base) build base ;;
    ls64) build ls64 -DGSP_STAT_LONG_SLICE=64 ;;
    ls256) build ls256 -DGSP_STAT_LONG_SLICE=256 ;;
    rawhi) build rawhi -DGSP_TC_RAWHI=1 ;;
    rawhi8) build rawhi8 -DGSP_TC_RAWHI=1 -DGSP_TC_XS=8 ;;
    rpw4) build rpw4 -DGSP_STAT_RPW=4 ;;
    rpw8) build rpw8 -DGSP_STAT_RPW=8 ;;
    med1) build med1 -DGSP_STAT_MED_TILES=1 ;;
    rpw32) build rpw32 -DGSP_STAT_RPW=32 ;;
    w4rpw32) build w4rpw32 -DGSP_STAT_WARPS=4 -DGSP_STAT_RPW=32 -DGSP_STAT_MINB=8 ;;
    *) echo "unknown variant $v"; exit 1 ;;
  esac
done
ls variants
