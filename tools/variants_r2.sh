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
    nocoop) build nocoop -DGSP_STAT_COOP=0 ;;
    hotcold) build hotcold -DGSP_HOTCOLD=1 ;;
    *) echo "unknown variant $v"; exit 1 ;;
  esac
done
ls variants
