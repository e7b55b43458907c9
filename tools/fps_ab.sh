#!/bin/bash
# A/B farthest point sampling across library variants in _lib/variants/
# usage: tools/fps_ab.sh name1 name2 ...   (on a GPU box)
for r in 1 2; do
  for v in "$@"; do
    echo "== $v"
    FPH_LIB=paper_2509_22432_b200/_lib/variants/$v.so python tools/fps_time.py $FPS_ARGS 2>&1
  done
done
