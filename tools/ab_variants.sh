#!/bin/bash
# A/B the flooding pass across library variants built into _lib/variants/
# usage: tools/ab_variants.sh name1 name2 ...   (on a GPU box)
S='[[1, 512, 0, 2.0]]'
for r in 1 2; do
  for v in "$@"; do
    echo "== $v"
    FPH_LIB=paper_2509_22432_b200/_lib/variants/$v.so python tools/sweep.py sphere_torus_1m "$S" 2>&1 | grep '"ms"'
  done
done
