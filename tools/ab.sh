#!/bin/bash
# A/B of two library builds on one box: tools/ab.sh <config> <reps> <libA> <libB>
# (FPH_LIB selects the build the package loads); prints ms/step, e2e, phase warp-cycles.
cfg=$1; reps=$2; shift 2
for r in $(seq $reps); do
  for lib in "$@"; do
    FPH_LIB=$lib python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_tmp.json 2>/dev/null
    python -c "
import json,sys;d=json.load(open('gpurun_out/ab_tmp.json')); print('$cfg', '$(basename $lib)', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['roofline']['kernel_ms_per_step'],3), [round(x/1e9,2) for x in d['work_per_step']['search']['warp_cycles_a_b_c_f']])"
  done
done
