#!/bin/bash
# same-box A/B of the in-tree build vs _ab_old/libdinfer.so (tools/ab_lib.sh):
# bench headline, alternating, 3 rounds.  usage: tools/ab_lib_bench.sh [bench args]
for r in 1 2 3; do
  for lib in old new; do
    if [ $lib = old ]; then export DINFER_LIB=_ab_old/libdinfer.so; else unset DINFER_LIB; fi
    python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']
print('r$r $lib step %.1f us  k12 %.1f  k34 %.1f  flushed %.1f' % (d['ms_per_step']*1e3, r['ms_per_launch']*1e3, d['phases_ms']['k34_select_smooth']*1e3, d['l2_flushed']['ms_per_step']*1e3))"
  done
done
