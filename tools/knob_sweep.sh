#!/bin/bash
# same-box sweep of one env knob on the bench headline, alternating, 3 rounds:
#   tools/knob_sweep.sh VAR "values" [bench args]
var=$1; vals=$2; shift 2
for r in 1 2 3; do
  for v in $vals; do
    env $var=$v python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']
print('r$r $var=$v step %.1f us  dominant %.1f us (frac %.3f)  k34 %.1f  flushed %.1f' % (d['ms_per_step']*1e3, r['ms_per_launch']*1e3, r['frac'], d['phases_ms']['k34_select_smooth']*1e3, d['l2_flushed']['ms_per_step']*1e3))"
  done
done
