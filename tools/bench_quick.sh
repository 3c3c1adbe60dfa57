#!/bin/bash
# Quick bench sweep (no cpu baseline): tools/bench_quick.sh TAG config...
TAG=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  python bench.py --no-cpu-baseline --config $c > gpurun_out/q_${TAG}_$c.json 2>/dev/null
  python -c "
import json,sys; d=json.load(open('gpurun_out/q_${TAG}_$c.json'))
print('%-8s step %7.1f us  min %7.1f  e2e %7.1f us  %s' % ('$c', d['ms_per_step']*1e3, d['ms_per_step_min']*1e3, d['e2e']['ms_per_step']*1e3, {k.split('_')[0]: round(v*1e3,1) for k,v in d['phases_ms'].items() if v}))"
done
