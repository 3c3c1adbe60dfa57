# A/B of an env knob on the bench headline: tools/ab.sh VAR VALUE_A VALUE_B [pairs] [bench args]
var=$1; a=$2; b=$3; n=${4:-3}; shift 4
for i in $(seq $n); do
  for v in $a $b; do
    env $var=$v python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v: %.1f us  flushed %.1f  e2e %.1f  k12/k1 %.1f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['roofline']['ms_per_launch']*1e3))"
  done
done
