#!/bin/bash
# K34 smoothing-block cap sweep (DINFER_K34_BLOCKS): parity tests at a small
# cap, then the bench headline at G = 1 and one rank of an 8-way shard.
# usage: tools/k34_sweep.sh TAG "caps" "G list" [extra bench args]
TAG=$1; CAPS=${2:-"0 64 32 16"}; GS=${3:-"1 8"}; EXTRA=$4
mkdir -p gpurun_out
DINFER_K34_BLOCKS=16 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest K34_BLOCKS=16 rc=$? $(tail -1 gpurun_out/${TAG}_pytest.log)"
for g in $GS; do
  for cap in $CAPS; do
    if [ "$g" = 1 ]; then a=""; else a="--shard-sim $g"; fi
    DINFER_K34_BLOCKS=$cap timeout 300 python bench.py --no-cpu-baseline $a $EXTRA > gpurun_out/${TAG}_g${g}_c$cap.json 2>/dev/null
    python - "$g" "$cap" "gpurun_out/${TAG}_g${g}_c$cap.json" <<'P'
import json,sys
g,cap,f=sys.argv[1:]
try:
    d=json.load(open(f)); r=d['roofline']
    print('G=%s cap=%3s step %6.1f us  k12 %6.1f us frac %.3f  k34 %5.1f  flushed %6.1f e2e %6.1f' % (g,cap,d['ms_per_step']*1e3, r['ms_per_launch']*1e3, r['frac'], d['phases_ms']['k34_select_smooth']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3))
except Exception as e: print(g,cap,'ERR',e)
P
  done
done
