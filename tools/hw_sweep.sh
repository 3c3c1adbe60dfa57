#!/bin/bash
# K12 hidden-slice width sweep at shard sizes: GPU tests at narrow slices, then
# bench --shard-sim G for every DINFER_K2_HW (multi-chunk 64-KB E stages).
# usage: tools/hw_sweep.sh TAG "HW list" "G list" [test HW list]
TAG=$1; HWS=${2:-"1024 512 256 128"}; GS=${3:-"1 2 4 8"}; THW=${4:-"256 128"}
mkdir -p gpurun_out
for hw in $THW; do
  DINFER_K2_HW=$hw timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_hw$hw.log 2>&1
  echo "pytest HW=$hw rc=$? $(tail -1 gpurun_out/${TAG}_pytest_hw$hw.log)"
done
for g in $GS; do
  for hw in $HWS; do
    if [ "$g" = 1 ]; then a=""; else a="--shard-sim $g"; fi
    DINFER_K2_HW=$hw timeout 300 python bench.py --no-cpu-baseline $a > gpurun_out/${TAG}_g${g}_hw$hw.json 2>/dev/null
    python - "$g" "$hw" "gpurun_out/${TAG}_g${g}_hw$hw.json" <<'P'
import json,sys
g,hw,f=sys.argv[1:]
try:
    d=json.load(open(f)); r=d['roofline']
    print('G=%s HW=%5s step %6.1f us  k12 %6.1f us frac %.3f  k34 %5.1f  flushed %6.1f' % (g,hw,d['ms_per_step']*1e3, r['ms_per_launch']*1e3, r['frac'], d['phases_ms']['k34_select_smooth']*1e3, d['l2_flushed']['ms_per_step']*1e3))
except Exception as e: print(g,hw,'ERR',e)
P
  done
done
