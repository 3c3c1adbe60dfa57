#!/bin/bash
# K12 geometry sweep: "HW STAGES PSTAGES ESTAGES" tuples x G (bench --shard-sim).
# usage: tools/pipe_sweep.sh TAG "G list" "hw,st,pst,est" ...
TAG=$1; GS=$2; shift 2
mkdir -p gpurun_out
for g in $GS; do
  for cfg in "$@"; do
    IFS=, read hw st pst est <<< "$cfg"
    if [ "$g" = 1 ]; then a=""; else a="--shard-sim $g"; fi
    f=gpurun_out/${TAG}_g${g}_${hw}_${st}_${pst}_${est}.json
    DINFER_K2_HW=$hw DINFER_K12_STAGES=$st DINFER_K12_PSTAGES=$pst DINFER_K12_ESTAGES=$est \
      timeout 300 python bench.py --no-cpu-baseline $a > $f 2>/dev/null
    python - "$g" "$cfg" "$f" <<'P'
import json,sys
g,cfg,f=sys.argv[1:]
try:
    d=json.load(open(f)); r=d['roofline']; ge=d['geometry']
    print('G=%s %-14s step %6.1f us  k12 %6.1f us frac %.3f  (stages %s smem %s)' % (g,cfg,d['ms_per_step']*1e3, r['ms_per_launch']*1e3, r['frac'], ge.get('k2_stages'), ge.get('fused_smem')))
except Exception as e: print(g,cfg,'ERR',e)
P
  done
done
