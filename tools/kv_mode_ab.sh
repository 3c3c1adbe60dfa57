#!/bin/bash
# same-box A/B of the projection's K split: cluster (DSMEM) vs global partials with ring depth st
for r in 1 2 3; do
  for cfg in "$@"; do
    IFS=, read cl st <<< "$cfg"
    echo "r$r cluster=$cl st=$st $(DINFER_KV_CLUSTER=$cl DINFER_KV_PJ_STAGES=$st python tools/kv_bench.py --reps 100 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['vicinity']['us'],1), round(d['full_refresh']['us'],1))")"
  done
done
