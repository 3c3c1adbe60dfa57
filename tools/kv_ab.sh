#!/bin/bash
# same-box A/B of kv_proj_tc ring geometries: "cps,stages" ... (3 alternating rounds)
for r in 1 2 3; do
  for cfg in "$@"; do
    IFS=, read cps st <<< "$cfg"
    echo "r$r cps=$cps st=$st $(DINFER_KV_PJ_CPS=$cps DINFER_KV_PJ_STAGES=$st python tools/kv_bench.py --reps 100 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['vicinity']['us'],1), round(d['full_refresh']['us'],1))")"
  done
done
