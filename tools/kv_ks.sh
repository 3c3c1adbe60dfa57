#!/bin/bash
# same-box A/B of the projection's cluster split of K (DINFER_KV_KS), 3 alternating rounds
for r in 1 2 3; do
  for ks in "$@"; do
    echo "r$r ks=$ks $(DINFER_KV_KS=$ks python tools/kv_bench.py --reps 100 | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['vicinity']['us'],1), round(d['full_refresh']['us'],1))")"
  done
done
