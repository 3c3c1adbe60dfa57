#!/bin/bash
# round-2 GPU pass: warp-issued MMAs everywhere + single-accumulator stacked E MMAs
mkdir -p gpurun_out
python -c "from paper_2510_08666_b200 import build; build.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2h_tests.log
ab() {  # name envs...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 $BARGS > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{n}.json")); r = d["roofline"]
g = d.get("graph_replay") or {}
ph = {k[:4]: round(v * 1e3, 1) for k, v in d["phases_ms"].items() if v}
print(f"{n:14s} step {d['ms_per_step']*1e3:7.1f} us  {r['kernel'][:4]} {r['ms_per_launch']*1e3:7.1f} us ({r['frac']:.3f})  "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f}  graph {g.get('ms_per_step', 0)*1e3:7.1f}  e2e {d['e2e']['ms_per_step']*1e3:7.1f}  "
      f"{ph} part {d['config']['partition'][:10]}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for rep in 1 2; do
  ab stack1
  ab stack0 DINFER_K12_STACK=0
  ab old DINFER_LIB=_ab_old/libdinfer.so
done
BARGS="--config 8b" ab 8b_new
BARGS="--config 8b" ab 8b_old DINFER_LIB=_ab_old/libdinfer.so
BARGS="--shard-sim 8" ab sim8_new
timeout 120 python tools/trace_k12.py --shard 1 2>&1 | tail -11
timeout 120 python tools/kv_bench.py
