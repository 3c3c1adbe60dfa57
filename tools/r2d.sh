#!/bin/bash
# round-2 GPU pass: stacked hi/lo E MMAs (HW 512) parity + A/B
mkdir -p gpurun_out
python -c "from paper_2510_08666_b200 import build; build.build()"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_tests.log 2>&1
echo "gpu tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
ab() {  # name envs...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{n}.json")); r = d["roofline"]
g = d.get("graph_replay") or {}
print(f"{n:14s} step {d['ms_per_step']*1e3:7.1f} us  K12 {r['ms_per_launch']*1e3:7.1f} us ({r['frac']:.3f})  "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f}  graph {g.get('ms_per_step', 0)*1e3:7.1f}  e2e {d['e2e']['ms_per_step']*1e3:7.1f}  "
      f"hw {d['geometry']['k2_hw']} part {d['config']['partition'][:10]}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for rep in 1 2; do
  ab stack1 DINFER_K12_STACK=1
  ab stack0 DINFER_K12_STACK=0
  ab stack0_hw512 DINFER_K12_STACK=0 DINFER_K2_HW=512
  ab stack1_rf DINFER_K12_STACK=1 DINFER_RANKFIN_G1=1
done
for G in 2 4 8; do
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim $G > gpurun_out/sim_$G.json 2>gpurun_out/sim_$G.err
  python - "$G" <<'PY'
import json, sys
G = sys.argv[1]
d = json.load(open(f"gpurun_out/sim_{G}.json")); r = d["roofline"]
g = d.get("graph_replay") or {}
print(f"shard-sim {G}: step {d['ms_per_step']*1e3:6.1f} us  K12 {r['ms_per_launch']*1e3:6.1f} us ({r['frac']:.3f})  step-frac {d['step_roofline']['frac']:.3f}  "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:6.1f}  graph {g.get('ms_per_step', 0)*1e3:6.1f}  phases {{k: round(v*1e3,1) for k,v in d['phases_ms'].items() if v}}  {d['config']['l2'][:60]}")
PY
done
