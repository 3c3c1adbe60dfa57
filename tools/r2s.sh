#!/bin/bash
# K34: one selection CTA per row, prefetched phase 1, one-round-trip partial loads
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2s_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2s_tests.log
for G in 1 8; do timeout 120 python tools/trace_k12.py --shard $G 2>&1 | tail -16; done
summ() {
python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); r = d["roofline"]
g = d.get("graph_replay") or {}
ph = {k[:4]: round(v * 1e3, 1) for k, v in d["phases_ms"].items() if v}
sr = d.get("step_roofline") or {}
print(f"{sys.argv[1][11:]:24s} step {d['ms_per_step']*1e3:7.1f} us  {r['kernel'][:4]} {r['ms_per_launch']*1e3:7.1f} us ({r['frac']:.3f}) step-frac {sr.get('frac', 0):.3f} "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f}  graph {g.get('ms_per_step', 0)*1e3:7.1f}  e2e {d['e2e']['ms_per_step']*1e3:7.1f}  "
      f"{ph} clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for rep in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2s_moe$rep.json 2>gpurun_out/r2s_moe.err; summ gpurun_out/r2s_moe$rep.json
done
for G in 2 4 8; do
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim $G > gpurun_out/r2s_sim$G.json 2>gpurun_out/r2s_sim$G.err
  summ gpurun_out/r2s_sim$G.json
done
DINFER_K12_RECORD=1 timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2s_moe_rec.json 2>gpurun_out/r2s_moe_rec.err; summ gpurun_out/r2s_moe_rec.json
