#!/bin/bash
# round-2 GPU pass: E-ring depth, shard-size traces, tcgen05 projections of the vicinity layer
mkdir -p gpurun_out
python -c "from paper_2510_08666_b200 import build; build.build()"
timeout 300 python -m pytest tests/test_gpu_kv.py -x -q > gpurun_out/r2e_kv.log 2>&1; echo "kv tests rc=$?"; tail -2 gpurun_out/r2e_kv.log
timeout 120 python tools/kv_bench.py > gpurun_out/r2e_kvbench.json 2>&1; cat gpurun_out/r2e_kvbench.json
for G in 1 8; do timeout 120 python tools/trace_k12.py --shard $G 2>&1 | tail -12; done
ab() {  # name envs...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 $BARGS > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
d = json.load(open(f"gpurun_out/ab_{n}.json")); r = d["roofline"]
g = d.get("graph_replay") or {}
ph = {k[:4]: round(v * 1e3, 1) for k, v in d["phases_ms"].items() if v}
print(f"{n:14s} step {d['ms_per_step']*1e3:7.1f} us  K12 {r['ms_per_launch']*1e3:7.1f} us ({r['frac']:.3f})  "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f}  graph {g.get('ms_per_step', 0)*1e3:7.1f}  e2e {d['e2e']['ms_per_step']*1e3:7.1f}  "
      f"{ph} hw {d['geometry']['k2_hw']} part {d['config']['partition'][:10]}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for rep in 1 2; do
  ab est3 DINFER_K12_ESTAGES=3
  ab est2 DINFER_K12_ESTAGES=2
done
for G in 2 4 8; do
  BARGS="--shard-sim $G" ab sim${G}_est3 DINFER_K12_ESTAGES=3
  BARGS="--shard-sim $G" ab sim${G}_est2 DINFER_K12_ESTAGES=2
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2e_tests.log
