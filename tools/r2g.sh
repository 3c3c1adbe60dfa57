#!/bin/bash
# round-2 GPU pass: warp-issued MMAs in K12 -- parity + same-box A/B against _ab_old
mkdir -p gpurun_out
python -c "from paper_2510_08666_b200 import build; build.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -x -q > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2g_tests.log
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
      f"{ph} part {d['config']['partition'][:10]}  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for rep in 1 2; do
  ab new
  ab old DINFER_LIB=_ab_old/libdinfer.so
done
BARGS="--shard-sim 8" ab sim8_new
BARGS="--shard-sim 8" ab sim8_old DINFER_LIB=_ab_old/libdinfer.so
for G in 1 8; do timeout 120 python tools/trace_k12.py --shard $G 2>&1 | tail -11; done
