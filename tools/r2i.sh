#!/bin/bash
# round-2 re-entry GPU pass: HEAD state -- all GPU tests, smoke, default bench line,
# per-rank shard steps (--shard-sim 2/4/8), 8B line, KV + generate loop, sanitizers.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"; cat gpurun_out/r2i_bench.json
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
summ gpurun_out/r2i_bench.json
for G in 2 4 8; do
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim $G > gpurun_out/r2i_sim$G.json 2>gpurun_out/r2i_sim$G.err
  summ gpurun_out/r2i_sim$G.json
done
timeout 300 python bench.py --no-cpu-baseline --config 8b > gpurun_out/r2i_8b.json 2>gpurun_out/r2i_8b.err; summ gpurun_out/r2i_8b.json
timeout 300 python bench.py --no-cpu-baseline --config 8b-bs64 --steps 10 > gpurun_out/r2i_8bbs64.json 2>gpurun_out/r2i_8bbs64.err; summ gpurun_out/r2i_8bbs64.json
timeout 120 python tools/kv_bench.py 2>&1 | tail -6
timeout 300 python tools/gen_bench.py 2>&1 | tail -6
for tool in memcheck racecheck synccheck; do
  DINFER_FUSED=2 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/step_loop.py --config tiny --steps 3 \
    > gpurun_out/r2i_san_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; tail -3 gpurun_out/r2i_san_$tool.log
done
