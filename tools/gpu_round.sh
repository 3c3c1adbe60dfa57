#!/bin/bash
# One GPU validation + measurement pass (run under gpurun from the repo root).
#   tools/gpu_round.sh TAG [bench-env-variants...]
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/tests_$TAG.log 2>&1
echo "tests_rc=$?"; tail -3 gpurun_out/tests_$TAG.log
summ() {
python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
ph = {k.split('_')[0]: round(v * 1000, 1) for k, v in d["phases_ms"].items() if v}
sr = d.get("step_roofline") or {}
r = d["roofline"]
print(f"  [{d['config'].get('name')}] step {d['ms_per_step']*1000:.1f} us  {d['value']:.0f} pos/s  step-roofline {sr.get('frac', 0):.3f}"
      f"  {r['kernel']} {r['achieved']:.0f} {r['unit']} ({r['frac']:.3f})  kernels(us) {ph}  e2e {d['e2e']['ms_per_step']*1000:.1f} us"
      f"  clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
}
for v in "default" "$@"; do
  if [ "$v" = "default" ]; then envs=""; else envs="$v"; fi
  env $envs timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_${TAG}_${v//[= ]/_}.json 2> gpurun_out/bench_${TAG}.err
  echo "bench [$v] rc=$?"; summ gpurun_out/bench_${TAG}_${v//[= ]/_}.json
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python tools/step_loop.py --steps 6 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_$TAG.csv
