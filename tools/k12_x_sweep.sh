#!/bin/bash
# Same-box sweep of K12 measurement-only experiments (DINFER_K12_X bits,
# kernels.h K1Args::xbits) on the bench headline: which part of K12 costs
# stream rate.  Results are not parity-valid for bits 1/2 (hidden / flog skipped).
#   tools/k12_x_sweep.sh [bits...]
mkdir -p gpurun_out
for x in ${@:-0 1 2 3 4 8 12 0}; do
  DINFER_K12_X=$x timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/kx_$x.json 2>/dev/null
  python - "$x" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/kx_{sys.argv[1]}.json"))
r = d["roofline"]
print(f"X={sys.argv[1]:>3}  step {d['ms_per_step']*1e3:7.1f} us  K12 {r['ms_per_launch']*1e3:7.1f} us  "
      f"{r['achieved']:6.0f} GB/s ({r['frac']:.3f})  flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f} us  "
      f"clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
done
