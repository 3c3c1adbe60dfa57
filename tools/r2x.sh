#!/bin/bash
# K34 latency pass: GPU tests, K34 fine timeline, benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2x_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r2x_tests.log
DINFER_EXTRA_NVCC=-DDINFER_K34_FINE python -c "from paper_2510_08666_b200 import build; build.build(force=True)"
for G in 1 8; do timeout 120 python tools/trace_k12.py --shard $G 2>&1 | grep "K34\|record added"; done
python - <<'PY'
import numpy as np
for G in (1, 8):
    d = np.load(f"gpurun_out/trace_k12_g{G}.npz"); k = d["k34"]; t0 = int(d["t0"])
    k = k[k[:, 1] > 0]
    us = lambda x: (x.astype(np.int64) - t0) / 1e3
    print("G", G)
    for i in [0, 4, 63]:
        print("  blk %2d body %.1f deps %.1f rowstats %.1f ph1 %.1f end %.1f" % (i, us(k[i, 0]), us(k[i, 1]), us(k[i, 4]), us(k[i, 2]), us(k[i, 3])))
PY
python -c "from paper_2510_08666_b200 import build; build.build(force=True)"
summ() {
python - "$1" <<'PY'
import json, sys
d = json.load(open(sys.argv[1])); r = d["roofline"]
g = d.get("graph_replay") or {}
ph = {k[:4]: round(v * 1e3, 1) for k, v in d["phases_ms"].items() if v}
print(f"{sys.argv[1][11:]:24s} step {d['ms_per_step']*1e3:7.1f} us  {r['kernel'][:4]} {r['ms_per_launch']*1e3:7.1f} us ({r['frac']:.3f}) "
      f"flushed {d['l2_flushed']['ms_per_step']*1e3:7.1f}  graph {g.get('ms_per_step', 0)*1e3:7.1f}  e2e {d['e2e']['ms_per_step']*1e3:7.1f}  {ph}")
PY
}
for rep in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2x_moe$rep.json 2>/dev/null; summ gpurun_out/r2x_moe$rep.json; done
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim 8 > gpurun_out/r2x_sim8.json 2>/dev/null; summ gpurun_out/r2x_sim8.json
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --config 8b > gpurun_out/r2x_8b.json 2>/dev/null; summ gpurun_out/r2x_8b.json
DINFER_K34_WARM=0 timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/r2x_moe_nowarm.json 2>/dev/null; summ gpurun_out/r2x_moe_nowarm.json
DINFER_K34_WARM=0 timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim 8 > gpurun_out/r2x_sim8_nowarm.json 2>/dev/null; summ gpurun_out/r2x_sim8_nowarm.json
