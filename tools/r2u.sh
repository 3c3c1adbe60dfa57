#!/bin/bash
# K34 fine trace: smoothing block body start / row stats merged / partials accumulated
mkdir -p gpurun_out
DINFER_EXTRA_NVCC=-DDINFER_K34_FINE python -c "from paper_2510_08666_b200 import build; build.build(force=True)"
for G in 1 8; do timeout 120 python tools/trace_k12.py --shard $G > /dev/null 2>&1; done
python - <<'PY'
import numpy as np
for G in (1, 8):
    d = np.load(f"gpurun_out/trace_k12_g{G}.npz"); k = d["k34"]; t0 = int(d["t0"])
    k = k[k[:, 1] > 0]
    us = lambda x: (x.astype(np.int64) - t0) / 1e3
    print("G", G)
    for i in [0, 4, 5, 30, 63]:
        print("  blk %2d body %.1f deps %.1f rowstats %.1f ph1 %.1f end %.1f" % (i, us(k[i, 0]), us(k[i, 1]), us(k[i, 4]), us(k[i, 2]), us(k[i, 3])))
PY
python -c "from paper_2510_08666_b200 import build; build.build(force=True)"
