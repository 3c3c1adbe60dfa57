set -e
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for i in 1 2; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.1f us flushed %.1f e2e %.1f k12 %.1f frac %.3f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, d['roofline']['ms_per_launch']*1e3, d['roofline']['frac']), d['clocks'])"; done
DINFER_K34_FLAGS=0 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('noflags %.1f us flushed %.1f e2e %.1f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3))"
python tools/trace_chain.py balance 2>&1 | tail -28
