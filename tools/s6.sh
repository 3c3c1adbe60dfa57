timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.1f us flushed %.1f e2e %.1f  %s %.1f us frac %.3f k34 %.2f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, r['kernel'], r['ms_per_launch']*1e3, r['frac'], d['phases_ms']['k34_select_smooth']*1e3))"; done
REPS=4 python tools/trace_chain.py balance 2>&1 | grep -E "K34|K12 exit|period" | tail -9
