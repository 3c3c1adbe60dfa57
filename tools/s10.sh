timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "calibrated or balanced" 2>&1 | tail -2
for i in 1 2; do
for nb in "" "--no-balance"; do python bench.py --config 8b --no-cpu-baseline $nb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('8b $nb %.1f us flushed %.1f e2e %.1f %s %.1f us frac %.3f %s' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, r['kernel'], r['ms_per_launch']*1e3, r['frac'], d['config']['partition']))"; done
done
DINFER_BALANCE_VERBOSE=1 DINFER_BALANCE_ROUNDS=3 python bench.py --config 8b --no-cpu-baseline 2>&1 | grep -E "dinfer_balance|ms_per" | cut -c1-200 | head -5
DINFER_BALANCE_ROUNDS=3 python bench.py --config 8b --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b rounds3 %.1f us' % (d['ms_per_step']*1e3))"
DINFER_BALANCE_DAMP=1.0 python bench.py --config 8b --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b damp1 %.1f us' % (d['ms_per_step']*1e3))"
