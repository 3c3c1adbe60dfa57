bash tools/ab.sh DINFER_BALANCE_MODE dirty chain 3
DINFER_BALANCE_MODE=chain DINFER_BALANCE_DAMP=0.6 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chain damp0.6: %.1f flushed %.1f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3))"
DINFER_BALANCE_MODE=chain DINFER_BALANCE_DAMP=0.5 DINFER_BALANCE_ROUNDS=2 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chain damp0.5 r2: %.1f flushed %.1f' % (d['ms_per_step']*1e3, d['l2_flushed']['ms_per_step']*1e3))"
DINFER_BALANCE_MODE=chain REPS=6 python tools/trace_chain.py balance 2>&1 | tail -3
