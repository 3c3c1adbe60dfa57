set -e
python -m pytest tests/test_gpu_parity.py -q -x -k "block_reset or determinism or fused_and_two" 2>&1 | tail -3
for i in 1 2; do python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['l2_flushed']['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"; done
python bench.py --config 8b --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['l2_flushed']['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'])"
