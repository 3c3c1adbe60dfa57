set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g1_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/g1_moe.json 2> gpurun_out/g1_moe.err; echo rc=$?
for g in 2 4 8; do timeout 300 python bench.py --no-cpu-baseline --shard-sim $g > gpurun_out/g1_sim$g.json 2>/dev/null; done
python - <<'P'
import json
for f in ['g1_moe','g1_sim2','g1_sim4','g1_sim8']:
    try:
        d=json.load(open('gpurun_out/%s.json'%f)); print(f, round(d['ms_per_step']*1e3,1), d['roofline']['frac'], d['phases_ms'])
    except Exception as e: print(f, e)
P
