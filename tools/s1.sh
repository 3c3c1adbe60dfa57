timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused or moe or embedding or credit_fused or ragged" 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/s7_bench.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s7_bench.json')); print('step %.1f us min %.1f e2e %.1f' % (d['ms_per_step']*1e3, d['ms_per_step_min']*1e3, d['e2e']['ms_per_step']*1e3), {k: round(v*1e3,1) for k,v in d['phases_ms'].items() if v}, d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'])"; done
