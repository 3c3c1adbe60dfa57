#!/bin/bash
# round-2 GPU pass: rank-finalize fold parity + K12 stream experiments
mkdir -p gpurun_out
python -c "from paper_2510_08666_b200 import build; build.build()"
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py -x -q > gpurun_out/r2c_tests_default.log 2>&1
echo "default tests rc=$?"; tail -2 gpurun_out/r2c_tests_default.log
DINFER_FUSED=2 DINFER_RANKFIN_G1=1 timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or sharded or ragged or block_start or host or combine" > gpurun_out/r2c_tests_fold.log 2>&1
echo "fold tests rc=$?"; tail -2 gpurun_out/r2c_tests_fold.log
DINFER_RANKFIN_G1=1 timeout 400 python -m pytest tests/test_gpu_timed_path.py -x -q > gpurun_out/r2c_tests_fold_moe.log 2>&1
echo "fold moe tests rc=$?"; tail -2 gpurun_out/r2c_tests_fold_moe.log
for x in 0 16 32 48; do
  echo "=== trace X=$x"; DINFER_K12_X=$x timeout 120 python tools/trace_step.py 2>&1 | grep -E "K12 per-CTA|step span|last tile|exit"
done
./tools/k12_x_sweep.sh 0 16 32 48 0
echo "=== rankfin G1 A/B"
for v in 0 1 0 1; do
  DINFER_RANKFIN_G1=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 > gpurun_out/rf_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/rf_$v.json'));r=d['roofline']
print('RANKFIN_G1=$v step %.1f us  K12 %.1f us frac %.3f  flushed %.1f  e2e %.1f phases %s' % (d['ms_per_step']*1e3, r['ms_per_launch']*1e3, r['frac'], d['l2_flushed']['ms_per_step']*1e3, d['e2e']['ms_per_step']*1e3, {k: round(v*1e3,1) for k,v in d['phases_ms'].items() if v}))"
done
