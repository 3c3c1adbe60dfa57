#!/bin/bash
# shard-step diagnosis: per-CTA K12 timelines at G = 1, 2, 8; racecheck after the ref fix
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1; echo "build rc=$?"
for G in 1 2 8; do timeout 120 python tools/trace_k12.py --shard $G 2>&1 | tail -12; done
for G in 8; do
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 --shard-sim $G --no-balance > gpurun_out/r2j_sim${G}_even.json 2>gpurun_out/r2j_sim$G.err
  python -c "import json; d=json.load(open('gpurun_out/r2j_sim${G}_even.json')); print('sim$G even', d['ms_per_step']*1e3, d['roofline']['ms_per_launch']*1e3, d['phases_ms'])"
done
DINFER_FUSED=2 timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/step_loop.py --config tiny --steps 3 \
    > gpurun_out/r2j_san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/r2j_san_racecheck.log
