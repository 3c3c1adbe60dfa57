#!/bin/bash
# Profiling pass for profiles/ (run under gpurun from the repo root).
#   tools/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
# 1) bench lines (default = headline, with cpu_baseline)
timeout 900 python bench.py > gpurun_out/${TAG}_bench_moe.json 2> gpurun_out/${TAG}_bench_moe.err; echo "bench moe rc=$?"
for c in 8b 8b-bs64 tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
# 2) ncu launch list of the bench command itself (per-launch durations, cold, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "ncu launches rc=$?"
# 3) one --set full capture per kernel (steady-state launches of the step loop)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k12_proj|k34_select" \
  --launch-skip 4 -c 2 -f -o gpurun_out/${TAG}_full_moe python tools/step_loop.py --steps 4 > gpurun_out/${TAG}_full_moe.out 2>&1
echo "ncu full moe rc=$?"
DINFER_FUSED=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_vocab|k2_smooth" \
  --launch-skip 6 -c 2 -f -o gpurun_out/${TAG}_full_moe_unfused python tools/step_loop.py --steps 4 \
  > gpurun_out/${TAG}_full_moe_unfused.out 2>&1
echo "ncu full moe unfused rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_vocab|k34_select" \
  --launch-skip 4 -c 2 -f -o gpurun_out/${TAG}_full_8b python tools/step_loop.py --config 8b --no-smooth --steps 4 \
  > gpurun_out/${TAG}_full_8b.out 2>&1
echo "ncu full 8b rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1b_vocab" \
  --launch-skip 1 -c 1 -f -o gpurun_out/${TAG}_full_8b_bs64 python tools/step_loop.py --config 8b --no-smooth --B 64 --S 64 --steps 3 \
  > gpurun_out/${TAG}_full_8b_bs64.out 2>&1
echo "ncu full 8b-bs64 rc=$?"
ls -la gpurun_out | tail -20
