#!/bin/bash
# bench lines + the ncu launch list of the bench command (steps 1-2 of profile_round.sh)
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_moe.json 2> gpurun_out/${TAG}_bench_moe.err; echo "bench moe rc=$?"
for c in 8b 8b-bs64 tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --no-balance --no-cpu-baseline > gpurun_out/${TAG}_bench_moe_even.json 2>/dev/null; echo "even rc=$?"
DINFER_FUSED=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_moe_unfused.json 2>/dev/null; echo "unfused rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "ncu launches rc=$?"
