#!/bin/bash
# bench lines for every BASELINE config + shard-sim 2/4/8 into gpurun_out/TAG_bench_*.json
TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_moe.json 2> gpurun_out/${TAG}_bench_moe.err; echo "bench moe rc=$?"
for c in 8b 8b-bs64 tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
done
for G in 2 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --shard-sim $G > gpurun_out/${TAG}_bench_moe_sim$G.json 2>/dev/null; echo "sim$G rc=$?"
done
