#!/bin/bash
# Final round-2 profiling pass (under gpurun, repo root): bench lines per
# config, the ncu launch list of the default bench command, ncu --set full of
# K12 + K34 (MoE, and one rank of an 8-way shard) and of the f3 kernels,
# gpurun_out/ (summarised into profiles/ with tools/ncu_summary.py).
TAG=${1:-r2f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_moe.json 2> gpurun_out/${TAG}_bench_moe.err; echo "bench moe rc=$?"
for c in 8b 8b-bs64 tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
for G in 2 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --shard-sim $G > gpurun_out/${TAG}_bench_moe_sim$G.json 2>/dev/null; echo "sim$G rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2>/dev/null; echo "reference rc=$?"
python tools/kv_bench.py --reps 100 > gpurun_out/${TAG}_kv.json 2>/dev/null; echo "kv rc=$?"
python tools/gen_bench.py > gpurun_out/${TAG}_gen.json 2>/dev/null; echo "gen rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "ncu launches rc=$?"
NF="ncu --set full --clock-control none --import-source on -f"
timeout 900 $NF -k regex:"k12_proj|k34_select" --launch-skip 4 -c 2 -o gpurun_out/${TAG}_full_moe python tools/step_loop.py --steps 4 > /dev/null 2>&1; echo "full moe rc=$?"
timeout 900 $NF -k regex:"k12_proj|k34_select" --launch-skip 6 -c 2 -o gpurun_out/${TAG}_full_moe_g8 python tools/trace_k12.py --shard 8 > /dev/null 2>&1; echo "full g8 rc=$?"
timeout 900 $NF -k regex:"kv_proj_tc|kv_attention_tc|kv_attention_merge" --launch-skip 30 -c 3 -o gpurun_out/${TAG}_full_kv python tools/kv_bench.py --reps 12 > /dev/null 2>&1; echo "full kv rc=$?"
ls gpurun_out | grep "^${TAG}_" | head -60
