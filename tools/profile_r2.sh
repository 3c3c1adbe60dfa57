#!/bin/bash
# Round-2 profiling pass (under gpurun, repo root): bench lines per config, the
# ncu launch list of the bench command, ncu --set full captures per kernel,
# compute-sanitizer runs.  Outputs in gpurun_out/ (summarised into profiles/).
TAG=r2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_moe.json 2> gpurun_out/${TAG}_bench_moe.err; echo "bench moe rc=$?"
for c in 8b 8b-bs64 tiny; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 600 python bench.py --no-balance --no-cpu-baseline > gpurun_out/${TAG}_bench_moe_even.json 2>/dev/null; echo "even rc=$?"
DINFER_FUSED=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench_moe_unfused.json 2>/dev/null; echo "unfused rc=$?"
for G in 2 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --shard-sim $G > gpurun_out/${TAG}_bench_moe_sim$G.json 2>/dev/null; echo "sim$G rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2>/dev/null; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_bench.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.out 2>&1; echo "ncu launches rc=$?"
NF="ncu --set full --clock-control none --import-source on -f"
timeout 900 $NF -k regex:"k12_proj|k34_select" --launch-skip 4 -c 2 -o gpurun_out/${TAG}_full_moe python tools/step_loop.py --steps 4 > /dev/null 2>&1; echo "full moe rc=$?"
DINFER_FUSED=0 timeout 900 $NF -k regex:"k1_vocab|k2_smooth" --launch-skip 6 -c 2 -o gpurun_out/${TAG}_full_moe_unfused python tools/step_loop.py --steps 4 > /dev/null 2>&1; echo "full unfused rc=$?"
timeout 900 $NF -k regex:"k1_vocab|k34_select" --launch-skip 4 -c 2 -o gpurun_out/${TAG}_full_8b python tools/step_loop.py --config 8b --no-smooth --steps 4 > /dev/null 2>&1; echo "full 8b rc=$?"
timeout 900 $NF -k regex:"k1b_vocab" --launch-skip 1 -c 1 -o gpurun_out/${TAG}_full_8b_bs64 python tools/step_loop.py --config 8b --no-smooth --B 64 --S 64 --steps 3 > /dev/null 2>&1; echo "full bs64 rc=$?"
timeout 900 $NF -k regex:"k12_proj|k34_select" --launch-skip 6 -c 2 -o gpurun_out/${TAG}_full_moe_g8 python tools/trace_k12.py --shard 8 > /dev/null 2>&1; echo "full g8 rc=$?"
DINFER_FUSED=2 timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python tools/step_loop.py --config tiny --steps 3 > gpurun_out/${TAG}_san_racecheck_k12.log 2>&1; echo "racecheck rc=$?"
DINFER_FUSED=2 timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/step_loop.py --config tiny --steps 3 > gpurun_out/${TAG}_san_synccheck_k12.log 2>&1; echo "synccheck rc=$?"
DINFER_FUSED=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "split or block_start or shard or determinism" > gpurun_out/${TAG}_san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"
./tools/hbm_read_ceiling 1288 > gpurun_out/${TAG}_read_ceiling.txt 2>&1; ./tools/red_bench > gpurun_out/${TAG}_red_bench.txt 2>&1
ls gpurun_out | grep "^${TAG}_" | head -60
