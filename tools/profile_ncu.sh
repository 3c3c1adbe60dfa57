#!/bin/bash
# ncu --set full captures of the step kernels (step 3 of profile_round.sh)
TAG=${1:-r1}
mkdir -p gpurun_out
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
