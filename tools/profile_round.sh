#!/bin/bash
# Profiling pass for profiles/ (run under gpurun from the repo root).
#   tools/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
# 1-2) bench lines for every config (+ even / two-kernel variants) and the ncu launch list
bash tools/profile_bench.sh ${TAG}
# 3) one --set full capture per kernel (steady-state launches of the step loop)
bash tools/profile_ncu.sh ${TAG}
ls -la gpurun_out | tail -20
