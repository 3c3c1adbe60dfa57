#!/bin/bash
# GPU parity at narrow hidden slices with batched E-phase stages, then the sweep.
mkdir -p gpurun_out
for cfg in "512 2" "256 2"; do
  set -- $cfg
  DINFER_K2_HW=$1 DINFER_K12_PSTAGES=$2 timeout 900 python -m pytest tests -m gpu -q \
    --deselect "tests/test_gpu_parity.py::test_fused_and_two_kernel_smoothing_paths" > gpurun_out/e1_pytest_hw$1.log 2>&1
  echo "pytest HW=$1 rc=$? $(tail -1 gpurun_out/e1_pytest_hw$1.log)"
  grep FAILED gpurun_out/e1_pytest_hw$1.log | head -5
done
bash tools/pipe_sweep.sh e1 "8 4 2 1" 1024,4,4,3 512,4,2,3 256,3,2,2
