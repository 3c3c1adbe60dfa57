timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "step_host or graph" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_generate.py tests/test_bench_contract.py -q -x -m gpu 2>&1 | tail -2
bash tools/ab.sh DINFER_STAGE_KERNELS 1 0 3
