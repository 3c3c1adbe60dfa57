timeout 900 python -m pytest tests/test_gpu_kv.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/kv_bench.py 2>&1 | tail -1
DINFER_KV_TC=0 timeout 300 python tools/kv_bench.py 2>&1 | tail -1
