timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "step_host" 2>&1 | tail -3
python tools/e2e_probe.py
DINFER_HOST_GRAPH=0 python tools/e2e_probe.py | grep step_host
