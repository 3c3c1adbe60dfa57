"""bench.py's JSON-line contract: the reference arm (the CPU oracle) here, the
GPU arm on a B200 (tiny configuration, so it runs in seconds)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "3")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"]


@pytest.mark.gpu
def test_gpu_arm_line_tiny():
    d = run_bench("--config", "tiny", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "l2_flushed"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 2 * 5  # K1 + K34 per step
    assert d["roofline"]["bound"] in ("hbm", "tensor") and d["roofline"]["frac"] > 0
    assert "no flush" in d["config"]["l2"]


@pytest.mark.gpu
@pytest.mark.parametrize("config,exchange", [("tiny", "p2p"), ("moe", "p2p")])
def test_gpu_arm_two_ranks_one_device(config, exchange):
    """The N = 2 code path of bench.py end to end on one GPU (both ranks on
    cuda:0, gloo process group; BENCH_SAME_DEVICE=1): vocab-sharded contexts,
    the peer-memory record exchange (CUDA IPC; NCCL refuses two ranks on one
    device, so its allgather is covered by the split-phase tests), the
    back-to-back timed loop.  Time-sliced on one device, so only the contract
    is checked, not the timing."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config,
           "--steps", "3", "--warmup", "3", "--exchange", exchange, "--no-balance"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["vocab_shards"] == 2 and d["config"]["exchange"] == exchange
    assert d["value"] > 0 and d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_gpu_arm_shard_sim():
    """--shard-sim 8: one rank of the 8-way LLaDA-MoE vocab shard on one GPU
    (loopback record exchange), rotating weight copies so each step reads
    bytes the L2 does not hold."""
    d = run_bench("--config", "moe", "--shard-sim", "8", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    c = d["config"]
    assert c["vocab_shards"] == 8 and c["V_local"] == 157184 // 8 and c["exchange"] == "loopback"
    assert "3 weight copies" in c["l2"]
    assert d["value"] > 0 and d["roofline"]["frac"] > 0
    assert d["graph_replay"]["ms_per_step"] > 0


def test_reference_config_keys_match_gpu_arm():
    """Both arms build `config` with the same function (bench.bench_config), so
    the driver sees the same keys; the reference arm adds only `oracle`."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.set_config("moe")
    g = b.bench_config(1, 157184, "none", b.default_partition(False), 1)
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert set(d["config"]) - {"oracle"} == set(g)
    assert {k: d["config"][k] for k in g} == g
