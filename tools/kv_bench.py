"""Time the vicinity KV-cache refresh forward (dinfer_kv_step) on a
synthetic attention layer at the LLaDA-MoE attention shape: H = 2048 (16
heads x 128), L = 64 + 1024.  Steady-state vicinity forward (region = block
32 + looks 16 + 16 = 64 positions) vs a full refresh (all L positions), CUDA
events, L2 flushed before each timed forward.
  python tools/kv_bench.py [--L 1088] [--H 2048] [--reps 50]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08666_b200 import VicinityKV  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=1088)
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    L, H = a.L, a.H
    g = torch.Generator(device="cuda").manual_seed(0)
    W = [(torch.randn((H, H), device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16) for _ in range(3)]
    X = torch.randn((L, H), device="cuda", generator=g).to(torch.bfloat16)
    Kc = torch.zeros((L, H), dtype=torch.bfloat16, device="cuda")
    Vc = torch.zeros_like(Kc)
    out = torch.zeros((L, H), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    kv = VicinityKV(L, H, 128, 16, 16, 4, stream=st.cuda_stream)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    start, end = 64 + 512, 64 + 544
    res = {}
    for name, t, full in (("vicinity", 9, False), ("full_refresh", 0, True)):
        ms = []
        for i in range(a.reps + 5):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lo, hi = kv.step(X, *W, Kc, Vc, start, end, t, out, full=full)
            e1.record(st)
            e1.synchronize()
            if i >= 5:
                ms.append(e0.elapsed_time(e1))
        R = hi - lo
        us = sum(ms) / len(ms) * 1e3
        bytes_ = 3 * H * H * 2 + 2 * L * H * 2 + R * H * (2 * 2 + 2 + 4)  # weights + caches + X, K/V, Q, out
        flops = 2 * R * H * 3 * H + 4 * R * L * H
        res[name] = {"region": [lo, hi], "us": us, "algorithmic_MB": bytes_ / 1e6, "GB/s": bytes_ / us / 1e3,
                     "TFLOP/s": flops / us / 1e6}
    kv.close()
    print(json.dumps({"L": L, "H": H, "heads": H // 128, **res}))


if __name__ == "__main__":
    main()
