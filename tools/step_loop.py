"""Run dinfer_step in a loop on the bench workload (no flush, no timing) --
a short, deterministic command to put under ncu.
  python tools/step_loop.py [--steps N] [--config moe|8b|tiny] [--no-smooth]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402

CONFIGS = {"moe": (2048, 157184), "8b": (4096, 126464), "tiny": (256, 1024)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--config", default="moe")
    ap.add_argument("--no-smooth", action="store_true")
    ap.add_argument("--B", type=int, default=1)
    ap.add_argument("--S", type=int, default=32)
    a = ap.parse_args()
    H, V = CONFIGS[a.config]
    B, S, K = a.B, a.S, 32
    smooth = not a.no_smooth
    dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
    W = synth.make_W(V, H, 1)
    h = dev(synth.planted_hidden(W, B * S, seed=0))
    Wd = dev(W)
    del W
    Ed = dev(synth.make_E(V, H, 2)) if smooth else None
    em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0]) if smooth else None
    ctx = Context(B, S, H, K, V, smooth_capable=smooth)
    dense = B * S > 256  # compute-bound K1b path: threshold decoding, no credit / smoothing
    p = make_params(decoder="threshold" if dense else "hierarchical", use_credit=not dense, use_smooth=smooth)
    mask = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    tok = torch.full((B, S), V - 1, dtype=torch.int32, device="cuda")
    cids = torch.full((B, S, K), -1, dtype=torch.int32, device="cuda")
    cval = torch.zeros((B, S, K), dtype=torch.float32, device="cuda")
    com = torch.zeros((B, S), dtype=torch.uint8, device="cuda")
    sm = torch.zeros((B, S, H), dtype=torch.float32, device="cuda") if smooth else None
    st = torch.zeros((B, S, 4), dtype=torch.float32, device="cuda")
    for _ in range(a.steps):
        mask.fill_(1)
        cids.fill_(-1)
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    ctx.sync()
    torch.cuda.synchronize()
    print("ok", ctx.geometry())


if __name__ == "__main__":
    main()
