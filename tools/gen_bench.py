"""Time the device-resident generation loop (dinfer_generate) at a BASELINE
shape: one CUDA-graph launch runs every forward of a generation; per-forward
time = graph time / F, compared with the same number of dinfer_step calls
launched from the host.  Hidden states are planted (synth), not vetted --
this measures time, not parity.
  python tools/gen_bench.py [--config moe|8b] [--blocks 8] [--reps 5]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08666_b200 import Context, make_gen_config, make_params, synth  # noqa: E402

CONFIGS = {"moe": (2048, 157184, "hierarchical", True, True), "8b": (4096, 126464, "threshold", False, False)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="moe")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    H, V, dec, credit, smooth = CONFIGS[a.config]
    B, S, K, P = 1, 32, 32, 16
    M = B * S
    dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
    W = synth.make_W(V, H, 1)
    # planted hidden per iteration: every block's positions ramp up over ~6 iterations
    iters = a.blocks * S
    sch = synth.PlantedSchedule(M, V, H, 0)
    hs = []
    for n in range(iters):
        tgt, amp = sch.targets_and_amplitudes(n % 8)
        hs.append(sch.hidden(W[tgt], amp))
    hsrc = dev(np.stack(hs))
    Wd = dev(W)
    del W
    Ed = dev(synth.make_E(V, H, 2)) if smooth else None
    em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0]) if smooth else None
    ctx = Context(B, S, H, K, V, smooth_capable=smooth)
    base = make_params(decoder=dec, use_credit=credit, use_smooth=smooth, theta_lo=0.62)
    L = P + a.blocks * S
    cfg = make_gen_config(L, P, synth.mask_id(V), synth.eos_id(V), early_termination=True, tau_target=0.9,
                          tau_decay_steps=2)
    X0 = torch.full((B, L), synth.mask_id(V), dtype=torch.int32)
    X0[:, :P] = 5
    X = X0.cuda()
    out = torch.zeros(B + 2, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    times = []
    for r in range(a.reps + 1):
        X.copy_(X0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ctx.generate(cfg, base, Wd, Ed, em, hsrc, X, out)
        e1.record(st)
        e1.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
    o = out.cpu().numpy()
    F = int(o[B])
    # the same F steps launched from the host (no loop bookkeeping, no hidden copy)
    mask = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    tok = torch.full((B, S), synth.mask_id(V), dtype=torch.int32, device="cuda")
    cids = torch.full((B, S, K), -1, dtype=torch.int32, device="cuda")
    cval = torch.zeros((B, S, K), device="cuda")
    com = torch.zeros((B, S), dtype=torch.uint8, device="cuda")
    sm = torch.zeros((B, S, H), device="cuda") if smooth else None
    p = make_params(decoder=dec, use_credit=credit, use_smooth=smooth)
    host = []
    for r in range(a.reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for n in range(F):
            ctx.step(hsrc[n], Wd, Ed, em, mask, tok, cids, cval, p, com, sm, None)
        e1.record(st)
        e1.synchronize()
        if r:
            host.append(e0.elapsed_time(e1))
    g, h_ = float(np.median(times)), float(np.median(host))
    print(json.dumps({"config": a.config, "blocks": a.blocks, "F": F, "T": int(o[0]), "tpf": o[0] / max(F, 1),
                      "loop_ms": g, "loop_us_per_forward": 1e3 * g / F,
                      "host_steps_ms": h_, "host_us_per_step": 1e3 * h_ / F}))


if __name__ == "__main__":
    main()
