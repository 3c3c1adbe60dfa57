"""Time the device-resident generation loop (dinfer_generate) at a BASELINE
shape: one CUDA-graph launch runs every forward of a generation; per-forward
time = graph time / F, compared with the same number of dinfer_step calls
launched from the host (no control flow: a lower bound), and with a
host-driven Alg. 1 loop (per forward a device->host mask read decides the
block's end, schedules computed on the host).  Hidden states are planted (synth), not vetted --
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
from paper_2510_08666_b200.dinfer import alpha_schedule, tau_schedule  # noqa: E402

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
    # A host-driven Alg. 1 loop (what the device loop replaces): per
    # forward the model stand-in's hidden copy, the step with the host-computed
    # schedules (tau_t, alpha_t), then a device->host read of the mask to decide
    # whether the block is done (host control flow needs it); at block end the
    # block is written into X, EOS checked on the host, the next block reset.
    hbuf = torch.empty_like(hsrc[0])
    Xh = torch.empty_like(X)
    alg1 = []
    F_host = 0
    for r in range(a.reps + 1):
        Xh.copy_(X0.cuda())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        n = 0
        for blk in range(a.blocks):
            ctx.block_reset(mask, tok, cids, cval, synth.mask_id(V))
            t = 0
            while True:
                hbuf.copy_(hsrc[n % iters])
                pt = make_params(decoder=dec, use_credit=credit, use_smooth=smooth, theta_lo=0.62,
                                 tau=tau_schedule(0.9, t, 2), theta_hi=tau_schedule(0.9, t, 2),
                                 alpha_t=alpha_schedule(0.1, 0.05, 0.3, t))
                ctx.step(hbuf, Wd, Ed, em, mask, tok, cids, cval, pt, com, sm, None)
                n += 1
                t += 1
                if not bool(mask.any().item()) or t >= S:  # device -> host read: the host decides
                    break
            Xh[:, P + blk * S:P + (blk + 1) * S] = tok.view(B, S)
            if bool((tok == synth.eos_id(V)).any().item()):
                break
        e1.record(st)
        e1.synchronize()
        if r:
            alg1.append(e0.elapsed_time(e1))
            F_host = n
    g, h_, al = float(np.median(times)), float(np.median(host)), float(np.median(alg1))
    print(json.dumps({"config": a.config, "blocks": a.blocks, "F": F, "T": int(o[0]), "tpf": o[0] / max(F, 1),
                      "loop_ms": g, "loop_us_per_forward": 1e3 * g / F,
                      "host_steps_ms": h_, "host_us_per_step": 1e3 * h_ / F,
                      "host_alg1_forwards": F_host, "host_alg1_us_per_forward": 1e3 * al / max(F_host, 1)}))


if __name__ == "__main__":
    main()
