"""Diagnostics: one step per (V, H, B, S) case, synchronised, to localise a
failing kernel.  python tools/dbg_step.py V H B S [smooth]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402

V, H, B, S = (int(x) for x in sys.argv[1:5])
smooth = len(sys.argv) < 6 or sys.argv[5] != "0"
M, K = B * S, 32
dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
W, E = synth.make_W(V, H, 1), synth.make_E(V, H, 2)
ctx = Context(B, S, H, K, V, smooth_capable=True)
print("geometry", ctx.geometry(), flush=True)
h = dev(synth.planted_hidden(W, M, seed=3))
Wd, Ed, em = dev(W), dev(E), dev(E[V - 1])
mask = torch.ones(M, dtype=torch.uint8, device="cuda")
tok = torch.full((M,), V - 1, dtype=torch.int32, device="cuda")
cids = torch.full((M, K), -1, dtype=torch.int32, device="cuda")
cval = torch.zeros((M, K), dtype=torch.float32, device="cuda")
com = torch.zeros(M, dtype=torch.uint8, device="cuda")
sm = torch.zeros((M, H), dtype=torch.float32, device="cuda")
st = torch.zeros((M, 4), dtype=torch.float32, device="cuda")
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=smooth, theta_lo=0.62, alpha_t=0.2)
try:
    for i in range(3):
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
        torch.cuda.synchronize()
        ctx.sync()
        print("step", i, "ok: committed", int(com.sum()), "smoothed norm", float(sm.norm()), flush=True)
except Exception as e:  # noqa: BLE001
    print("FAILED", e)
    if os.environ.get("DINFER_K12_PROBE"):
        import ctypes
        from paper_2510_08666_b200.dinfer import lib
        f = lib().dinfer_debug_probe
        f.restype = ctypes.POINTER(ctypes.c_int)
        f.argtypes = [ctypes.c_void_p]
        ptr = f(ctx._h)
        g = ctx.geometry()["k1_grid"] if False else 148
        rows = [[ptr[b * 64 + w] for w in range(64)] for b in range(g)]
        for b, r in enumerate(rows):
            if r[0] != -1 or r[1] != -1 or r[8] != -1:
                print("block", b, "prog", r[:8])
                print("   bars", [(hex(r[8 + 2 * w] & 0xffffffff), hex(r[9 + 2 * w] & 0xffffffff)) for w in range(28)])
