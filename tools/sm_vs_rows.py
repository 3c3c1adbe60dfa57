"""Does a K12 CTA's W-phase time follow its SM or its vocab rows?  Even
partition, roles rotated by 0 and by G/2 (DINFER_TRACE=1, MoE shape)."""
import ctypes
import os
import sys

os.environ["DINFER_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08666_b200 import Context, lib, make_params, synth  # noqa: E402

H, V, B, S, K = 2048, 157184, 1, 32, 32
dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
W = synth.make_W(V, H, 1)
h = dev(synth.planted_hidden(W, B * S, seed=0))
Wd = dev(W)
del W
Ed = dev(synth.make_E(V, H, 2))
em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0])
ctx = Context(B, S, H, K, V, smooth_capable=True)
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True)
z = lambda *sh, **kw: torch.zeros(sh, device="cuda", **kw)
mask, tok = z(B, S, dtype=torch.uint8), z(B, S, dtype=torch.int32)
cids, cval = z(B, S, K, dtype=torch.int32), z(B, S, K, dtype=torch.float32)
com, sm, st = z(B, S, dtype=torch.uint8), z(B, S, H, dtype=torch.float32), z(B, S, 4, dtype=torch.float32)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
f = lib().dinfer_debug_role_shift
f.argtypes = [ctypes.c_void_p, ctypes.c_int32]
G = ctx.geometry()["k1_grid"]


def run(shift, n=8):
    f(ctx._h, shift)
    ws = []
    for it in range(n + 1):
        flush.fill_(1.0)
        mask.fill_(1)
        cids.fill_(-1)
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
        torch.cuda.synchronize()
        k1, _, _ = ctx.trace()
        if it:
            ws.append((k1[:, 2].astype(np.int64) - k1[:, 0].astype(np.int64)) / 1e3)
    return np.mean(ws, axis=0)  # by blockIdx


a = run(0)
b = run(G // 2)
rot = np.roll(b, -(G // 2))  # b indexed by the role it played: role r = blockIdx + G/2
# a[i]: blockIdx i with role i.  b[i]: blockIdx i with role i + G/2.
print(f"W phase by blockIdx: shift 0 {a.min():.1f}..{a.max():.1f}, shift G/2 {b.min():.1f}..{b.max():.1f}")
print(f"corr keyed by SM (same blockIdx): {np.corrcoef(a, b)[0, 1]:.2f};  keyed by rows (same role): "
      f"{np.corrcoef(a, np.roll(b, G // 2))[0, 1]:.2f}")
