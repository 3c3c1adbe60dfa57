"""What the block reset between back-to-back steps costs: K chained
(block reset + step) pairs vs K chained steps alone (the state then decays
to all-decided; K12's streamed bytes are the same, K34's smoothing shrinks),
one event pair each, MoE shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402

H, V, B, S, K = 2048, 157184, 1, 32, 32
dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
W = synth.make_W(V, H, 1)
h = dev(synth.planted_hidden(W, B * S, seed=0))
Wd = dev(W)
del W
Ed = dev(synth.make_E(V, H, 2))
em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0])
stream = torch.cuda.Stream()
ctx = Context(B, S, H, K, V, stream=stream.cuda_stream)
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True, alpha_t=0.1)
z = lambda *sh, dt=torch.float32: torch.zeros(sh, dtype=dt, device="cuda")
mask, tok = z(B, S, dt=torch.uint8), z(B, S, dt=torch.int32)
cids, cval = z(B, S, K, dt=torch.int32), z(B, S, K)
com, sm, st = z(B, S, dt=torch.uint8), z(B, S, H), z(B, S, 4)
N = 40


def run(reset_each):
    ctx.block_reset(mask, tok, cids, cval, V - 1)
    for _ in range(3):
        ctx.block_reset(mask, tok, cids, cval, V - 1)
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.block_reset(mask, tok, cids, cval, V - 1)
    e0.record(stream)
    for _ in range(N):
        if reset_each:
            ctx.block_reset(mask, tok, cids, cval, V - 1)
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / N * 1e3


for rep in range(3):
    a, b = run(True), run(False)
    print(f"reset + step {a:.1f} us   step only {b:.1f} us   (difference {a - b:.1f} us)")
ctx.close()
