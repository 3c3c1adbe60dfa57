"""K12 per-CTA exit spread of the LAST of 8 chained steps (one context, block
reset + step back to back, as bench.py's headline loop), over REPS repetitions:
is the residual spread systematic (correlation across repetitions)?
  python tools/trace_single.py [even]"""
import os
import sys

os.environ["DINFER_TRACE"] = "1"
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
if "even" not in sys.argv:
    ctx.balance(h, Wd, Ed, em, p, iters=4, mode="back_to_back")
z = lambda *sh, dt=torch.float32: torch.zeros(sh, dtype=dt, device="cuda")
mask, tok = z(B, S, dt=torch.uint8), z(B, S, dt=torch.int32)
cids, cval = z(B, S, K, dt=torch.int32), z(B, S, K)
com, sm, st = z(B, S, dt=torch.uint8), z(B, S, H), z(B, S, 4)
torch.cuda.synchronize()
ex, wd = [], []
for rep in range(int(os.environ.get("REPS", "8"))):
    for it in range(8):
        ctx.block_reset(mask, tok, cids, cval, V - 1)
        ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    torch.cuda.synchronize()
    k1, k2, _ = ctx.trace()
    t0 = int(k1[:, 1].min())  # first W MMA of the grid
    ex.append((k1[:, 3].astype(np.int64) - t0) / 1e3)
    wd.append((k1[:, 2].astype(np.int64) - t0) / 1e3)
ex, wd = np.array(ex), np.array(wd)
print(f"exit (from the grid's first W MMA): per-rep max-median {np.mean(ex.max(1) - np.median(ex, 1)):.1f} us, "
      f"max-min {np.mean(ex.max(1) - ex.min(1)):.1f} us, sd {ex.std(1).mean():.1f}")
print(f"W done: per-rep max-median {np.mean(wd.max(1) - np.median(wd, 1)):.1f} us, sd {wd.std(1).mean():.1f}")
if len(ex) > 1:
    print(f"per-CTA exit correlation rep 0 vs last: {np.corrcoef(ex[0], ex[-1])[0, 1]:.2f}; "
          f"sd of per-CTA mean exits {ex.mean(0).std():.1f} us (systematic part)")
ctx.close()
