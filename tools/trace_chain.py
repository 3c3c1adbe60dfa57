"""Per-CTA timelines of two CHAINED steps (block reset + step, back to back on
one stream, as bench.py's headline loop runs them): two contexts share the
stream and alternate, so the trace of step n-1 (ctx A) and step n (ctx B)
survive side by side on one %globaltimer axis (DINFER_TRACE=1).
  python tools/trace_chain.py [balance]"""
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
ctxs = [Context(B, S, H, K, V, stream=stream.cuda_stream) for _ in range(2)]
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True, alpha_t=0.1)
if "balance" in sys.argv:
    for c in ctxs:
        c.balance(h, Wd, Ed, em, p, iters=4, mode="back_to_back")
mk = lambda: dict(mask=torch.ones((B, S), dtype=torch.uint8, device="cuda"),
                  tok=torch.full((B, S), V - 1, dtype=torch.int32, device="cuda"),
                  cids=torch.full((B, S, K), -1, dtype=torch.int32, device="cuda"),
                  cval=torch.zeros((B, S, K), dtype=torch.float32, device="cuda"),
                  com=torch.zeros((B, S), dtype=torch.uint8, device="cuda"),
                  sm=torch.zeros((B, S, H), dtype=torch.float32, device="cuda"),
                  st=torch.zeros((B, S, 4), dtype=torch.float32, device="cuda"))
bufs = [mk(), mk()]
torch.cuda.synchronize()
hist = []
for rep in range(int(os.environ.get('REPS', '3'))):
    for it in range(8):
        c, b = ctxs[it & 1], bufs[it & 1]
        c.block_reset(b["mask"], b["tok"], b["cids"], b["cval"], V - 1)
        c.step(h, Wd, Ed, em, b["mask"], b["tok"], b["cids"], b["cval"], p, b["com"], b["sm"], b["st"])
    torch.cuda.synchronize()
    (a1, a2, a34), (b1, b2, b34) = ctxs[0].trace(), ctxs[1].trace()
    a34, b34 = a34[a34[:, 0] > 0], b34[b34[:, 0] > 0]
    t0 = int(a1[:, 0].min())
    us = lambda x: (x.astype(np.int64) - t0) / 1e3

    def row(name, x):
        x = us(x)
        print(f"  {name:26s} min {x.min():7.1f}  p10 {np.percentile(x, 10):7.1f}  med {np.median(x):7.1f}  "
              f"p90 {np.percentile(x, 90):7.1f}  max {x.max():7.1f} us")

    print(f"--- rep {rep}: step n-1 (ctx A) and step n (ctx B), us from A's first K12 CTA start")
    for tag, k1, k2, k34 in (("A", a1, a2, a34), ("B", b1, b2, b34)):
        for i, n in enumerate(["K12 start", "K12 first W MMA", "K12 W epilogue done", "K12 exit"]):
            row(f"{tag} {n}", k1[:, i])
        for i, n in enumerate(["(W epi done)", "E first MMA", "E MMAs done", "(exit)"]):
            row(f"{tag} {n}", k2[:, i])
        for i, n in enumerate(["K34 start", "K34 deps visible", "K34 stats merged", "K34 exit"]):
            row(f"{tag} {n}", k34[:, i])
    period = (int(b1[:, 0].min()) - t0) / 1e3
    print(f"  step period (K12 start to K12 start): {period:.1f} us; "
          f"B K12 start after A K12 last exit: {(int(b1[:, 0].min()) - int(a2[:, 3].max())) / 1e3:.1f} us; "
          f"A K34 span {(int(a34[:, 3].max()) - int(a34[:, 0].min())) / 1e3:.1f} us")
    hist.append(((a1[:, 2].astype(np.int64) - int(a1[:, 1].min())) / 1e3,
                 (a1[:, 3].astype(np.int64) - int(a1[:, 1].min())) / 1e3))
# systematic or noise?  per-CTA W-done / exit (from the first W MMA) across reps,
# and (even partition: CTAs 2g, 2g+1 form vocab group g) within-pair differences
wd = np.array([h[0] for h in hist])
ex = np.array([h[1] for h in hist])
if len(hist) > 1:
    cw = np.corrcoef(wd[0], wd[-1])[0, 1]
    ce = np.corrcoef(ex[0], ex[-1])[0, 1]
    print(f"per-CTA correlation first vs last rep: W done {cw:.2f}, exit {ce:.2f}")
mw, me = wd.mean(axis=0), ex.mean(axis=0)
print(f"mean over reps: W done {mw.min():.1f}..{mw.max():.1f} (sd {mw.std():.1f}); exit {me.min():.1f}..{me.max():.1f} "
      f"(sd {me.std():.1f}); single-rep exit sd {ex.std(axis=1).mean():.1f}")
if "balance" not in sys.argv:
    dpair = np.abs(wd[:, 0::2] - wd[:, 1::2])
    epair = np.maximum(ex[:, 0::2], ex[:, 1::2])
    print(f"within-pair |W done diff|: median {np.median(dpair):.1f} p90 {np.percentile(dpair, 90):.1f} us; "
          f"pair exit (max of two) sd {epair.std(axis=1).mean():.1f}")
for c in ctxs:
    c.close()
