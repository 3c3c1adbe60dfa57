"""Per-CTA timelines of K1, K2 and K34 for one step (DINFER_TRACE=1).
  python tools/trace_step.py [8b|tiny]"""
import os
import sys

os.environ["DINFER_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402

H, V = (4096, 126464) if "8b" in sys.argv else (256, 1024) if "tiny" in sys.argv else (2048, 157184)
smooth = "8b" not in sys.argv and "tiny" not in sys.argv
B, S, K = 1, 32, 32
dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
W = synth.make_W(V, H, 1)
h = dev(synth.planted_hidden(W, B * S, seed=0))
Wd = dev(W)
del W
Ed = dev(synth.make_E(V, H, 2)) if smooth else None
em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0]) if smooth else None
ctx = Context(B, S, H, K, V, smooth_capable=smooth)
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=smooth)
if "balance" in sys.argv:
    ctx.balance(h, Wd, Ed, em, p, iters=4)
mask = torch.ones((B, S), dtype=torch.uint8, device="cuda")
tok = torch.full((B, S), V - 1, dtype=torch.int32, device="cuda")
cids = torch.full((B, S, K), -1, dtype=torch.int32, device="cuda")
cval = torch.zeros((B, S, K), dtype=torch.float32, device="cuda")
com = torch.zeros((B, S), dtype=torch.uint8, device="cuda")
sm = torch.zeros((B, S, H), dtype=torch.float32, device="cuda") if smooth else None
st = torch.zeros((B, S, 4), dtype=torch.float32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
runs = []
for it in range(6):
    flush.fill_(1.0)
    mask.fill_(1)
    cids.fill_(-1)
    ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    torch.cuda.synchronize()
    runs.append(tuple(x.copy() for x in ctx.trace()))
k1, k2, k34 = runs[-1]
k34 = k34[k34[:, 0] > 0]
t0 = int(k1[:, 0].min())
us = lambda a: (a.astype(np.int64) - t0) / 1e3


def row(name, a):
    a = us(a)
    print(f"  {name:22s} min {a.min():7.1f}  p10 {np.percentile(a, 10):7.1f}  med {np.median(a):7.1f}  "
          f"p90 {np.percentile(a, 90):7.1f}  max {a.max():7.1f} us")


print("K1 (148 CTAs), us from first K1 CTA start:")
for i, n in enumerate(["start", "first W stage", "last tile done", "exit"]):
    row(n, k1[:, i])
if smooth:
    print("K2:")
    for i, n in enumerate(["start", "first MMA (E+P)", "MMAs done", "exit"]):
        row(n, k2[:, i])
    print(f"  step span: {us(k2[:, 3]).max():.1f} us (K1 start -> last K2 CTA exit)")
    g = ctx.geometry()
    if g.get("fused"):
        e_bytes = V * H * 2 / len(k2)
        dur = (k2[:, 2].astype(np.int64) - k2[:, 1].astype(np.int64)) / 1e3
        wdur = (k1[:, 2].astype(np.int64) - k1[:, 1].astype(np.int64)) / 1e3
        print(f"  K12 per-CTA W phase {np.median(wdur):.1f} us (med), E phase {np.median(dur):.1f} us (med) -> "
              f"E {e_bytes / np.median(dur) / 1e3 * len(k2) / 1e3:.2f} TB/s aggregate at the median; geometry {g}")
print(f"K34 ({len(k34)} traced blocks; the first B*ceil(S/8) are selection CTAs):")
for i, n in enumerate(["start", "deps visible", "stats merged", "exit"]):
    row(n, k34[:, i])
for j in range(4):
    print(f"  selection CTA {j}:", [round(float(x), 1) for x in us(k34[j, :4])])

# Systematic or random?  Per-SM K1 main-loop duration across repeated steps.
if len(runs) > 2:
    dur = {}
    for r1, _, _ in runs[1:]:
        for row in r1:
            dur.setdefault(int(row[4]), []).append((int(row[2]) - int(row[1])) / 1e3)
    sms = sorted(dur)
    d = np.array([dur[s_] for s_ in sms if len(dur[s_]) == len(runs) - 1])
    if len(d):
        mean = d.mean(axis=1)
        corr = np.corrcoef(d[:, 0], d[:, 1])[0, 1] if d.shape[1] > 1 else float("nan")
        print(f"K1 per-SM main-loop us over {d.shape[1]} steps: spread of per-SM means {mean.min():.1f}..{mean.max():.1f}, "
              f"step-to-step correlation {corr:.2f}")
        order = np.argsort(mean)
        print("  slowest SMs:", [(sms[i], round(float(mean[i]), 1)) for i in order[-6:]])
        print("  fastest SMs:", [(sms[i], round(float(mean[i]), 1)) for i in order[:6]])
