"""Is the K12 CTA -> SM mapping stable across launches, and is the per-CTA
duration an SM property?  (DINFER_TRACE=1; MoE shape.)"""
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
ctx = Context(B, S, H, K, V, smooth_capable=True)
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True)
mask = torch.ones((B, S), dtype=torch.uint8, device="cuda")
tok = torch.full((B, S), V - 1, dtype=torch.int32, device="cuda")
cids = torch.full((B, S, K), -1, dtype=torch.int32, device="cuda")
cval = torch.zeros((B, S, K), dtype=torch.float32, device="cuda")
com = torch.zeros((B, S), dtype=torch.uint8, device="cuda")
sm = torch.zeros((B, S, H), dtype=torch.float32, device="cuda")
st = torch.zeros((B, S, 4), dtype=torch.float32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
runs = []
for it in range(12):
    flush.fill_(1.0)
    mask.fill_(1)
    cids.fill_(-1)
    ctx.step(h, Wd, Ed, em, mask, tok, cids, cval, p, com, sm, st)
    torch.cuda.synchronize()
    k1, k2, _ = ctx.trace()
    runs.append((k1.copy(), k2.copy()))
runs = runs[2:]
smid = np.array([r[0][:, 4] for r in runs])  # [run][cta]
print("CTA->SM mapping identical across launches:", bool((smid == smid[0]).all()),
      "; fraction of CTAs on the same SM as launch 0:", float((smid == smid[0]).mean()))
t0 = np.array([r[0][:, 0].min() for r in runs])
exit_ = np.array([(r[0][:, 3].astype(np.int64) - r[0][:, 0].min()) / 1e3 for r in runs])
wdur = np.array([(r[0][:, 2].astype(np.int64) - r[0][:, 1].astype(np.int64)) / 1e3 for r in runs])
edur = np.array([(r[1][:, 2].astype(np.int64) - r[1][:, 1].astype(np.int64)) / 1e3 for r in runs])
# per-SM means (index by SM id)
bysm_w, bysm_e = {}, {}
for r in range(len(runs)):
    for c in range(smid.shape[1]):
        bysm_w.setdefault(int(smid[r, c]), []).append(wdur[r, c])
        bysm_e.setdefault(int(smid[r, c]), []).append(edur[r, c])
sms = sorted(bysm_w)
mw = np.array([np.mean(bysm_w[s]) for s in sms]); me = np.array([np.mean(bysm_e[s]) for s in sms])
print(f"per-SM W phase mean {mw.min():.1f}..{mw.max():.1f} us, E phase {me.min():.1f}..{me.max():.1f} us; "
      f"corr(W, E) across SMs {np.corrcoef(mw, me)[0, 1]:.2f}")
half = len(runs) // 2
a = np.array([np.mean(bysm_w[s][:half]) for s in sms]); b_ = np.array([np.mean(bysm_w[s][half:]) for s in sms])
print(f"W phase per-SM split-half correlation {np.corrcoef(a, b_)[0, 1]:.2f}")
print("exit spread per launch (max - median):", [round(float(x.max() - np.median(x)), 1) for x in exit_])
# per-CTA (blockIdx) stability
cw = wdur.mean(axis=0)
print(f"per-CTA W phase mean {cw.min():.1f}..{cw.max():.1f}; split-half corr by CTA "
      f"{np.corrcoef(wdur[:half].mean(0), wdur[half:].mean(0))[0, 1]:.2f}")
