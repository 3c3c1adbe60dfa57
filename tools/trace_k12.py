"""Per-CTA timeline of the fused K12 step (DINFER_TRACE=1) in the bench's
back-to-back regime: block-start steps chained on one stream, weight copies
rotated when the shard is smaller than 3x the L2; the LAST step is read.
  python tools/trace_k12.py [--shard G] [--steps 8]
--shard G: one rank of a G-way vocab shard (loopback record exchange).
Phases per CTA (us from the earliest K12 CTA start):
  start, first W stage landed, W phase done, first E MMA, E MMAs done,
  partial written (K2-slot exit), kernel exit (after the rank finalize)."""
import argparse
import math
import os
import sys

os.environ["DINFER_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shard", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    a = ap.parse_args()
    H, V, B, S, K = 2048, 157184, 1, 32, 32
    G = a.shard
    v0, v1 = synth.shard_range(V, 0, G)
    dev = lambda u: torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()
    Wfull = synth.make_W(V, H, 1)
    h = dev(synth.planted_hidden(Wfull, B * S, seed=0))
    W0 = dev(Wfull[v0:v1])
    del Wfull
    E0 = dev(synth.make_E(V, H, 2, rows=(v0, v1)))
    em = dev(synth.make_E(V, H, 2, rows=(V - 1, V))[0])
    R = max(1, min(4, math.ceil(3 * 126e6 / ((v1 - v0) * H * 4))))
    Ws, Es = [W0] + [W0.clone() for _ in range(R - 1)], [E0] + [E0.clone() for _ in range(R - 1)]
    st = torch.cuda.Stream()
    ctx = Context(B, S, H, K, V, V_local=v1 - v0, v_offset=v0, world=G, rank=0, stream=st.cuda_stream)
    if G > 1:
        ctx.exchange_loopback()
    p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True, alpha_t=0.1, block_start=True,
                    mask_id=V - 1)
    mask = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    tok = torch.full((B, S), V - 1, dtype=torch.int32, device="cuda")
    cids = torch.full((B, S, K), -1, dtype=torch.int32, device="cuda")
    cval = torch.zeros((B, S, K), dtype=torch.float32, device="cuda")
    com = torch.zeros((B, S), dtype=torch.uint8, device="cuda")
    sm = torch.zeros((B, S, H), dtype=torch.float32, device="cuda")
    stt = torch.zeros((B, S, 4), dtype=torch.float32, device="cuda")
    for i in range(a.steps):
        ctx.step(h, Ws[i % R], Es[i % R], em, mask, tok, cids, cval, p, com, sm, stt)
    torch.cuda.synchronize()
    ctx.sync()
    k1, k2, k34 = ctx.trace()
    k34 = k34[k34[:, 0] > 0]
    t0 = int(k1[:, 0].min())
    us = lambda x: (x.astype(np.int64) - t0) / 1e3
    g = ctx.geometry()
    print(f"shard {G}: V_local {v1 - v0}, {R} weight copies, geometry {g}")
    cols = [("start", k1[:, 0]), ("first W stage", k1[:, 1]), ("W done", k1[:, 2]), ("first E MMA", k2[:, 1]),
            ("E MMAs done", k2[:, 2]), ("write-out start", k2[:, 0]), ("record added", k2[:, 3]), ("exit", k1[:, 3])]
    for n, c in cols:
        x = us(c)
        print(f"  {n:16s} min {x.min():7.1f}  p10 {np.percentile(x, 10):7.1f}  med {np.median(x):7.1f}  "
              f"p90 {np.percentile(x, 90):7.1f}  max {x.max():7.1f} us")
    wph = (k1[:, 2].astype(np.int64) - k1[:, 1].astype(np.int64)) / 1e3
    eph = (k2[:, 2].astype(np.int64) - k2[:, 1].astype(np.int64)) / 1e3
    wb = (v1 - v0) * H * 2
    print(f"  per-CTA W phase med {np.median(wph):.1f} us ({wb / np.median(wph) / 1e6:.2f} TB/s at the median), "
          f"E phase med {np.median(eph):.1f} us ({wb / np.median(eph) / 1e6:.2f} TB/s)")
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(f"gpurun_out/trace_k12_g{G}.npz", k1=k1, k2=k2, k34=k34, t0=t0)
    x = us(k34[:, 1]), us(k34[:, 3])
    print(f"  K34: deps visible min {x[0].min():.1f} med {np.median(x[0]):.1f}; exit max {x[1].max():.1f} us "
          f"(last K12 exit {us(k1[:, 3]).max():.1f})")
    # K34 stamps per block: [entry, deps visible, phase mark, end, smid]; block 0 selects (mark = phase 1
    # done), the others smooth (mark = accumulators loaded)
    sel, smo = k34[:1], k34[1:]
    for name, blk in (("selection", sel), ("smoothing", smo)):
        if len(blk) == 0:
            continue
        e, d, m, z = (us(blk[:, j]) for j in range(4))
        print(f"  K34 {name:9s} entry med {np.median(e):6.1f}  deps med {np.median(d):6.1f}  "
              f"mark med {np.median(m):6.1f} max {m.max():6.1f}  end med {np.median(z):6.1f} max {z.max():6.1f} us")
    ctx.close()


if __name__ == "__main__":
    main()
