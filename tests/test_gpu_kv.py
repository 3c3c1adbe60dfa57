"""GPU parity of the vicinity KV-cache refresh (P:125-133,
P:368) against the oracle's vicinity_step on seeded synthetic layers:
region identical; cache rows inside the region within one bf16 rounding of
the oracle; rows outside the region bitwise untouched (stale); the attention
output within 2e-3 (normwise per row) of the oracle attention on the same
cache, and within 1e-2 of the oracle carried fully independently."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2510_08666_b200 import build
    build.build()
    return torch


def bf16_dev(x64):
    import torch
    return torch.from_numpy(np.asarray(x64, np.float64)).to(torch.float32).to(torch.bfloat16).cuda()


def to64(t):
    import torch
    return t.to(torch.float64).cpu().numpy()


def run_blocks(torch_cuda, L, H, prompt, S, nblocks, iters, seed, looks=(16, 16), warmup=4, check_rows=None):
    import torch
    from paper_2510_08666_b200 import VicinityKV
    rng = np.random.default_rng(seed)
    W = [O.round_bf16(rng.standard_normal((H, H)) / math.sqrt(H)) for _ in range(3)]
    X = O.round_bf16(rng.standard_normal((L, H)))
    Wd = [bf16_dev(w) for w in W]
    kv = VicinityKV(L, H, 128, looks[0], looks[1], warmup)
    Kc = torch.zeros((L, H), dtype=torch.bfloat16, device="cuda")
    Vc = torch.zeros((L, H), dtype=torch.bfloat16, device="cuda")
    out = torch.full((L, H), float("nan"), dtype=torch.float32, device="cuda")
    Ko, Vo = np.zeros((L, H)), np.zeros((L, H))  # the oracle's own cache, carried independently
    nh = H // 128
    first = True
    for blk in range(nblocks):
        start, end = prompt + blk * S, prompt + (blk + 1) * S
        for t in range(iters + 1):
            full = first or t == iters  # creation and the completed block's full refresh
            first = False
            # the layer input evolves: the block's rows every iteration, a few far rows now and then
            X[start:end] = O.round_bf16(X[start:end] + 0.3 * rng.standard_normal((S, H)))
            if t % 2 == 1:
                r = rng.integers(0, L, 3)
                X[r] = O.round_bf16(rng.standard_normal((3, H)))
            Xd = bf16_dev(X)
            Kb, Vb = Kc.clone(), Vc.clone()
            lo, hi = kv.step(Xd, *Wd, Kc, Vc, start, end, t, out, full=full)
            torch.cuda.synchronize()
            ref = O.vicinity_step(X, *W, Ko, Vo, start, end, t, nh, looks[0], looks[1], warmup, full=full)
            assert (lo, hi) == (ref["lo"], ref["hi"]), f"region blk {blk} t {t}"
            Ko, Vo = ref["K"], ref["V"]
            K64, V64 = to64(Kc), to64(Vc)
            # outside the region: bitwise untouched
            for a, b in ((Kc, Kb), (Vc, Vb)):
                assert torch.equal(a[:lo], b[:lo]) and torch.equal(a[hi:], b[hi:]), f"stale rows blk {blk} t {t}"
            # inside: one bf16 rounding of the fp32 projection (+ fp32-vs-fp64 accumulation near 0)
            for g, o in ((K64, Ko), (V64, Vo)):
                err = np.abs(g[lo:hi] - o[lo:hi]) - (2.0 ** -7) * np.abs(o[lo:hi]) - 2e-5
                assert err.max() <= 0, f"cache rows blk {blk} t {t}: {err.max():.3g}"
            rows = np.arange(lo, hi) if check_rows is None else np.intersect1d(np.arange(lo, hi), check_rows)
            og = out.cpu().numpy().astype(np.float64)[rows]
            Q = O.round_bf16(X[rows] @ W[0].T)
            same_cache = O.attention(Q, K64, V64, nh)
            rel = np.linalg.norm(og - same_cache, axis=1) / np.linalg.norm(same_cache, axis=1)
            assert rel.max() <= 2e-3, f"attention vs oracle on the GPU's cache {rel.max():.3g} blk {blk} t {t}"
            indep = ref["O"][rows - lo]
            rel2 = np.linalg.norm(og - indep, axis=1) / np.linalg.norm(indep, axis=1)
            assert rel2.max() <= 1e-2, f"attention vs independent oracle {rel2.max():.3g} blk {blk} t {t}"
    kv.close()


def test_vicinity_small_two_heads(torch_cuda):
    """L = 192 (prompt 64 + 4 blocks of 32), H = 256: warmup, vicinity windows,
    block-end full refresh, clipping at the sequence end."""
    run_blocks(torch_cuda, 192, 256, 64, 32, 4, 6, seed=1)


def test_vicinity_ragged_and_wide_looks(torch_cuda):
    """L = 200 (partial key tile), H = 384 (3 heads), looks 40 / 8, warmup 1."""
    run_blocks(torch_cuda, 200, 384, 40, 32, 3, 4, seed=2, looks=(40, 8), warmup=1)


def test_vicinity_exactness_limit(torch_cuda):
    """Looks covering the sequence: every forward is a full recompute."""
    run_blocks(torch_cuda, 128, 256, 32, 32, 2, 3, seed=3, looks=(128, 128), warmup=0)


@pytest.mark.slow
def test_vicinity_llada_moe_layer(torch_cuda):
    """LLaDA-MoE attention shape: H = 2048 (16 heads of 128), L = 64 + 1024
    (prompt + gen length 1024); two blocks, attention checked on sampled rows."""
    run_blocks(torch_cuda, 1088, 2048, 64, 32, 2, 5, seed=4, check_rows=np.arange(0, 1088, 37))


@pytest.mark.parametrize("geom", [("0", "4", "1"), ("1", "2", "2"), ("1", "3", "1")])
def test_vicinity_launch_modes_bitwise(torch_cuda, monkeypatch, geom):
    """The PDL chain (projections -> attention -> merge) and the projection's
    ring geometry (stages x K chunks per stage) change scheduling only: the
    cache rows and the attention output are bitwise those of the default
    launch (PDL on, 4 x 1), at the LLaDA-MoE attention shape (vicinity and
    full-refresh regions; the full refresh uses 224-position tiles whose
    epilogue tile exceeds a shallow ring)."""
    import torch
    from paper_2510_08666_b200 import VicinityKV
    L, H = 1088, 2048
    g = torch.Generator(device="cuda").manual_seed(7)
    W = [(torch.randn((H, H), device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16) for _ in range(3)]
    X = torch.randn((L, H), device="cuda", generator=g).to(torch.bfloat16)

    def run():
        kv = VicinityKV(L, H, 128, 16, 16, 4)
        Kc = torch.zeros((L, H), dtype=torch.bfloat16, device="cuda")
        Vc = torch.zeros_like(Kc)
        out = torch.zeros((L, H), dtype=torch.float32, device="cuda")
        res = []
        for t, full in ((0, True), (9, False)):
            kv.step(X, *W, Kc, Vc, 64 + 512, 64 + 544, t, out, full=full)
            torch.cuda.synchronize()
            res += [Kc.clone(), Vc.clone(), out.clone()]
        kv.close()
        return res

    ref = run()
    pdl, st, cps = geom
    monkeypatch.setenv("DINFER_KV_PDL", pdl)
    monkeypatch.setenv("DINFER_KV_PJ_STAGES", st)
    monkeypatch.setenv("DINFER_KV_PJ_CPS", cps)
    got = run()
    for a, b in zip(ref, got):
        assert torch.equal(a, b), geom
