"""GPU parity: the CUDA path (via the C ABI) against the fp64 oracle on the
same seeded, margin-vetted synthetic inputs.  Decisions, ids, mask and credit
slots bit-exact; m / lse / p~ / smoothed within 2e-3 (north_star)."""
import numpy as np
import pytest

import oracle as O
from paper_2510_08666_b200 import synth
from tests.gpu_harness import GpuState, compare, gpu_params, replay, to_dev_bf16
from tests.trajectory import vetted_trajectory

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2510_08666_b200 import build
    build.build()
    return torch


_W_CACHE = {}


def weights(V, H):
    key = (V, H)
    if key not in _W_CACHE:
        _W_CACHE.clear()
        _W_CACHE[key] = (synth.make_W(V, H, 1), synth.make_E(V, H, 2))
    return _W_CACHE[key]


def run_trajectory(torch_cuda, V, H, B, S, K, seed, params_fn, use_credit, max_iters=None, embed=False, **kw):
    from paper_2510_08666_b200 import Context
    W, E = weights(V, H)
    _, _, _, steps = vetted_trajectory(W, E, B, S, seed, params_fn, max_iters=max_iters,
                                       use_credit_table=use_credit, **kw)
    ctx = Context(B, S, H, K, V, smooth_capable=B * S <= 256)  # M > 256: dense stats-only path
    Wd, Ed = to_dev_bf16(W), to_dev_bf16(E)
    emd = to_dev_bf16(E[synth.mask_id(V)])
    replay(ctx, Wd, Ed, emd, steps, B, S, H, K, V, E_bits=E if embed else None)
    ctx.close()
    return steps


def thr_params(tau=0.9):
    return lambda t: O.Params(decoder=O.DEC_THRESHOLD, tau=tau)


def hier_credit_smooth(t):
    return O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=O.tau_schedule(0.92, t, 4), theta_lo=0.62,
                    use_credit=True, use_smooth=True, alpha_t=O.alpha_schedule(0.1, 0.05, 0.3, t))


# ---------------------------------------------------------------- tiny config (BASELINE configs[0])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tiny_threshold_block(torch_cuda, seed):
    steps = run_trajectory(torch_cuda, 1024, 256, 1, 32, 32, seed, thr_params(0.9), False)
    assert not steps[-1]["result"]["mask"].any()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tiny_hier_credit_smooth_block(torch_cuda, seed):
    run_trajectory(torch_cuda, 1024, 256, 2, 32, 32, seed, hier_credit_smooth, True)


@pytest.mark.parametrize("seed", [3, 4])
def test_tiny_threshold_credit_smooth_variants(torch_cuda, seed):
    pf = lambda t: O.Params(decoder=O.DEC_THRESHOLD, tau=O.tau_schedule(0.8, t, 4), use_credit=True,
                            c_alpha=0.7, c_beta=0.8, c_gamma=0.4, use_smooth=True, alpha_t=0.3)
    run_trajectory(torch_cuda, 1024, 256, 2, 32, 32, seed, pf, True)
    pf2 = lambda t: O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=0.92, theta_lo=0.62, hier_runs_after_hi=True)
    run_trajectory(torch_cuda, 1024, 256, 1, 32, 32, seed, pf2, False)


# ---------------------------------------------------------------- ragged / edge shapes
def test_ragged_tail_and_odd_shapes(torch_cuda):
    """V = 1000 (slab tails of 8-row boxes), S = 20 (N padding), H = 384
    (128-wide smoothing slices), B = 3."""
    run_trajectory(torch_cuda, 1000, 384, 3, 20, 24, 5, hier_credit_smooth, True)


@pytest.mark.parametrize("hw", ["128", "256", "512", "1024"])
def test_k2_slice_widths(torch_cuda, monkeypatch, hw):
    """The smoothing mix gives the same result for every hidden-slice width
    (DINFER_K2_HW tuning override): H = 1024, V = 4096."""
    monkeypatch.setenv("DINFER_K2_HW", hw)
    run_trajectory(torch_cuda, 4096, 1024, 1, 32, 32, 8, hier_credit_smooth, True, max_iters=4)


@pytest.mark.parametrize("hres", ["0", "1"])
def test_k1_hidden_resident_or_streamed(torch_cuda, monkeypatch, hres):
    """K1 with the hidden block resident in smem or streamed with every W stage."""
    monkeypatch.setenv("DINFER_K1_HRES", hres)
    run_trajectory(torch_cuda, 3000, 512, 2, 32, 32, 10, hier_credit_smooth, True, max_iters=4)


@pytest.mark.parametrize("fused,stack", [("0", "1"), ("2", "1"), ("2", "0")])
def test_fused_and_two_kernel_smoothing_paths(torch_cuda, monkeypatch, fused, stack):
    """Smoothing steps run K12 (K1 + K2 in one kernel, N <= 64; DINFER_FUSED=2
    forces it even for vocabularies too small to fill the machine) or the
    two-kernel K1 -> K2 path (DINFER_FUSED=0); both must match the oracle: ragged vocab /
    odd shapes (V = 1000, H = 384, B = 3, S = 20), HS = 2 groups (H = 2048, the
    other-slab accumulator set in use), N = 64 (B = 2, S = 32)."""
    from paper_2510_08666_b200 import Context
    monkeypatch.setenv("DINFER_FUSED", fused)
    monkeypatch.setenv("DINFER_K12_STACK", stack)  # 1: one accumulator + stacked hi/lo MMA; 0: two sets
    ctx = Context(1, 32, 2048, 32, 4096, smooth_capable=True)
    g = ctx.geometry()
    ctx.close()
    assert g["fused"] == (fused != "0")
    if fused != "0":
        assert g["k2_hw"] == 1024 and g["k1_grid"] == 2 * g["k2_groups"]
    run_trajectory(torch_cuda, 1000, 384, 3, 20, 24, 5, hier_credit_smooth, True, max_iters=5)
    run_trajectory(torch_cuda, 4096, 2048, 1, 32, 32, 11, hier_credit_smooth, True, max_iters=4)
    run_trajectory(torch_cuda, 2048, 1024, 2, 32, 32, 12, hier_credit_smooth, True, max_iters=3)


@pytest.mark.parametrize("stack", ["1", "0"])
def test_fused_four_hidden_slices(torch_cuda, monkeypatch, stack):
    """K12 with SPG = HS = 4 slabs per vocab group (the other slabs' rows sum
    three partner slabs): H = 4096 with N = 32 (1024-wide slices), and
    H = 2048 with N = 64 (S = 64: 512-wide slices); both accumulator layouts."""
    from paper_2510_08666_b200 import Context
    monkeypatch.setenv("DINFER_FUSED", "2")
    monkeypatch.setenv("DINFER_K12_STACK", stack)
    for (V, H, B, S) in ((8192, 4096, 1, 32), (4096, 2048, 1, 64)):
        ctx = Context(B, S, H, 32, V, smooth_capable=True)
        g = ctx.geometry()
        ctx.close()
        assert g["fused"] == 1 and g["k1_grid"] == 4 * g["k2_groups"], g
        run_trajectory(torch_cuda, V, H, B, S, 32 if S == 32 else 64, 15, hier_credit_smooth, True, max_iters=3)


@pytest.mark.parametrize("fused", ["0", "2"])
def test_next_input_embedding(torch_cuda, monkeypatch, fused):
    """f2: dinfer_step_embed writes the next iteration's bf16 model input in
    the same K34 launch -- W_emb[token] for decided rows (bit-exact), bf16 of
    e_{t+1} for masked rows -- over whole trajectories (tiny B = 2, ragged
    V = 1000 / H = 384 / S = 20, and H = 2048 with two hidden slices)."""
    monkeypatch.setenv("DINFER_FUSED", fused)
    run_trajectory(torch_cuda, 1024, 256, 2, 32, 32, 0, hier_credit_smooth, True, embed=True)
    run_trajectory(torch_cuda, 1000, 384, 3, 20, 24, 5, hier_credit_smooth, True, max_iters=5, embed=True)
    run_trajectory(torch_cuda, 4096, 2048, 1, 32, 32, 11, hier_credit_smooth, True, max_iters=4, embed=True)


def hier_credit_fused_smooth(t):
    p = hier_credit_smooth(t)
    p.c_alpha = 2.0
    p.smooth_credit_fused = True
    return p


@pytest.mark.parametrize("fused", ["0", "2"])
def test_credit_fused_smoothing(torch_cuda, monkeypatch, fused):
    """f4: smoothing with softmax(f + c_alpha ln(1 + C)) (the distribution the
    decoder decided on) instead of the raw softmax, on both smoothing paths and
    together with the next-iteration input; the test also checks that the two
    variants differ well beyond the tolerance on these trajectories."""
    monkeypatch.setenv("DINFER_FUSED", fused)
    steps = run_trajectory(torch_cuda, 1024, 256, 2, 32, 32, 1, hier_credit_fused_smooth, True)
    run_trajectory(torch_cuda, 1000, 384, 3, 20, 24, 5, hier_credit_fused_smooth, True, max_iters=5, embed=True)
    run_trajectory(torch_cuda, 4096, 2048, 1, 32, 32, 11, hier_credit_fused_smooth, True, max_iters=4)
    W, E = weights(1024, 256)
    em = O.bf16_bits_to_f64(E[synth.mask_id(1024)])
    worst = 0.0
    for st in steps:
        p_raw = O.Params(**{**vars(st["params"]), "smooth_credit_fused": False})
        raw = O.step(O.bf16_bits_to_f64(st["h"]), O.bf16_bits_to_f64(W), O.bf16_bits_to_f64(E), em, st["mask"], st["tokens"], st["C"],
                     p_raw)["smoothed"]
        fz = st["result"]["smoothed"]
        ok = ~np.isnan(raw[..., 0])
        if ok.any():
            d = np.linalg.norm(raw[ok] - fz[ok], axis=-1) / np.linalg.norm(fz[ok], axis=-1)
            worst = max(worst, float(d.max()))
    assert worst > 10 * 2e-3, f"fused and raw smoothing indistinguishable here ({worst:.3g})"


def test_next_input_embedding_rejects_unsupported(torch_cuda):
    from paper_2510_08666_b200 import Context, DInferError
    import torch
    V, H, B, S, K = 1024, 256, 1, 32, 8
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V, smooth_capable=True)
    st = GpuState(B, S, H, K, synth.mask_id(V))
    emb = torch.zeros((B, S, H), dtype=torch.int16, device="cuda")
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=1))
    with pytest.raises(DInferError) as ei:  # no smoothing -> no e_{t+1} to feed
        ctx.step_embed(h, to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1]), st.mask, st.tokens, None, None,
                       gpu_params(O.Params()), st.committed, None, st.stats, emb)
    assert ei.value.status == 6
    with pytest.raises(DInferError) as ei:  # credit-fused smoothing without credit
        ctx.step(h, to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1]), st.mask, st.tokens, None, None,
                 gpu_params(O.Params(use_smooth=True, smooth_credit_fused=True)), st.committed, st.smoothed, st.stats)
    assert ei.value.status == 6
    ctx.close()


@pytest.mark.parametrize("mode,groups", [("after_forward", "0"), ("back_to_back", "0"), ("back_to_back", "1")])
def test_balanced_partition_matches_oracle(torch_cuda, monkeypatch, mode, groups):
    """dinfer_balance re-pairs CTAs and moves each group's split point to the
    measured per-SM rates (either calibration mode); the step's results must
    not change beyond fp32 summation order (decisions bit-exact), including
    with a skewed split, and with resized vocab groups (DINFER_BALANCE_GROUPS=1).
    An unknown mode is rejected."""
    monkeypatch.setenv("DINFER_BALANCE_GROUPS", groups)
    monkeypatch.setenv("DINFER_K12_STACK", "0")  # the two-slab geometry dinfer_balance calibrates
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 32768, 2048, 1, 32, 32
    W, E = weights(V, H)
    _, _, _, steps = vetted_trajectory(W, E, B, S, 13, hier_credit_smooth, max_iters=4, use_credit_table=True)
    ctx = Context(B, S, H, K, V, smooth_capable=True)
    assert ctx.geometry()["fused"] == 1
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[synth.mask_id(V)])
    h0, p0 = to_dev_bf16(steps[0]["h"].reshape(B * S, H)), gpu_params(steps[0]["params"])
    import ctypes
    from paper_2510_08666_b200.dinfer import lib
    rc = lib().dinfer_balance(ctx._h, h0.data_ptr(), Wd.data_ptr(), Ed.data_ptr(), emd.data_ptr(), ctypes.byref(p0),
                              3, 7)
    assert rc != 0  # DINFER_ERR_ARG: no such mode
    ctx.balance(h0, Wd, Ed, emd, p0, iters=3, mode=mode)
    replay(ctx, Wd, Ed, emd, steps, B, S, H, K, V)
    ctx.balance_reset()
    replay(ctx, Wd, Ed, emd, steps, B, S, H, K, V)
    ctx.close()


@pytest.mark.parametrize("mode", ["after_forward", "back_to_back"])
def test_calibrated_k1_slabs_match_oracle(torch_cuda, mode):
    """Stats-only contexts: dinfer_balance resizes K1's slabs to the measured
    per-SM rates; decisions stay bit-exact, statistics within tolerance
    (summation order only), and balance_reset restores the even slabs."""
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 32768, 2048, 1, 32, 32
    W, E = weights(V, H)
    _, _, _, steps = vetted_trajectory(W, E, B, S, 21, thr_params(0.9), max_iters=4)
    ctx = Context(B, S, H, K, V, smooth_capable=False)
    Wd = to_dev_bf16(W)
    ctx.balance(to_dev_bf16(steps[0]["h"].reshape(B * S, H)), Wd, None, None, gpu_params(steps[0]["params"]),
                iters=3, mode=mode)
    replay(ctx, Wd, None, None, steps, B, S, H, K, V)
    ctx.balance_reset()
    replay(ctx, Wd, None, None, steps, B, S, H, K, V)
    ctx.close()


def test_without_pdl(torch_cuda, monkeypatch):
    monkeypatch.setenv("DINFER_PDL", "0")
    run_trajectory(torch_cuda, 2048, 512, 2, 32, 32, 9, hier_credit_smooth, True, max_iters=4)


def test_max_M_256(torch_cuda):
    run_trajectory(torch_cuda, 2048, 128, 8, 32, 8, 6, thr_params(0.9), False, max_iters=3)


def test_S64_block(torch_cuda):
    run_trajectory(torch_cuda, 4096, 256, 2, 64, 64, 7, hier_credit_smooth, True, max_iters=6)


def test_empty_rows_are_noops(torch_cuda):
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 1024, 256, 2, 32, 4
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V)
    st = GpuState(B, S, H, K, synth.mask_id(V))
    st.mask[1].zero_()
    st.tokens[1] = torch.arange(S, dtype=torch.int32, device="cuda")
    h = synth.planted_hidden(W, B * S, seed=3)
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True))
    st.smoothed.fill_(7.0)
    ctx.step(to_dev_bf16(h), to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1]), st.mask, st.tokens, st.cids,
             st.cval, p, st.committed, st.smoothed, st.stats)
    ctx.sync()
    out = st.snapshot()
    assert not out["committed"][1].any() and out["committed"][0].sum() >= 1
    assert np.array_equal(out["tokens"][1], np.arange(S))
    assert (out["cids"][1] == -1).all()
    assert np.all(out["smoothed"][1] == 7.0)


def test_determinism_repeat(torch_cuda):
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 4096, 512, 1, 32, 8
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V)
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=9))
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True))
    ref = None
    for _ in range(20):
        st = GpuState(B, S, H, K, synth.mask_id(V))
        ctx.step(h, Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed, st.stats)
        torch.cuda.synchronize()
        out = st.snapshot()
        if ref is None:
            ref = out
        for k in ("committed", "tokens", "cids", "cval", "m", "lse", "ptilde"):
            assert np.array_equal(out[k], ref[k]), k
        assert np.array_equal(np.nan_to_num(out["smoothed"]), np.nan_to_num(ref["smoothed"]))


@pytest.mark.parametrize("fused", ["0", "2"])
def test_block_reset_back_to_back(torch_cuda, monkeypatch, fused):
    """dinfer_block_reset + dinfer_step chained back to back (PDL, no host sync,
    the bench's headline loop): every step equals a step on fresh state."""
    import torch
    monkeypatch.setenv("DINFER_FUSED", fused)
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 4096, 512, 1, 32, 8
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V)
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=11))
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True))
    fresh = GpuState(B, S, H, K, synth.mask_id(V))
    ctx.step(h, Wd, Ed, emd, fresh.mask, fresh.tokens, fresh.cids, fresh.cval, p, fresh.committed, fresh.smoothed,
             fresh.stats)
    torch.cuda.synchronize()
    ref = fresh.snapshot()
    assert ref["committed"].any()  # the step changes the state the reset has to undo
    st = GpuState(B, S, H, K, synth.mask_id(V))
    st.mask.zero_()
    st.tokens.fill_(3)
    st.cids.fill_(5)
    st.cval.fill_(2.0)
    torch.cuda.synchronize()
    for _ in range(4):
        ctx.block_reset(st.mask, st.tokens, st.cids, st.cval, synth.mask_id(V))
        ctx.step(h, Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed, st.stats)
    ctx.sync()
    out = st.snapshot()
    for k in ("committed", "tokens", "mask", "cids", "cval", "m", "lse", "ptilde"):
        assert np.array_equal(out[k], ref[k]), k
    assert np.array_equal(np.nan_to_num(out["smoothed"]), np.nan_to_num(ref["smoothed"]))
    ctx.close()


@pytest.mark.parametrize("fused,K", [("0", 8), ("2", 8), ("2", 40)])
def test_block_start_step_equals_reset_plus_step(torch_cuda, monkeypatch, fused, K):
    """params.block_start: a step on garbage state (not read) writes the same
    mask / tokens / credit slots / outputs as block reset + step (K <= 32
    register slots and the strided K > 32 path; fused and two-kernel)."""
    import torch
    monkeypatch.setenv("DINFER_FUSED", fused)
    from paper_2510_08666_b200 import Context
    V, H, B, S = 4096, 512, 2, 32
    W, E = weights(V, H)
    mid = synth.mask_id(V)
    ctx = Context(B, S, H, K, V)
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=17))
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[mid])
    op = O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True)
    ref = GpuState(B, S, H, K, mid)
    ctx.block_reset(ref.mask, ref.tokens, ref.cids, ref.cval, mid)
    ctx.step(h, Wd, Ed, emd, ref.mask, ref.tokens, ref.cids, ref.cval, gpu_params(op), ref.committed, ref.smoothed,
             ref.stats)
    ctx.sync()
    want = ref.snapshot()
    st = GpuState(B, S, H, K, mid)
    st.mask.zero_()
    st.tokens.fill_(5)
    st.cids.fill_(3)
    st.cval.fill_(-1.0)  # would be flagged if read
    p = gpu_params(op)
    p.block_start, p.mask_id = 1, mid
    torch.cuda.synchronize()
    for _ in range(2):  # back to back: the second step reads nothing the first wrote
        ctx.step(h, Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed, st.stats)
    ctx.sync()  # no device flag: the garbage state was not read
    got = st.snapshot()
    for k in ("committed", "tokens", "mask", "cids", "cval", "m", "lse", "ptilde"):
        assert np.array_equal(got[k], want[k]), k
    assert np.array_equal(np.nan_to_num(got["smoothed"]), np.nan_to_num(want["smoothed"]))
    p.mask_id = V  # out of range
    with pytest.raises(Exception):
        ctx.step(h, Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed, st.stats)
    ctx.close()


# ---------------------------------------------------------------- split phases / vocab sharding on one GPU
@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_split_phase_matches_oracle(torch_cuda, G):
    """Emulate G vocab shards on one GPU: one context per rank (no NCCL),
    dinfer_step_local per shard, records concatenated in rank order,
    dinfer_step_combine on the result -- the exact data flow of the NCCL
    allgather path.  Compared with the unsharded oracle."""
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 2048, 256, 2, 32, 32
    W, E = weights(V, H)
    _, _, _, steps = vetted_trajectory(W, E, B, S, 11, hier_credit_smooth, use_credit_table=True)
    Vl = V // G
    ctxs = [Context(B, S, H, K, V, V_local=Vl, v_offset=r * Vl, world=G, rank=r) for r in range(G)]
    Wd = [to_dev_bf16(W[r * Vl:(r + 1) * Vl]) for r in range(G)]
    Ed = [to_dev_bf16(E[r * Vl:(r + 1) * Vl]) for r in range(G)]
    emd = to_dev_bf16(E[synth.mask_id(V)])
    words = ctxs[0].record_words(True)
    recs = torch.zeros((G, words), dtype=torch.float32, device="cuda")
    st = GpuState(B, S, H, K, synth.mask_id(V))
    for t, step in enumerate(steps):
        p = step["params"]
        gp = gpu_params(p)
        hid = to_dev_bf16(step["h"].reshape(B * S, H))
        for r in range(G):
            ctxs[r].step_local(hid, Wd[r], Ed[r], st.mask, st.cids, gp, recs[r])
        ctxs[0].step_combine(recs, emd, st.mask, st.tokens, st.cids, st.cval, gp, st.committed, st.smoothed,
                             st.stats)
        torch.cuda.synchronize()
        ctxs[0].sync()
        compare(st.snapshot(), step["result"], step["mask"], p, where=f"G={G} iter {t}")


def test_step_host_matches_device_step(torch_cuda):
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 2048, 256, 1, 32, 8
    W, E = weights(V, H)
    h = synth.planted_hidden(W, B * S, seed=12)
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True, alpha_t=0.2))
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])
    ctx = Context(B, S, H, K, V)
    st = GpuState(B, S, H, K, V - 1)
    ctx.step(to_dev_bf16(h), Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed,
             st.stats)
    torch.cuda.synchronize()
    dev = st.snapshot()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hh = pin(h.view(np.int16))
    mask, tok = pin(np.ones((B, S), np.uint8)), pin(np.full((B, S), V - 1, np.int32))
    cids, cval = pin(np.full((B, S, K), -1, np.int32)), pin(np.zeros((B, S, K), np.float32))
    com, sm, sts = pin(np.zeros((B, S), np.uint8)), pin(np.full((B, S, H), np.nan, np.float32)), \
        pin(np.zeros((B, S, 4), np.float32))
    ctx.step_host(hh, Wd, Ed, emd, mask, tok, cids, cval, p, com, sm, sts)
    assert np.array_equal(com.numpy().astype(bool), dev["committed"])
    assert np.array_equal(tok.numpy(), dev["tokens"])
    assert np.array_equal(cids.numpy(), dev["cids"]) and np.array_equal(cval.numpy(), dev["cval"])
    still = mask.numpy().astype(bool)
    assert np.array_equal(sm.numpy()[still], dev["smoothed"][still])
    # the split form: enqueue, then wait + unpack
    mask.fill_(1); tok.fill_(V - 1); cids.fill_(-1); cval.zero_(); com.zero_(); sm.fill_(float("nan"))
    ctx.step_host_async(hh, Wd, Ed, emd, mask, tok, cids, cval, p, com, sm, sts)
    ctx.step_host_wait()
    assert np.array_equal(com.numpy().astype(bool), dev["committed"])
    assert np.array_equal(tok.numpy(), dev["tokens"])
    assert np.array_equal(cids.numpy(), dev["cids"]) and np.array_equal(cval.numpy(), dev["cval"])
    assert np.array_equal(sm.numpy()[still], dev["smoothed"][still])
    from paper_2510_08666_b200 import DInferError
    with pytest.raises(DInferError):
        ctx.step_host_wait()  # nothing pending


def test_step_host_graph_cache_rotating_weights(torch_cuda):
    """dinfer_step_host keeps a few captured graphs (LRU, keyed by the baked-in
    pointers and flags): callers rotating buffers -- here three weight sets,
    two of them copies of the same weights at other addresses, one different,
    more sets than cache slots in the second round -- must get, on every call,
    exactly the device step on the weights they passed."""
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 2048, 256, 1, 32, 8
    sets = []
    for seed_w in (0, 0, 5, 0, 7, 5):  # 6 buffers, 3 distinct weight sets
        W, E = weights(V, H) if seed_w == 0 else (synth.make_W(V, H, seed_w), synth.make_E(V, H, seed_w + 1))
        sets.append((W, to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])))
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True, alpha_t=0.2))
    ctx_d, ctx_h = Context(B, S, H, K, V), Context(B, S, H, K, V)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    mask, tok = pin(np.ones((B, S), np.uint8)), pin(np.full((B, S), V - 1, np.int32))
    cids, cval = pin(np.full((B, S, K), -1, np.int32)), pin(np.zeros((B, S, K), np.float32))
    com, sts = pin(np.zeros((B, S), np.uint8)), pin(np.zeros((B, S, 4), np.float32))
    sm = pin(np.full((B, S, H), np.nan, np.float32))
    for it, i in enumerate([0, 1, 2, 0, 1, 2, 3, 4, 5, 0, 4, 2]):
        W, Wd, Ed, emd = sets[i]
        h = synth.planted_hidden(W, B * S, seed=60 + it)
        hh = pin(h.view(np.int16))
        st = GpuState(B, S, H, K, V - 1)
        ctx_d.step(to_dev_bf16(h), Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed,
                   st.stats)
        torch.cuda.synchronize()
        dev = st.snapshot()
        mask.fill_(1); tok.fill_(V - 1); cids.fill_(-1); cval.zero_(); com.zero_(); sm.fill_(float("nan"))
        ctx_h.step_host(hh, Wd, Ed, emd, mask, tok, cids, cval, p, com, sm, sts)
        assert np.array_equal(com.numpy().astype(bool), dev["committed"]), it
        assert np.array_equal(tok.numpy(), dev["tokens"]), it
        assert np.array_equal(cids.numpy(), dev["cids"]) and np.array_equal(cval.numpy(), dev["cval"]), it
        still = mask.numpy().astype(bool)
        assert np.array_equal(sm.numpy()[still], dev["smoothed"][still]), it


@pytest.mark.parametrize("pinned", [True, False])
def test_step_host_graph_replay_follows_schedules(torch_cuda, pinned):
    """dinfer_step_host replays one captured CUDA graph across iterations; the
    per-step tau / alpha_t (linear schedules, App. A.1 / B.1) reach the kernels
    through the packed state upload. Each iteration must equal the device
    step run with the same parameters. Pageable buffers take the plain path."""
    import torch
    from paper_2510_08666_b200 import Context, make_params
    V, H, B, S, K = 2048, 256, 1, 32, 8
    W, E = weights(V, H)
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])
    ctx_d, ctx_h = Context(B, S, H, K, V), Context(B, S, H, K, V)
    st = GpuState(B, S, H, K, V - 1)
    wrap = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()) if pinned else \
        (lambda a: torch.from_numpy(np.ascontiguousarray(a)))
    mask, tok = wrap(np.ones((B, S), np.uint8)), wrap(np.full((B, S), V - 1, np.int32))
    cids, cval = wrap(np.full((B, S, K), -1, np.int32)), wrap(np.zeros((B, S, K), np.float32))
    com, sts = wrap(np.zeros((B, S), np.uint8)), wrap(np.zeros((B, S, 4), np.float32))
    sm = wrap(np.full((B, S, H), np.nan, np.float32))
    for t in range(4):
        h = synth.planted_hidden(W, B * S, seed=40 + t, t=t)
        p = make_params(decoder="hierarchical" if t < 3 else "threshold", tau=0.9 - 0.1 * t, theta_hi=0.8,
                        theta_lo=0.3 - 0.05 * t, use_credit=True, c_alpha=0.5 + 0.1 * t, c_beta=0.9,
                        c_gamma=0.3 + 0.15 * t, use_smooth=True, alpha_t=0.1 * (t + 1))
        ctx_d.step(to_dev_bf16(h), Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed,
                   st.smoothed, st.stats)
        torch.cuda.synchronize()
        dev = st.snapshot()
        hh = wrap(h.view(np.int16))
        was = mask.numpy().astype(bool).copy()
        ctx_h.step_host(hh, Wd, Ed, emd, mask, tok, cids, cval, p, com, sm, sts)
        assert np.array_equal(mask.numpy().astype(bool), dev["mask"]), t
        assert np.array_equal(com.numpy().astype(bool), dev["committed"]), t
        assert np.array_equal(tok.numpy(), dev["tokens"]), t
        assert np.array_equal(cids.numpy(), dev["cids"]) and np.array_equal(cval.numpy(), dev["cval"]), t
        assert np.array_equal(sts.numpy(), st.stats.cpu().numpy()), t
        assert np.array_equal(sm.numpy()[was], dev["smoothed"][was]), t


def test_credit_slot_overflow_is_reported(torch_cuda):
    """K = 1 slot cannot hold two different tokens: the device flag surfaces
    as DINFER_ERR_DEVICE through dinfer_sync."""
    import torch
    from paper_2510_08666_b200 import Context, DInferError
    V, H, B, S, K = 1024, 256, 1, 32, 1
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V)
    st = GpuState(B, S, H, K, V - 1)
    st.cids.fill_(V - 5)  # every slot occupied by a token that is never the argmax
    st.cval.fill_(0.5)
    p = gpu_params(O.Params(decoder=O.DEC_THRESHOLD, tau=0.99, use_credit=True))
    h = synth.planted_hidden(W, B * S, seed=13)
    ctx.step(to_dev_bf16(h), to_dev_bf16(W), None, None, st.mask, st.tokens, st.cids, st.cval, p, st.committed,
             None, st.stats)
    with pytest.raises(DInferError) as ei:
        ctx.sync()
    assert ei.value.status == 7
    ctx.sync()  # sticky flag cleared


@pytest.mark.parametrize("K", [8, 40])
@pytest.mark.parametrize("bad", ["negative", "out_of_range"])
def test_invalid_credit_slot_is_reported(torch_cuda, K, bad):
    """A negative credit value or an id outside the vocabulary in an
    undecided row's slots is a device-checked precondition: DINFER_ERR_DEVICE
    through dinfer_sync (K <= 32 register path and the strided K > 32 path)."""
    from paper_2510_08666_b200 import Context, DInferError
    V, H, B, S = 1024, 256, 1, 32
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V)
    st = GpuState(B, S, H, K, V - 1)
    p = gpu_params(O.Params(decoder=O.DEC_THRESHOLD, tau=0.9, use_credit=True))
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=13))
    Wd = to_dev_bf16(W)
    ctx.step(h, Wd, None, None, st.mask, st.tokens, st.cids, st.cval, p, st.committed, None, st.stats)
    ctx.sync()  # valid state: no flag
    st = GpuState(B, S, H, K, V - 1)
    if bad == "negative":
        st.cids[0, 3, 0] = 7
        st.cval[0, 3, 0] = -0.25
    else:
        st.cids[0, 3, 0] = V + 5
        st.cval[0, 3, 0] = 0.25
    ctx.step(h, Wd, None, None, st.mask, st.tokens, st.cids, st.cval, p, st.committed, None, st.stats)
    with pytest.raises(DInferError) as ei:
        ctx.sync()
    assert ei.value.status == 7
    ctx.sync()
    ctx.close()


# ---------------------------------------------------------------- full paper shapes
@pytest.mark.slow
def test_moe_shape_hier_credit_smooth(torch_cuda):
    """LLaDA-MoE shape (BASELINE configs[2]): H=2048, V=157184, block 32, bs1,
    hierarchical + credit + smoothing; the first 4 iterations of a block, in
    the launch configuration bench.py times (K12 fused, 148 CTAs)."""
    from paper_2510_08666_b200 import Context
    ctx = Context(1, 32, 2048, 32, 157184, smooth_capable=True)
    assert ctx.geometry()["fused"] == 1
    ctx.close()
    run_trajectory(torch_cuda, 157184, 2048, 1, 32, 32, 0, hier_credit_smooth, True, max_iters=4)


@pytest.mark.slow
def test_8b_shape_threshold(torch_cuda):
    """LLaDA-8B shape (BASELINE configs[1]): H=4096 (hidden streamed with W),
    V=126464, block 32, bs1, threshold decoding; 3 iterations."""
    run_trajectory(torch_cuda, 126464, 4096, 1, 32, 32, 1, thr_params(0.9), False, max_iters=3)


# ---------------------------------------------------------------- compute-bound path (M > 256, K1b)
def test_dense_path_threshold_and_hier(torch_cuda):
    """M = 512 positions (B=4 x S=128) -> the dense K1b path; whole trajectory."""
    run_trajectory(torch_cuda, 4096, 256, 4, 128, 8, 21, thr_params(0.9), False, max_iters=5)
    pf = lambda t: O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=O.tau_schedule(0.92, t, 4), theta_lo=0.62)
    run_trajectory(torch_cuda, 4096, 256, 4, 128, 8, 22, pf, False, max_iters=5)


def test_dense_path_ragged(torch_cuda):
    """M = 300 (partial 256-position block), V = 1000 (partial vocab block), H = 384."""
    run_trajectory(torch_cuda, 1000, 384, 3, 100, 8, 23, thr_params(0.85), False, max_iters=4)


def test_dense_path_rejects_credit_and_smoothing(torch_cuda):
    from paper_2510_08666_b200 import Context, DInferError
    with pytest.raises(DInferError):
        Context(4, 128, 256, 8, 4096, smooth_capable=True)  # smoothing workspace not offered for M > 256
    ctx = Context(4, 128, 256, 8, 4096, smooth_capable=False)
    W, E = weights(4096, 256)
    st = GpuState(4, 128, 256, 8, 4095)
    h = to_dev_bf16(synth.planted_hidden(W, 512, seed=1))
    with pytest.raises(DInferError) as ei:
        ctx.step(h, to_dev_bf16(W), None, None, st.mask, st.tokens, st.cids, st.cval,
                 gpu_params(O.Params(use_credit=True)), st.committed, None, st.stats)
    assert ei.value.status == 6


@pytest.mark.slow
def test_8b_bs64_block64_sampled_rows(torch_cuda):
    """LLaDA-8B shape bs64 x block 64 (BASELINE configs[4]): the GPU runs all
    64 batch rows (M = 4096); two batch rows are margin-vetted trajectories
    checked against the oracle (selection is per batch row), the rest are
    planted filler."""
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 126464, 4096, 64, 64, 8
    W, _ = weights(V, H)
    Wd = to_dev_bf16(W)
    sample = {5: 31, 40: 32}  # batch row -> trajectory seed
    trajs = {}
    for b, seed in sample.items():
        _, _, _, steps = vetted_trajectory(W, W[:8], 1, S, seed, thr_params(0.9), max_iters=2)
        trajs[b] = steps
    filler = synth.planted_hidden(W, B * S, seed=33).reshape(B, S, H)
    ctx = Context(B, S, H, K, V, smooth_capable=False)
    st = GpuState(B, S, H, K, synth.mask_id(V))
    for t in range(2):
        h = filler.copy()
        for b in sample:
            h[b] = trajs[b][t]["h"][0]
        p = trajs[5][t]["params"]
        ctx.step(to_dev_bf16(h.reshape(B * S, H)), Wd, None, None, st.mask, st.tokens, None, None, gpu_params(p),
                 st.committed, None, st.stats)
        torch.cuda.synchronize()
        ctx.sync()
        out = st.snapshot()
        for b in sample:
            gold = trajs[b][t]["result"]
            one = {k: (v[b:b + 1] if isinstance(v, np.ndarray) and v.ndim >= 1 and v.shape[0] == B else v)
                   for k, v in out.items()}
            compare(one, gold, trajs[b][t]["mask"], p, where=f"row {b} iter {t}")


# ---------------------------------------------------------------- round-2 API fixes
def test_inclusive_thresholds(torch_cuda):
    """params.inclusive (variant c1'): a position whose fp32 p~
    sits exactly on tau commits with '>=' and not with '>' (both sides of
    the comparison are the device's fp32 values: tau is set to the p~ the
    device reported)."""
    import torch
    from paper_2510_08666_b200 import Context, make_params
    V, H, B, S, K = 1024, 256, 1, 32, 8
    W, E = weights(V, H)
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=5))
    Wd = to_dev_bf16(W)
    ctx = Context(B, S, H, K, V, smooth_capable=False)
    st = GpuState(B, S, H, K, V - 1)
    ctx.step(h, Wd, None, None, st.mask, st.tokens, None, None, make_params(tau=1.0), st.committed, None, st.stats)
    torch.cuda.synchronize()
    pt = st.stats[0, :, 2].cpu().numpy()
    order = np.argsort(-pt)
    s_hi = int(order[1])  # the second best: not the fallback
    tau = float(pt[s_hi])
    assert pt[order[0]] > tau and np.sum(pt == tau) == 1
    for incl, want in ((False, {int(order[0])} | {int(s) for s in np.nonzero(pt > tau)[0]}),
                       (True, {int(s) for s in np.nonzero(pt >= tau)[0]})):
        st = GpuState(B, S, H, K, V - 1)
        ctx.step(h, Wd, None, None, st.mask, st.tokens, None, None, make_params(tau=tau, inclusive=incl),
                 st.committed, None, st.stats)
        torch.cuda.synchronize()
        got = set(np.nonzero(st.committed.cpu().numpy()[0])[0].tolist())
        assert got == want, (incl, got, want)
        assert (s_hi in got) == incl
    ctx.close()


def test_combine_block_start_writes_smoothed_rows(torch_cuda):
    """dinfer_step_combine with params.block_start on an all-decided (garbage)
    mask: every row counts as undecided at step start, so the smoothing output
    is written for every row still masked (the mask snapshot must
    not be copied from the unread mask input)."""
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K = 2048, 256, 1, 32, 8
    W, E = weights(V, H)
    mid = synth.mask_id(V)
    G = 2
    Vl = V // G
    ctxs = [Context(B, S, H, K, V, V_local=Vl, v_offset=r * Vl, world=G, rank=r) for r in range(G)]
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=19))
    emd = to_dev_bf16(E[mid])
    op = O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True, alpha_t=0.2)
    words = ctxs[0].record_words(True)
    recs = torch.zeros((G, words), dtype=torch.float32, device="cuda")
    ref = GpuState(B, S, H, K, mid)
    for r in range(G):
        ctxs[r].step_local(h, to_dev_bf16(W[r * Vl:(r + 1) * Vl]), to_dev_bf16(E[r * Vl:(r + 1) * Vl]), ref.mask,
                           ref.cids, gpu_params(op), recs[r])
    ctxs[0].step_combine(recs, emd, ref.mask, ref.tokens, ref.cids, ref.cval, gpu_params(op), ref.committed,
                         ref.smoothed, ref.stats)
    torch.cuda.synchronize()
    want = ref.snapshot()
    p = gpu_params(op)
    p.block_start, p.mask_id = 1, mid
    st = GpuState(B, S, H, K, mid)
    st.mask.zero_()  # garbage: all decided
    st.cids.fill_(3)
    recs2 = torch.zeros_like(recs)
    for r in range(G):
        ctxs[r].step_local(h, to_dev_bf16(W[r * Vl:(r + 1) * Vl]), to_dev_bf16(E[r * Vl:(r + 1) * Vl]), st.mask,
                           st.cids, p, recs2[r])
    ctxs[0].step_combine(recs2, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed, st.stats)
    torch.cuda.synchronize()
    ctxs[0].sync()
    got = st.snapshot()
    for k in ("committed", "tokens", "mask", "cids", "cval", "m", "lse", "ptilde"):
        assert np.array_equal(got[k], want[k]), k
    still = want["mask"]
    assert still.any()
    # bitwise on the K1 -> K2 path; the fused K12 path (DINFER_FUSED=2) adds the
    # CTAs' accumulators with L2 reductions: equal to fp32 rounding order only
    np.testing.assert_allclose(got["smoothed"][still], want["smoothed"][still], rtol=1e-5, atol=1e-6)
    assert np.isfinite(got["smoothed"][still]).all()


def test_second_host_async_is_rejected(torch_cuda):
    """One pending dinfer_step_host_async per ctx (include/dinfer.h): a second
    call before _wait returns ERR_ARG and enqueues nothing."""
    import torch
    from paper_2510_08666_b200 import Context, DInferError
    V, H, B, S, K = 1024, 256, 1, 32, 8
    W, E = weights(V, H)
    Wd = to_dev_bf16(W)
    ctx = Context(B, S, H, K, V, smooth_capable=False)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hh = pin(synth.planted_hidden(W, B * S, seed=3).view(np.int16))
    mask, tok = pin(np.ones((B, S), np.uint8)), pin(np.full((B, S), V - 1, np.int32))
    com = pin(np.zeros((B, S), np.uint8))
    p = gpu_params(O.Params(decoder=O.DEC_THRESHOLD, tau=0.9))
    ctx.step_host_async(hh, Wd, None, None, mask, tok, None, None, p, com)
    with pytest.raises(DInferError) as ei:
        ctx.step_host_async(hh, Wd, None, None, mask, tok, None, None, p, com)
    assert ei.value.status == 1
    ctx.step_host_wait()
    assert com.numpy().sum() >= 1
    ctx.step_host_async(hh, Wd, None, None, mask, tok, None, None, p, com)  # accepted again
    ctx.step_host_wait()
    ctx.close()


def test_k12_reference_switch_for_far_larger_partner_max(torch_cuda, monkeypatch):
    """K12's single accumulator (stack mode) weighs the partner slabs' rows
    relative to the own slab's max; when a partner slab's max exceeds it by
    more than 32 nats the finished own-row sums are rescaled in TMEM to the
    partner's max (the rare path).  Planted: position 1 has one logit of ~40
    in a vocab row of the second slab of a group whose first slab stays near
    0 (and position 0 one of ~60, so the tau = 1 fallback commits position 0
    and position 1's smoothed row -- the rescaled one -- is compared with the
    oracle's fp64 softmax(z) W_emb, App. A.1)."""
    import torch
    from paper_2510_08666_b200 import Context
    monkeypatch.setenv("DINFER_FUSED", "2")
    monkeypatch.setenv("DINFER_K12_STACK", "1")
    V, H, B, S, K = 8192, 2048, 1, 32, 8  # groups of 3-4 chunks: both slabs non-empty
    W, E = weights(V, H)
    W = W.copy()
    h = synth.planted_hidden(W, B * S, seed=21).reshape(B * S, H)
    ctx = Context(B, S, H, K, V, smooth_capable=True)
    g = ctx.geometry()
    assert g["fused"] == 1 and g["k1_grid"] == 2 * g["k2_groups"]
    # group 3's rows are chunks [3 * nch / VG, 4 * nch / VG) of 32 rows; its second slab starts halfway
    nch, VG = (V + 31) // 32, g["k2_groups"]
    g0, g1 = 3 * nch // VG, 4 * nch // VG
    v_far = (g0 + (g1 - g0) // 2) * 32 + (g1 - g0) * 8  # a row of the group's second slab
    v_top = 7 * nch // VG * 32 + 5
    hf = O.bf16_bits_to_f64(h)
    for s_, v_, f_ in ((1, v_far, 40.0), (0, v_top, 60.0)):
        hv = hf[s_]
        W[v_] = synth.bf16_round(f_ * hv / np.dot(hv, hv))
    W64, E64 = O.bf16_bits_to_f64(W), O.bf16_bits_to_f64(E)
    p = O.Params(decoder=O.DEC_THRESHOLD, tau=1.0, use_credit=False, use_smooth=True, alpha_t=0.3)
    mask = np.ones((B, S), bool)
    res = O.step(hf.reshape(B, S, H), W64, E64, E64[synth.mask_id(V)], mask, np.full((B, S), synth.mask_id(V)),
                 None, p)
    assert res["committed"][0].nonzero()[0].tolist() == [0]
    f1 = O.logits(hf[1:2], W64)[0]
    assert f1[v_far] > 35 and f1[g0 * 32:(g0 + (g1 - g0) // 2) * 32].max() < 5  # the planted gap
    st = GpuState(B, S, H, K, synth.mask_id(V))
    ctx.step(to_dev_bf16(h), to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[synth.mask_id(V)]), st.mask, st.tokens,
             None, None, gpu_params(p), st.committed, st.smoothed, st.stats)
    torch.cuda.synchronize()
    ctx.sync()
    compare(st.snapshot(), res, mask, p, where="reference switch")
    ctx.close()


def test_nccl_allgather_path_one_rank(torch_cuda, monkeypatch):
    """The NCCL fallback exchange (BJ:5: records combined with NCCL) on a
    one-rank communicator (the only NCCL topology one GPU allows: NCCL rejects
    two ranks on one device): K12 in record mode, ncclAllGather of the packed
    rank record, K34 over the gathered records -- against the oracle along a
    vetted trajectory, and the allgather phase actually timed."""
    from paper_2510_08666_b200 import Context
    monkeypatch.setenv("DINFER_NCCL_WORLD1", "1")
    run_trajectory(torch_cuda, 4096, 1024, 1, 32, 32, 8, hier_credit_smooth, True, max_iters=4)
    run_trajectory(torch_cuda, 1000, 384, 3, 20, 24, 5, hier_credit_smooth, True, max_iters=4)
    # the step went through the allgather
    V, H, B, S, K = 4096, 1024, 1, 32, 32
    W, E = weights(V, H)
    ctx = Context(B, S, H, K, V, smooth_capable=True)
    ctx.set_timing(True)
    st = GpuState(B, S, H, K, synth.mask_id(V))
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=3))
    p = gpu_params(hier_credit_smooth(0))
    ctx.step(h, to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[synth.mask_id(V)]), st.mask, st.tokens, st.cids,
             st.cval, p, st.committed, st.smoothed, st.stats)
    torch_cuda.cuda.synchronize()
    ctx.sync()
    assert ctx.get_timing()["c1_allgather"] > 0.0
    ctx.close()


def test_step_host_graph_sharded_loopback(torch_cuda):
    """dinfer_step_host at world 2 with the peer-memory exchange (loopback: the
    rank's own record stands for both) replays captured graphs too: each call
    equals the device step of a second context -- decisions and credit slots
    bitwise, smoothed within 1e-5 (the record's fp32 L2 reductions are
    reproducible to rounding order only)."""
    import torch
    from paper_2510_08666_b200 import Context
    V, H, B, S, K, G = 8192, 2048, 1, 32, 8, 2
    W, E = weights(V, H)
    Vl = V // G
    Wd, Ed = to_dev_bf16(W[:Vl]), to_dev_bf16(E[:Vl])
    emd = to_dev_bf16(E[V - 1])
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True, alpha_t=0.2))
    ctx_d = Context(B, S, H, K, V, V_local=Vl, v_offset=0, world=G, rank=0)
    ctx_h = Context(B, S, H, K, V, V_local=Vl, v_offset=0, world=G, rank=0)
    ctx_d.exchange_loopback()
    ctx_h.exchange_loopback()
    assert ctx_h.geometry()["fused"] == 1
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    mask, tok = pin(np.ones((B, S), np.uint8)), pin(np.full((B, S), V - 1, np.int32))
    cids, cval = pin(np.full((B, S, K), -1, np.int32)), pin(np.zeros((B, S, K), np.float32))
    com, sts = pin(np.zeros((B, S), np.uint8)), pin(np.zeros((B, S, 4), np.float32))
    sm = pin(np.full((B, S, H), np.nan, np.float32))
    for it in range(4):
        h = synth.planted_hidden(W, B * S, seed=80 + it)
        st = GpuState(B, S, H, K, V - 1)
        ctx_d.step(to_dev_bf16(h), Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval, p, st.committed, st.smoothed,
                   st.stats)
        torch.cuda.synchronize()
        ctx_d.sync()
        dev = st.snapshot()
        mask.fill_(1); tok.fill_(V - 1); cids.fill_(-1); cval.zero_(); com.zero_(); sm.fill_(float("nan"))
        ctx_h.step_host(pin(h.view(np.int16)), Wd, Ed, emd, mask, tok, cids, cval, p, com, sm, sts)
        ctx_h.sync()
        assert np.array_equal(com.numpy().astype(bool), dev["committed"]), it
        assert np.array_equal(tok.numpy(), dev["tokens"]), it
        assert np.array_equal(cids.numpy(), dev["cids"]), it
        assert np.allclose(cval.numpy(), dev["cval"], rtol=1e-6, atol=0), it
        still = mask.numpy().astype(bool)
        a, b = sm.numpy()[still], dev["smoothed"][still]
        assert np.all(np.linalg.norm(a - b, axis=-1) <= 1e-5 * np.linalg.norm(b, axis=-1)), it
    ctx_d.close()
    ctx_h.close()
