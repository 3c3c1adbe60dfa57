"""Randomised property tests of the oracle (hypothesis; -m "not gpu"):
invariants that must hold for ANY small input, not just the fixtures --
each one a statement the paper fixes (cited) or an exact algebraic identity.
A plausible slip (a dropped term, a wrong index, a transposed operand, a
reversed comparison) breaks at least one of them on some drawn case."""
import math

import numpy as np
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle as O

SETTINGS = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def step_case(draw):
    B = draw(st.integers(1, 2))
    S = draw(st.integers(1, 12))
    H = draw(st.integers(2, 8))
    V = draw(st.integers(3, 40))
    seed = draw(st.integers(0, 2 ** 31 - 1))
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((V, H))
    E = rng.standard_normal((V, H))
    h = rng.standard_normal((B, S, H)) * draw(st.floats(0.1, 4.0))
    mask = rng.random((B, S)) < draw(st.floats(0.2, 1.0))
    tok = np.where(mask, V - 1, rng.integers(0, V, (B, S)))
    C = np.zeros((B, S, V))
    for b in range(B):
        for s in range(S):
            C[b, s, rng.choice(V, min(V, 3), replace=False)] = rng.random(min(V, 3)) * 2
    p = O.Params(decoder=draw(st.sampled_from([O.DEC_THRESHOLD, O.DEC_HIERARCHICAL])),
                 tau=draw(st.floats(0.0, 1.0)), theta_hi=draw(st.floats(0.5, 1.0)), theta_lo=draw(st.floats(0.0, 0.5)),
                 use_credit=draw(st.booleans()), c_alpha=draw(st.floats(0.0, 2.0)),
                 c_beta=draw(st.floats(0.05, 0.95)), c_gamma=draw(st.floats(0.05, 0.95)),
                 use_smooth=True, alpha_t=draw(st.floats(0.0, 1.0)),
                 hier_runs_after_hi=draw(st.booleans()), smooth_credit_fused=draw(st.booleans()))
    return h, W, E, E[V - 1], mask, tok, (C if p.use_credit else None), p


@SETTINGS
@given(step_case())
def test_step_invariants(case):
    """>= 1 commit per row with undecided positions (reading c2); every
    commit is an undecided position and takes the argmax of the fused logits
    (P:305); decided rows never change; credit touches only
    undecided rows (P:327 block scope, reading c7); smoothing is produced
    exactly for rows still masked."""
    h, W, E, em, mask, tok, C, p = case
    r = O.step(h, W, E, em, mask, tok, C, p)
    B, S = mask.shape
    for b in range(B):
        f = O.logits(h[b], W)
        ft = O.credit_fuse(f, r["C"][b], p.c_alpha) if p.use_credit else f
        if mask[b].any():
            assert r["committed"][b].sum() >= 1
        else:
            assert not r["committed"][b].any()
        for s in range(S):
            if r["committed"][b, s]:
                assert mask[b, s]
                assert r["tokens"][b, s] == int(np.argmax(ft[s]))
                assert not r["mask"][b, s]
            elif not mask[b, s]:
                assert r["tokens"][b, s] == tok[b, s] and not r["mask"][b, s]
            if p.use_credit and not mask[b, s]:
                np.testing.assert_array_equal(r["C"][b, s], C[b, s])
            if r["mask"][b, s]:
                assert np.all(np.isfinite(r["smoothed"][b, s]))
            else:
                assert np.all(np.isnan(r["smoothed"][b, s]))


@SETTINGS
@given(step_case(), st.integers(2, 5))
def test_shard_merge_is_exact(case, G):
    """Splitting the vocabulary into G contiguous shards and merging the
    per-shard (m, v*, l, acc) records reproduces the unsharded
    statistics: max, lowest-id argmax, log-sum-exp and the smoothing sum."""
    h, W, E, em, mask, tok, C, p = case
    V = W.shape[0]
    if G > V:
        return
    f = O.logits(h[0], W)
    m, vstar, lse, pstar = O.softmax_stats(f)
    bounds = [V * j // G for j in range(G + 1)]
    recs = [O.shard_record(f[:, bounds[j]:bounds[j + 1]], bounds[j], E[bounds[j]:bounds[j + 1]]) for j in range(G)]
    mr = O.merge_records(recs)
    np.testing.assert_array_equal(mr["m"], m)
    np.testing.assert_array_equal(mr["vstar"], vstar)
    np.testing.assert_allclose(mr["lse"], lse, rtol=1e-12)
    np.testing.assert_allclose(mr["acc"] / np.exp(mr["lse"] - mr["m"])[:, None], O.softmax(f) @ E, rtol=1e-10,
                               atol=1e-12)


@SETTINGS
@given(st.integers(1, 30), st.integers(0, 10), st.floats(0.05, 0.95), st.floats(0.05, 0.95),
       st.lists(st.floats(0.01, 1.0), min_size=1, max_size=8))
def test_credit_geometric_closed_form(V, v, beta, gamma, ps):
    """Credit on a stable top-1 token follows sum_j beta^(k-1-j) p_j^gamma
    exactly (Eq. credit-update); other tokens stay at zero."""
    v = v % V
    C = np.zeros((1, V))
    for pp in ps:
        C = O.credit_update(C, np.array([v]), np.array([pp]), np.array([True]), beta, gamma)
    k = len(ps)
    want = math.fsum(beta ** (k - 1 - j) * ps[j] ** gamma for j in range(k))
    assert abs(C[0, v] - want) <= 1e-12 * max(1.0, want)
    assert np.count_nonzero(C) == 1


@SETTINGS
@given(st.integers(4, 400), st.integers(0, 398), st.integers(1, 64), st.integers(0, 10), st.integers(0, 40),
       st.integers(0, 40), st.integers(0, 6))
def test_refresh_region_contains_block_and_is_clipped(L, start, S, t, pre, aft, warm):
    """The vicinity refresh region (reading c25) always contains the block,
    lies in [0, L), is everything during warmup, and otherwise is exactly the
    block widened by the looks."""
    start = start % L
    end = min(L, start + S)
    lo, hi = O.refresh_region(L, start, end, t, pre, aft, warm)
    assert 0 <= lo <= start and end <= hi <= L
    if t < warm:
        assert (lo, hi) == (0, L)
    else:
        assert lo == max(0, start - pre) and hi == min(L, end + aft)
