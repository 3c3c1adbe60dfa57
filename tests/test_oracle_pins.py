"""Pins for the CPU oracle (run with -m "not gpu").

Each test checks oracle/ against something other than itself: a value printed
in SPEC.md's worked examples (tests/golden/, cited), a closed form, a special
case that reduces to a textbook operation, brute force in pure Python on tiny
inputs, or an invariant the paper states.  A plausible slip anywhere in the
oracle (a dropped term, a sign, a transposed operand, log vs log1p, >= vs >,
a wrong tie-break) fails at least one of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# --------------------------------------------------------------- logits
def test_logits_signed_basis_closed_form():
    """W rows = +-e_{v mod H}: f[s, v] = sign_v * h[s, v mod H] exactly.  Catches
    a transposed W or a wrong contraction axis."""
    rng = np.random.default_rng(0)
    H, V, M = 8, 21, 3
    W = np.zeros((V, H))
    sign = np.where(rng.uniform(size=V) < 0.5, -1.0, 1.0)
    for v in range(V):
        W[v, v % H] = sign[v]
    h = rng.standard_normal((M, H))
    f = O.logits(h, W)
    for s in range(M):
        for v in range(V):
            assert f[s, v] == sign[v] * h[s, v % H]


def test_logits_brute_force_pure_python():
    rng = np.random.default_rng(1)
    h = rng.standard_normal((2, 5)); W = rng.standard_normal((7, 5))
    f = O.logits(h, W)
    for s in range(2):
        for v in range(7):
            assert f[s, v] == pytest.approx(math.fsum(h[s, k] * W[v, k] for k in range(5)), rel=1e-14)


# ---------------------------------------------------- softmax stats
def test_stats_uniform_closed_form():
    """h = 0 -> all logits 0 -> lse = ln V, p* = 1/V, v* = 0 (lowest id on ties, c3)."""
    V = 1024
    f = np.zeros((3, V))
    m, vs, lse, ps = O.softmax_stats(f)
    assert np.all(vs == 0)
    np.testing.assert_allclose(lse, math.log(V), rtol=1e-15)
    np.testing.assert_allclose(ps, 1.0 / V, rtol=1e-13)


def test_stats_signed_basis_lse_closed_form():
    """Signed basis W: lse = ln sum_k (n+_k e^{h_k} + n-_k e^{-h_k})."""
    rng = np.random.default_rng(2)
    H, V = 16, 1024
    W = np.zeros((V, H)); sign = np.where(rng.uniform(size=V) < 0.5, -1.0, 1.0)
    for v in range(V):
        W[v, v % H] = sign[v]
    h = rng.standard_normal((4, H)) * 3
    m, vs, lse, ps = O.softmax_stats(O.logits(h, W))
    for s in range(4):
        tot = 0.0
        for k in range(H):
            npos = sum(1 for v in range(V) if v % H == k and sign[v] > 0)
            nneg = sum(1 for v in range(V) if v % H == k and sign[v] < 0)
            tot += npos * math.exp(h[s, k]) + nneg * math.exp(-h[s, k])
        assert lse[s] == pytest.approx(math.log(tot), rel=1e-13)


def test_stats_brute_force_and_tie_lowest_id():
    rng = np.random.default_rng(3)
    f = np.round(rng.standard_normal((5, 37)) * 2, 1)    # coarse -> ties happen
    f[0, 3] = f[0, 30] = f[0].max() + 1.0                 # planted tie
    m, vs, lse, ps = O.softmax_stats(f)
    for s in range(5):
        row = list(f[s])
        mx = max(row)
        assert vs[s] == min(v for v in range(37) if row[v] == mx)
        z = math.fsum(math.exp(x) for x in row)
        assert lse[s] == pytest.approx(math.log(z), rel=1e-13)
        assert ps[s] == pytest.approx(math.exp(row[vs[s]]) / z, rel=1e-12)
    assert vs[0] == 3


def test_stats_two_level_closed_form_and_pstar_is_one_over_l():
    """f = [a, 0, ..., 0]: p* = e^a / (e^a + V - 1); and p* = 1 / sum e^{f - m}."""
    V, a = 157184, 13.5
    f = np.zeros((1, V)); f[0, 77] = a
    m, vs, lse, ps = O.softmax_stats(f)
    assert vs[0] == 77
    assert ps[0] == pytest.approx(math.exp(a) / (math.exp(a) + V - 1), rel=1e-13)
    assert ps[0] == pytest.approx(1.0 / np.exp(f[0] - m[0]).sum(), rel=1e-13)


def test_softmax_rows_sum_to_one():
    f = np.random.default_rng(4).standard_normal((6, 300)) * 5
    np.testing.assert_allclose(O.softmax(f).sum(axis=1), 1.0, rtol=1e-12)


def test_planted_confidence_matches_sigmoid():
    """Planted h = s w_t / ||w_t||^2 gives p* ~ sigmoid(s - ln V)."""
    from paper_2510_08666_b200 import synth
    V, H = 1024, 256
    W = O.bf16_bits_to_f64(synth.make_W(V, H, seed=1))
    for s_amp in (8.0, 10.0, 12.0):
        h = s_amp * W[5] / (W[5] @ W[5])
        m, vs, lse, ps = O.softmax_stats(O.logits(h[None, :], W))
        assert vs[0] == 5
        pred = 1.0 / (1.0 + math.exp(-(s_amp - math.log(V))))
        assert abs(ps[0] - pred) < 0.03


# ------------------------------------------------------ credit (App. B.2)
def test_credit_update_spec_examples():
    g = _gold("spec_worked_examples.json")["credit_update"]
    for ex in g[:2]:
        C = np.zeros((1, 4)); C[0, 2] = ex["prior"]
        for _ in range(ex["steps"]):
            C = O.credit_update(C, np.array([2]), np.array([ex["pstar"]]), np.array([True]),
                                ex["beta"], ex["gamma"])
        assert C[0, 2] == pytest.approx(ex["expected"], rel=1e-12), ex["cite"]
    ex = g[2]
    C = np.zeros((1, 4)); C[0, 1] = ex["prior_other"]
    C = O.credit_update(C, np.array([2]), np.array([0.5]), np.array([True]), ex["beta"], ex["gamma"])
    assert C[0, 1] == pytest.approx(ex["expected_other"], rel=1e-12), ex["cite"]


def test_credit_geometric_closed_form_and_bound():
    """Same v*, prob p for k steps from 0: C = p^g (1 - b^k)/(1 - b) <= p^g/(1-b)."""
    beta, gamma, p = 0.9, 0.5, 0.37
    C = np.zeros((1, 3))
    for k in range(1, 40):
        C = O.credit_update(C, np.array([1]), np.array([p]), np.array([True]), beta, gamma)
        closed = p ** gamma * (1 - beta ** k) / (1 - beta)
        assert C[0, 1] == pytest.approx(closed, rel=1e-12)
        assert C[0, 1] <= p ** gamma / (1 - beta) + 1e-15
        assert C[0, 0] == 0 and C[0, 2] == 0


def test_credit_decided_rows_frozen():
    C = np.full((2, 3), 0.5)
    C2 = O.credit_update(C, np.array([0, 0]), np.array([0.9, 0.9]), np.array([False, True]), 0.9, 0.5)
    np.testing.assert_array_equal(C2[0], C[0])
    assert C2[1, 1] == pytest.approx(0.45)


def test_credit_monotone_while_stable_under_true_precondition():
    """C_t[v*] >= C_{t-1}[v*] iff p_t^g >= (1-b) C_{t-1}; a drop in p can decrease C."""
    beta, gamma = 0.9, 0.5
    C = np.zeros((1, 2)); prev = 0.0
    for p in (0.9, 0.9, 0.9):
        C = O.credit_update(C, np.array([0]), np.array([p]), np.array([True]), beta, gamma)
        assert p ** gamma >= (1 - beta) * prev and C[0, 0] >= prev
        prev = C[0, 0]
    C = O.credit_update(C, np.array([0]), np.array([0.01]), np.array([True]), beta, gamma)
    assert 0.01 ** gamma < (1 - beta) * prev and C[0, 0] < prev


def test_credit_fuse_spec_example_and_identities():
    ex = _gold("spec_worked_examples.json")["credit_fuse"][0]
    ft = O.credit_fuse(np.array([ex["f"]]), np.array([ex["C"]]), ex["alpha"])
    np.testing.assert_allclose(ft[0], ex["expected_ftilde"], rtol=1e-15)
    v, p, _ = O.confidence(ft)
    assert v[0] == ex["expected_argmax"]
    # a real flip: raw argmax 1, fused argmax 0 (ln 2 > 0.5); 2-token closed form
    ft = O.credit_fuse(np.array([[2.0, 2.5]]), np.array([[1.0, 0.0]]), 1.0)
    v, p, _ = O.confidence(ft)
    assert v[0] == 0
    assert p[0] == pytest.approx(1 / (1 + math.exp(2.5 - 2.0 - math.log(2))), rel=1e-13)
    f = np.random.default_rng(5).standard_normal((3, 9))
    np.testing.assert_array_equal(O.credit_fuse(f, np.random.default_rng(6).uniform(size=(3, 9)), 0.0), f)
    np.testing.assert_array_equal(O.credit_fuse(f, np.zeros((3, 9)), 0.7), f)


def test_credit_fused_lse_shortcut_identity():
    """lse~ = ln(e^lse + sum_{v in cred} e^{f_v} ((1+C_v)^a - 1)): an algebraic
    identity independent of the dense fuse (pins log1p and the alpha power)."""
    rng = np.random.default_rng(7)
    f = rng.standard_normal((4, 50)) * 3
    C = np.zeros((4, 50))
    for s in range(4):
        C[s, rng.choice(50, 5, replace=False)] = rng.uniform(0, 3, 5)
    alpha = 0.8
    _, _, lse_t = O.confidence(O.credit_fuse(f, C, alpha))
    _, _, lse, _ = O.softmax_stats(f)
    for s in range(4):
        extra = math.fsum(math.exp(f[s, v]) * ((1 + C[s, v]) ** alpha - 1) for v in range(50) if C[s, v] > 0)
        assert lse_t[s] == pytest.approx(math.log(math.exp(lse[s]) + extra), rel=1e-12)


def test_credit_step_cs1_vector():
    """V=4, f=[2,1,.5,0], prior C=[0,.9,0,0], b=.9, g=.5, a=1.
    Credit after update: C[v*] = p*^g (v*=0), C[1] = .81; p~ from the 4-term
    closed form."""
    f = np.array([[2.0, 1.0, 0.5, 0.0]])
    C = np.array([[0.0, 0.9, 0.0, 0.0]])
    m, vs, lse, ps = O.softmax_stats(f)
    z = math.exp(2) + math.exp(1) + math.exp(0.5) + 1
    assert ps[0] == pytest.approx(math.exp(2) / z, rel=1e-13) and vs[0] == 0
    C2 = O.credit_update(C, vs, ps, np.array([True]), 0.9, 0.5)
    assert C2[0, 0] == pytest.approx(math.sqrt(math.exp(2) / z), rel=1e-13)
    assert C2[0, 1] == pytest.approx(0.81, rel=1e-13)
    v, p, lt = O.confidence(O.credit_fuse(f, C2, 1.0))
    num = math.exp(2) * (1 + C2[0, 0])
    den = num + math.exp(1) * 1.81 + math.exp(0.5) + 1
    assert v[0] == 0 and p[0] == pytest.approx(num / den, rel=1e-13)
    assert p[0] == pytest.approx(0.6322536210, abs=1e-9)


def test_credit_alpha_zero_equals_threshold_decoding():
    """Reduction law: credit with alpha = 0 commits exactly what
    threshold decoding commits, every step of a trajectory."""
    rng = np.random.default_rng(8)
    B, S, H, V = 1, 12, 8, 40
    W = rng.standard_normal((V, H)); E = rng.standard_normal((V, H))
    mask = np.ones((B, S), bool); tok = np.full((B, S), V - 1)
    C = np.zeros((B, S, V))
    mask2, tok2 = mask.copy(), tok.copy()
    pc = O.Params(decoder=O.DEC_THRESHOLD, tau=0.5, use_credit=True, c_alpha=0.0)
    pt = O.Params(decoder=O.DEC_THRESHOLD, tau=0.5)
    for it in range(S):
        h = rng.standard_normal((B, S, H)) * 2
        r1 = O.step(h, W, E, None, mask, tok, C, pc)
        r2 = O.step(h, W, E, None, mask2, tok2, None, pt)
        np.testing.assert_array_equal(r1["committed"], r2["committed"])
        np.testing.assert_array_equal(r1["tokens"], r2["tokens"])
        mask, tok, C = r1["mask"], r1["tokens"], r1["C"]
        mask2, tok2 = r2["mask"], r2["tokens"]
        if not mask.any():
            break


# ------------------------------------------------------------ threshold
def test_threshold_spec_examples():
    for ex in _gold("spec_worked_examples.json")["threshold"]:
        p = np.array(ex["pstar"])
        A = O.threshold_decode(p, np.ones(len(p), bool), ex["tau"])
        assert sorted(np.nonzero(A)[0].tolist()) == ex["expected"], ex["cite"]


def test_threshold_strict_and_fallback_and_degenerate():
    cases = _gold("hierarchical_examples.json")["cases"]
    t1 = [c for c in cases if c["name"] == "T1_threshold_strict"][0]
    A = O.threshold_decode(np.array(t1["ptilde"]), np.array(t1["mask"], bool), t1["tau"])
    assert np.nonzero(A)[0].tolist() == t1["expected_A"]
    # tau = 1.0: exactly one commit per step, even at p~ = 1.0 (c1)
    A = O.threshold_decode(np.array([1.0, 1.0, 0.3]), np.ones(3, bool), 1.0)
    assert A.tolist() == [True, False, False]
    # all above tau: whole block in one step
    assert O.threshold_decode(np.full(5, 0.99), np.ones(5, bool), 0.9).all()
    # decided positions are never committed
    A = O.threshold_decode(np.array([0.99, 0.2]), np.array([False, True]), 0.9)
    assert A.tolist() == [False, True]


def test_threshold_tau_one_takes_S_steps():
    rng = np.random.default_rng(9)
    S = 16; mask = np.ones(S, bool); steps = 0
    while mask.any():
        p = rng.uniform(0.5, 1.0, S)
        A = O.threshold_decode(p, mask, 1.0)
        assert A.sum() == 1
        mask &= ~A; steps += 1
    assert steps == S


# -------------------------------------------------- hierarchical (App. B.1)
def test_hierarchical_hand_examples():
    for c in _gold("hierarchical_examples.json")["cases"]:
        if c.get("decoder") == "threshold":
            continue
        p, m = np.array(c["ptilde"]), np.array(c["mask"], bool)
        A = O.hierarchical_decode(p, m, c["theta_hi"], c["theta_lo"])
        assert np.nonzero(A)[0].tolist() == c["expected_A"], c["name"]
        A2 = O.hierarchical_decode(p, m, c["theta_hi"], c["theta_lo"], runs_after_hi=True)
        assert np.nonzero(A2)[0].tolist() == c["expected_A_prime"], c["name"]
        if "expected_A_inclusive" in c:
            A3 = O.hierarchical_decode(p, m, c["theta_hi"], c["theta_lo"], inclusive=True)
            assert np.nonzero(A3)[0].tolist() == c["expected_A_inclusive"], c["name"]


def test_inclusive_variant_pins():
    """Variant c1' (comparisons '>='), hand-evaluated fixtures:
    T1 commits the position sitting exactly on tau; tau = 1.0 commits every
    saturated position (p~ = 1.0) instead of only the fallback; away from the
    thresholds both readings agree."""
    cases = _gold("hierarchical_examples.json")["cases"]
    t1 = [c for c in cases if c["name"] == "T1_threshold_strict"][0]
    A = O.threshold_decode(np.array(t1["ptilde"]), np.array(t1["mask"], bool), t1["tau"], inclusive=True)
    assert np.nonzero(A)[0].tolist() == t1["expected_A_inclusive"]
    A = O.threshold_decode(np.array([1.0, 1.0, 0.3]), np.ones(3, bool), 1.0, inclusive=True)
    assert A.tolist() == [True, True, False]
    rng = np.random.default_rng(12)
    for _ in range(200):
        S = int(rng.integers(1, 40))
        p = np.round(rng.uniform(0, 1, S), 3) + 2e-4  # never on a 3-decimal threshold
        m = rng.uniform(size=S) < 0.7
        for tau in (0.5, 0.8, 0.9):
            assert (O.threshold_decode(p, m, tau) == O.threshold_decode(p, m, tau, True)).all()
        assert (O.hierarchical_decode(p, m, 0.92, 0.62) == O.hierarchical_decode(p, m, 0.92, 0.62, inclusive=True)).all()


def test_hierarchical_saturated_and_floor():
    assert O.hierarchical_decode(np.full(8, 0.95), np.ones(8, bool), 0.92, 0.62).all()
    A = O.hierarchical_decode(np.array([0.1, 0.5, 0.2, 0.3]), np.ones(4, bool), 0.92, 0.62)
    assert A.sum() == 1 and A[1]


def test_hierarchical_superset_of_threshold_and_per_run_guarantee():
    rng = np.random.default_rng(10)
    for _ in range(300):
        S = int(rng.integers(1, 40))
        m = rng.uniform(size=S) < 0.7
        if not m.any():
            continue
        p = rng.uniform(size=S)
        tau = float(rng.uniform(0.3, 0.95))
        Ah = O.hierarchical_decode(p, m, tau, tau)
        At = O.threshold_decode(p, m, tau)
        assert np.all(Ah[At])
        Ah = O.hierarchical_decode(p, m, 0.92, 0.62)
        assert Ah.sum() >= 1 and not np.any(Ah & ~m)
        for first, last in O.undecided_runs(m):                 # c9 guarantee
            if p[first:last + 1].max() > 0.62:
                assert Ah[first:last + 1].any()


def test_hierarchical_ideal_depth_log2():
    """Ideal centre-peaked trace: every step the centre of each run is the only
    confident position; n masked positions finish in ceil(log2(n+1)) steps
    (P:299 'approach O(log n)')."""
    for n in (1, 2, 3, 7, 8, 31, 32, 64):
        mask = np.ones(n, bool); steps = 0
        while mask.any():
            p = np.full(n, 0.3)
            for first, last in O.undecided_runs(mask):
                p[(first + last) // 2] = 0.8
            A = O.hierarchical_decode(p, mask, 0.92, 0.62)
            mask &= ~A; steps += 1
        assert steps == math.ceil(math.log2(n + 1)), n


# ------------------------------------------------------------ smoothing (App. A.1)
def test_smoothing_alpha_zero_is_e_mask():
    rng = np.random.default_rng(11)
    f = rng.standard_normal((3, 20)); E = rng.standard_normal((20, 6)); em = rng.standard_normal(6)
    np.testing.assert_array_equal(O.smooth(f, E, em, 0.0), np.tile(em, (3, 1)))


def test_smoothing_uniform_is_mean_and_onehot_is_row():
    rng = np.random.default_rng(12)
    V, H = 64, 5
    E = rng.standard_normal((V, H)); em = rng.standard_normal(H)
    out = O.smooth(np.zeros((1, V)), E, em, 0.3)
    np.testing.assert_allclose(out[0], em + 0.3 * E.mean(axis=0), rtol=1e-12)
    f = np.full((1, V), -1e9); f[0, 17] = 0.0
    out = O.smooth(f, E, em, 0.3)
    np.testing.assert_allclose(out[0], em + 0.3 * E[17], atol=1e-6)


def test_smoothing_sm1_vector_and_convexity():
    """f = [2, 1, .5, 0], E = [[1,0],[0,1],[1,1],[-1,2]],
    e_mask = [.5, -.5], alpha = .1; brute-force weights in pure Python."""
    f = np.array([[2.0, 1.0, 0.5, 0.0]]); E = np.array([[1., 0.], [0., 1.], [1., 1.], [-1., 2.]])
    em = np.array([0.5, -0.5])
    z = math.fsum(math.exp(x) for x in f[0])
    de = [math.fsum(math.exp(f[0, v]) / z * E[v, k] for v in range(4)) for k in range(2)]
    out = O.smooth(f, E, em, 0.1)
    np.testing.assert_allclose(out[0], [0.5 + 0.1 * de[0], -0.5 + 0.1 * de[1]], rtol=1e-13)
    np.testing.assert_allclose(out[0], [0.5630114461, -0.4500864413], atol=1e-9)
    rng = np.random.default_rng(13)
    F = rng.standard_normal((10, 30)) * 4; E = rng.standard_normal((30, 7))
    de = O.smooth(F, E, np.zeros(7), 1.0)
    assert np.all(de <= E.max(axis=0) + 1e-12) and np.all(de >= E.min(axis=0) - 1e-12)


# ------------------------------------------------------------ credit-fused smoothing (f4)
def test_smooth_credit_fused_reductions_and_shortcut():
    """c_alpha = 0 and C = 0 reduce to raw smoothing; the credited-token
    shortcut (raw partial sums plus a correction over credited tokens only,
    the form the GPU computes) equals the dense definition; pure-Python brute
    force on a 5-token vocabulary."""
    rng = np.random.default_rng(31)
    V, H, R = 40, 5, 4
    f = rng.standard_normal((R, V)) * 3; E = rng.standard_normal((V, H)); em = rng.standard_normal(H)
    C = np.zeros((R, V))
    for r in range(R):
        C[r, rng.choice(V, 3, replace=False)] = rng.random(3) * 2
    np.testing.assert_allclose(O.smooth_credit_fused(f, C, E, em, 0.3, 0.0), O.smooth(f, E, em, 0.3), rtol=1e-13)
    np.testing.assert_allclose(O.smooth_credit_fused(f, np.zeros_like(C), E, em, 0.3, 1.3), O.smooth(f, E, em, 0.3),
                               rtol=1e-13)
    a = 0.8
    for r in range(R):
        m = f[r].max()
        acc = np.exp(f[r] - m) @ E
        l = np.exp(f[r] - m).sum()
        cred = np.nonzero(C[r])[0]
        w = np.exp(f[r, cred] - m) * ((1 + C[r, cred]) ** a - 1)
        short = em + 0.2 * (acc + w @ E[cred]) / (l + w.sum())
        np.testing.assert_allclose(O.smooth_credit_fused(f[r:r + 1], C[r:r + 1], E, em, 0.2, a)[0], short,
                                   rtol=1e-12)
    f5 = [1.0, 0.5, -0.2, 2.0, 0.0]; C5 = [0.0, 1.5, 0.0, 0.0, 0.7]; E5 = [[1, 2], [0, 1], [3, -1], [-2, 0], [1, 1]]
    ft = [f5[v] + 0.6 * math.log(1 + C5[v]) for v in range(5)]
    z = math.fsum(math.exp(x) for x in ft)
    de = [math.fsum(math.exp(ft[v]) / z * E5[v][k] for v in range(5)) for k in range(2)]
    got = O.smooth_credit_fused(np.array([f5]), np.array([C5]), np.array(E5, float), np.zeros(2), 1.0, 0.6)[0]
    np.testing.assert_allclose(got, de, rtol=1e-13)


def test_step_credit_fused_smoothing_uses_updated_credit():
    """Through a whole step: the fused variant smooths with the credit table
    AFTER this step's update (the one the decision used), and equals the raw
    variant when c_alpha = 0."""
    rng = np.random.default_rng(32)
    V, H, B, S = 48, 6, 1, 8
    W = rng.standard_normal((V, H)); E = rng.standard_normal((V, H)); em = rng.standard_normal(H)
    h = rng.standard_normal((B, S, H))
    mask = np.ones((B, S), bool); tok = np.full((B, S), V - 1)
    C = np.zeros((B, S, V)); C[0, :, 3] = 0.5; C[0, :, 7] = 1.2
    p = O.Params(tau=0.99, use_credit=True, c_alpha=0.9, use_smooth=True, alpha_t=0.25, smooth_credit_fused=True)
    res = O.step(h, W, E, em, mask, tok, C, p)
    f = O.logits(h[0], W)
    for s in np.nonzero(res["mask"][0])[0]:
        want = O.smooth(O.credit_fuse(f[s:s + 1], res["C"][0, s:s + 1], 0.9), E, em, 0.25)[0]
        np.testing.assert_allclose(res["smoothed"][0, s], want, rtol=1e-12)
    p0 = O.Params(**{**vars(p), "c_alpha": 0.0})
    r0 = O.step(h, W, E, em, mask, tok, C, p0)
    r1 = O.step(h, W, E, em, mask, tok, C, O.Params(**{**vars(p0), "smooth_credit_fused": False}))
    np.testing.assert_allclose(r0["smoothed"], r1["smoothed"], rtol=1e-13, equal_nan=True)


# ------------------------------------------------------------ next-iteration input (f2)
def test_next_input_embedding_rows():
    """Decided rows are the ordinary embedding lookup (numpy fancy indexing as
    the independent reference), masked rows are e_{t+1}; a fully decided block
    is exactly the plain lookup."""
    rng = np.random.default_rng(21)
    V, H, B, S = 50, 6, 2, 9
    E = rng.standard_normal((V, H)); tok = rng.integers(0, V, (B, S)); mask = rng.random((B, S)) < 0.5
    sm = rng.standard_normal((B, S, H))
    out = O.next_input_embedding(E, tok, mask, sm)
    np.testing.assert_array_equal(out, np.where(mask[..., None], sm, E[tok]))
    np.testing.assert_array_equal(O.next_input_embedding(E, tok, np.zeros((B, S), bool), sm), E[tok])


def test_next_input_embedding_after_step_and_onehot_limit():
    """Through a whole oracle step: with alpha_t = 0 every still-masked row is
    e_mask exactly and every committed row is W_emb[committed id]; the
    decided-row embedding is the one-hot limit of the smoothed one
    (alpha = 1, e_mask = 0, all mass on the committed token)."""
    rng = np.random.default_rng(22)
    V, H, B, S = 64, 8, 1, 12
    W = rng.standard_normal((V, H)); E = rng.standard_normal((V, H)); em = rng.standard_normal(H)
    h = rng.standard_normal((B, S, H)) * 2
    mask = np.ones((B, S), bool); tok = np.full((B, S), V - 1)
    res = O.step(h, W, E, em, mask, tok, None, O.Params(tau=0.3, use_smooth=True, alpha_t=0.0))
    out = O.next_input_embedding(E, res["tokens"], res["mask"], res["smoothed"])
    assert res["committed"].any() and res["mask"].any()
    for s in range(S):
        if res["mask"][0, s]:
            np.testing.assert_array_equal(out[0, s], em)
        else:
            v = res["tokens"][0, s]
            assert v == np.argmax(h[0, s] @ W.T)
            np.testing.assert_array_equal(out[0, s], E[v])
            f = np.full((1, V), -1e9); f[0, v] = 0.0
            np.testing.assert_allclose(O.smooth(f, E, np.zeros(H), 1.0)[0], out[0, s], atol=1e-9)


# ------------------------------------------------------------ schedules
def test_schedules_spec_examples_and_monotone():
    g = _gold("spec_worked_examples.json")
    for ex in g["alpha_schedule"]:
        assert O.alpha_schedule(ex["init"], ex["growth"], ex["preset"], ex["t"]) == pytest.approx(ex["expected"]), ex["cite"]
    for ex in g["tau_schedule"]:
        assert O.tau_schedule(ex["target"], ex["t"], ex["decay_steps"]) == pytest.approx(ex["expected"]), ex["cite"]
    a = [O.alpha_schedule(0.1, 0.05, 0.3, t) for t in range(20)]
    tau = [O.tau_schedule(0.8, t, 4) for t in range(20)]
    assert all(x <= y for x, y in zip(a, a[1:])) and all(x >= y for x, y in zip(tau, tau[1:]))


# ------------------------------------------------------------ shard merge (§8(e))
@pytest.mark.parametrize("G", [2, 4, 8])
def test_shard_merge_equals_unsharded(G):
    rng = np.random.default_rng(20 + G)
    M, V, H = 6, 64, 5
    f = rng.standard_normal((M, V)) * 4; E = rng.standard_normal((V, H))
    f[2, 10] = f[2, 50] = f[2].max() + 2                # cross-shard tie -> lowest id
    recs = [O.shard_record(f[:, r * V // G:(r + 1) * V // G], r * V // G, E[r * V // G:(r + 1) * V // G])
            for r in range(G)]
    mg = O.merge_records(recs)
    m, vs, lse, ps = O.softmax_stats(f)
    np.testing.assert_array_equal(mg["vstar"], vs)
    np.testing.assert_allclose(mg["lse"], lse, rtol=1e-13)
    np.testing.assert_allclose(mg["pstar"], ps, rtol=1e-12)
    np.testing.assert_allclose(mg["acc"] / mg["l"][:, None], O.softmax(f) @ E, rtol=1e-11, atol=1e-13)
    assert vs[2] == 10


# ------------------------------------------------------------ whole step invariants
def test_step_progress_and_commit_is_argmax():
    rng = np.random.default_rng(30)
    B, S, H, V = 2, 16, 8, 50
    W = rng.standard_normal((V, H)); E = rng.standard_normal((V, H)); em = E[V - 1]
    for dec in (O.DEC_THRESHOLD, O.DEC_HIERARCHICAL):
        mask = np.ones((B, S), bool); tok = np.full((B, S), V - 1); C = np.zeros((B, S, V))
        p = O.Params(decoder=dec, tau=0.9, use_credit=True, use_smooth=True, alpha_t=0.2)
        for it in range(S + 1):
            h = rng.standard_normal((B, S, H))
            r = O.step(h, W, E, em, mask, tok, C, p)
            for b in range(B):
                if mask[b].any():
                    assert r["committed"][b].sum() >= 1
                f = O.logits(h[b], W)
                ft = O.credit_fuse(f, r["C"][b], p.c_alpha)
                for s in np.nonzero(r["committed"][b])[0]:
                    assert r["tokens"][b, s] == np.argmax(ft[s])
                    assert mask[b, s]
                still = r["mask"][b]
                assert np.all(np.isnan(r["smoothed"][b][~still]))
                assert np.all(np.isfinite(r["smoothed"][b][still]))
            mask, tok, C = r["mask"], r["tokens"], r["C"]
            if not mask.any():
                break
        assert not mask.any()


def test_step_empty_row_is_noop():
    rng = np.random.default_rng(31)
    W = rng.standard_normal((20, 4))
    r = O.step(rng.standard_normal((1, 5, 4)), W, W, W[0], np.zeros((1, 5), bool),
               np.arange(5)[None, :], None, O.Params())
    assert not r["committed"].any() and np.array_equal(r["tokens"], np.arange(5)[None, :])


# ------------------------------------------------------------ vicinity KV-cache refresh (f3)
def test_refresh_region_spec_examples():
    """block [64,128), looks 16 after warmup -> [48,144);
    step 0 with warmup 4 -> everything; clipping at both ends; a block's
    completion (full) -> everything."""
    L = 256
    assert O.refresh_region(L, 64, 128, 4, 16, 16, 4) == (48, 144)
    assert O.refresh_region(L, 64, 128, 0, 16, 16, 4) == (0, L)
    assert O.refresh_region(L, 64, 128, 3, 16, 16, 4) == (0, L)
    assert O.refresh_region(L, 0, 32, 9, 16, 16, 4) == (0, 48)
    assert O.refresh_region(L, 224, 256, 9, 16, 16, 4) == (208, 256)
    assert O.refresh_region(L, 64, 128, 9, 16, 16, 4, full=True) == (0, L)


def test_round_bf16_against_bit_patterns():
    """Round-to-nearest-even to 8 significand bits: exact bf16 values are fixed
    points; midpoints go to the even neighbour; bf16 bit decoding agrees."""
    vals = O.bf16_bits_to_f64(np.arange(0x3f00, 0x4100, dtype=np.uint16))
    np.testing.assert_array_equal(O.round_bf16(vals), vals)
    assert O.round_bf16(np.array([1.0 + 2 ** -8]))[0] == 1.0                 # tie -> even (1.0)
    assert O.round_bf16(np.array([1.0 + 3 * 2 ** -8]))[0] == 1.0 + 2 ** -6   # tie -> even (1 + 2^-6)
    assert O.round_bf16(np.array([1.0 + 2 ** -8 + 1e-12]))[0] == 1.0 + 2 ** -7
    assert O.round_bf16(np.array([-3.0]))[0] == -3.0


def test_attention_brute_force_and_closed_forms():
    """Pure-Python softmax attention on 2 heads; K = 0 gives the mean of V per
    head (uniform weights); one key gives that key's V row."""
    rng = np.random.default_rng(41)
    R, L, H, nh = 3, 5, 4, 2
    Q = rng.standard_normal((R, H)); K = rng.standard_normal((L, H)); V = rng.standard_normal((L, H))
    out = O.attention(Q, K, V, nh)
    d = H // nh
    for r in range(R):
        for hh in range(nh):
            sc = [math.fsum(Q[r, hh * d + j] * K[k, hh * d + j] for j in range(d)) / math.sqrt(d) for k in range(L)]
            z = math.fsum(math.exp(x) for x in sc)
            for j in range(d):
                want = math.fsum(math.exp(sc[k]) / z * V[k, hh * d + j] for k in range(L))
                assert abs(out[r, hh * d + j] - want) < 1e-12
    np.testing.assert_allclose(O.attention(Q, np.zeros((L, H)), V, nh), np.tile(V.mean(axis=0), (R, 1)), rtol=1e-13)
    np.testing.assert_allclose(O.attention(Q, K[:1], V[:1], nh), np.tile(V[0], (R, 1)), rtol=1e-13)


def _layer(rng, L, H):
    W = [rng.standard_normal((H, H)) / math.sqrt(H) for _ in range(3)]
    return [O.round_bf16(w) for w in W]


def test_vicinity_exactness_limit_and_staleness():
    """Looks covering the whole sequence degenerate to a full recompute
    (bitwise in the oracle); otherwise rows outside the region keep
    their stale K/V exactly while the region's rows are recomputed from the
    current input; a full refresh makes the forward equal the no-cache one."""
    rng = np.random.default_rng(42)
    L, H, nh = 48, 16, 2
    Wq, Wk, Wv = _layer(rng, L, H)
    X0 = O.round_bf16(rng.standard_normal((L, H)))
    full = O.vicinity_step(X0, Wq, Wk, Wv, np.zeros((L, H)), np.zeros((L, H)), 16, 24, 0, nh, full=True)
    X1 = X0.copy(); X1[16:24] = O.round_bf16(rng.standard_normal((8, H)))   # the block's inputs evolve
    X1[35:40] = O.round_bf16(rng.standard_normal((5, H)))                    # and some far rows (stale keys)
    nocache = O.vicinity_step(X1, Wq, Wk, Wv, full["K"], full["V"], 16, 24, 9, nh, full=True)
    wide = O.vicinity_step(X1, Wq, Wk, Wv, full["K"], full["V"], 16, 24, 9, nh, prefix_look=L, after_look=L)
    np.testing.assert_array_equal(wide["O"], nocache["O"])
    np.testing.assert_array_equal(wide["K"], nocache["K"])
    vic = O.vicinity_step(X1, Wq, Wk, Wv, full["K"], full["V"], 16, 24, 9, nh, prefix_look=4, after_look=4)
    assert (vic["lo"], vic["hi"]) == (12, 28)
    np.testing.assert_array_equal(vic["K"][:12], full["K"][:12])             # stale outside the region
    np.testing.assert_array_equal(vic["V"][28:], full["V"][28:])
    np.testing.assert_array_equal(vic["K"][12:28], nocache["K"][12:28])      # fresh inside
    # queries are the region's rows; they differ from the no-cache forward through the stale keys only
    assert vic["O"].shape == (16, H)
    assert np.abs(vic["O"] - nocache["O"][12:28]).max() > 1e-6
    np.testing.assert_array_equal(vic["K"][35:40], full["K"][35:40])
    np.testing.assert_array_equal(O.attention(O.round_bf16(X1[12:28] @ Wq.T), vic["K"], vic["V"], nh), vic["O"])
