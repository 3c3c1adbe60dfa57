"""Pins for the oracle's blockwise generation loop (Alg. 1, PAPER.md:76-103;
schedules P:281-285, block-scoped credit P:327, EOS early termination P:174;
readings c11, c12, c21-c23 in DESIGN.md).  Run with -m "not gpu".

Each test pins the loop against a property the paper (or the arithmetic)
fixes: the sequential-degeneration and saturated-confidence forward counts,
the EOS fill of the remaining blocks, agreement of the early-terminated run
with the full run before the first EOS, schedule values, and the credit reset.
"""
import numpy as np

import oracle as O
from paper_2510_08666_b200 import synth

V, H, S = 1024, 256, 32
MASK, EOS = synth.mask_id(V), synth.eos_id(V)


def _weights():
    W = synth.make_W(V, H, 1)
    return O.bf16_bits_to_f64(W), W


def _saturated(W_u16, tgt, amp=40.0):
    """Hidden rows planted so p* ~ 1 on token tgt (|logit gap| >> ln V)."""
    w = synth.bf16_to_f32(W_u16[tgt]).astype(np.float64)
    h = amp * w / (w ** 2).sum(axis=-1, keepdims=True)
    return O.bf16_bits_to_f64(synth.bf16_round(h.astype(np.float32)))


def _X0(B, prompt_len, nblocks, seed=0):
    rng = np.random.default_rng(seed)
    X = np.full((B, prompt_len + nblocks * S), MASK, dtype=np.int64)
    X[:, :prompt_len] = rng.integers(0, V - 2, size=(B, prompt_len))
    return X


def test_sequential_degeneration_one_commit_per_step():
    """tau = 1 under strict '>' (c1) never clears: the fallback commits exactly
    one position per row per step, so F = gen_len (SPEC S:444 lower bound)."""
    W64, W = _weights()
    B, P, nb = 2, 3, 2
    rng = np.random.default_rng(1)
    tgt = rng.integers(0, V - 2, size=(B, S))
    cfg = O.GenConfig(prompt_len=P, S=S, mask_id=MASK, eos_id=EOS, tau_target=1.0)
    out = O.generate(lambda n, st: _saturated(W, tgt, amp=8.0 + 0.1 * n), W64, None, None,
                     _X0(B, P, nb), cfg, O.Params(decoder=O.DEC_THRESHOLD, tau=1.0))
    assert out["F"] == nb * S
    assert not (out["X"] == MASK).any()


def test_saturated_confidence_one_forward_per_block():
    """All positions far above tau commit at once: F = number of blocks, and
    the committed ids are the planted targets."""
    W64, W = _weights()
    B, P, nb = 2, 5, 3
    rng = np.random.default_rng(2)
    tgts = rng.integers(0, V - 2, size=(nb, B, S))
    cfg = O.GenConfig(prompt_len=P, S=S, mask_id=MASK, eos_id=EOS, tau_target=0.9)
    X0 = _X0(B, P, nb)
    out = O.generate(lambda n, st: _saturated(W, tgts[n]), W64, None, None, X0, cfg,
                     O.Params(decoder=O.DEC_THRESHOLD, tau=0.9))
    assert out["F"] == nb
    assert np.array_equal(out["X"][:, :P], X0[:, :P])            # prompt untouched
    for k in range(nb):
        assert np.array_equal(out["X"][:, P + k * S:P + (k + 1) * S], tgts[k])
    assert np.array_equal(out["T"], [nb * S] * B)


def _eos_run(early, B=1):
    W64, W = _weights()
    P, nb = 4, 4
    rng = np.random.default_rng(3)
    tgts = rng.integers(0, V - 2, size=(nb, B, S))
    tgts[1, 0, 7] = EOS                      # row 0 emits EOS in block 1 at offset 7
    cfg = O.GenConfig(prompt_len=P, S=S, mask_id=MASK, eos_id=EOS, tau_target=0.9,
                      early_termination=early)
    out = O.generate(lambda n, st: _saturated(W, tgts[min(n, nb - 1)]), W64, None, None,
                     _X0(B, P, nb), cfg, O.Params(decoder=O.DEC_THRESHOLD, tau=0.9))
    return out, P, nb


def test_early_termination_fills_remaining_blocks_with_eos():
    """once EOS is generated in a block, the loop halts after it and
    every later block is EOS; the EOS block itself is decoded (reading c22).
    T = tokens before the first EOS."""
    out, P, nb = _eos_run(True)
    X = out["X"][0]
    assert out["F"] == 2
    assert (X[P + 2 * S:] == EOS).all()
    assert X[P + S + 7] == EOS and (X[P + S:P + 2 * S] != MASK).all()
    assert out["T"][0] == S + 7


def test_early_termination_agrees_with_full_run_before_eos():
    """SPEC invariant: outputs with and without early termination agree on
    positions up to the first EOS; early termination never runs more forwards."""
    on, P, nb = _eos_run(True)
    off, _, _ = _eos_run(False)
    first = P + on["T"][0]
    assert np.array_equal(on["X"][0, :first + 1], off["X"][0, :first + 1])
    assert off["F"] == nb and on["F"] < off["F"]
    assert on["T"][0] == off["T"][0]


def test_early_termination_waits_for_every_row():
    """Rows step in lockstep (c21): the loop halts only when every row has
    emitted EOS; a finished row's later blocks are EOS-filled no-ops."""
    out, P, nb = _eos_run(True, B=2)
    assert out["F"] == nb                    # row 1 never emits EOS
    assert (out["X"][0, P + 2 * S:] == EOS).all()
    assert out["T"][1] == nb * S and out["T"][0] == S + 7


def test_iteration_params_schedules():
    """tau_t decays linearly from 1.0 to the target over decay_steps (c11) and
    drives theta_hi for the hierarchical decoder (theta_lo fixed); alpha_t =
    min(init + growth t, preset)."""
    cfg = O.GenConfig(prompt_len=0, S=S, mask_id=MASK, eos_id=EOS, tau_target=0.8, tau_decay_steps=4,
                      alpha_init=0.1, alpha_growth=0.05, alpha_preset=0.3)
    thr = O.Params(decoder=O.DEC_THRESHOLD, use_smooth=True)
    assert [round(O.iteration_params(thr, cfg, t).tau, 12) for t in range(6)] == [1.0, 0.95, 0.9, 0.85, 0.8, 0.8]
    assert [round(O.iteration_params(thr, cfg, t).alpha_t, 12) for t in (0, 1, 4, 10)] == [0.1, 0.15, 0.3, 0.3]
    hier = O.Params(decoder=O.DEC_HIERARCHICAL, theta_lo=0.62)
    p2 = O.iteration_params(hier, cfg, 2)
    assert abs(p2.theta_hi - 0.9) < 1e-12 and p2.theta_lo == 0.62


def test_credit_table_resets_at_every_block():
    """Credits are block-scoped: the first iteration of every block
    starts from C = 0, and the table carries within a block."""
    W64, W = _weights()
    B, P, nb = 1, 2, 2
    E = synth.make_E(V, H, 2)
    E64 = O.bf16_bits_to_f64(E)
    sch = [synth.PlantedSchedule(B * S, V, H, seed=10 + k) for k in range(nb)]
    hid = {}

    def hidden_of(n, st):
        if n not in hid:
            k = 0 if n < 3 else 1
            tgt, a = sch[k].targets_and_amplitudes(n)
            hid[n] = O.bf16_bits_to_f64(sch[k].hidden(W[tgt], a)).reshape(B, S, H)
        return hid[n]

    trace = []
    cfg = O.GenConfig(prompt_len=P, S=S, mask_id=MASK, eos_id=EOS, tau_target=0.9)
    O.generate(hidden_of, W64, E64, E64[MASK], _X0(B, P, nb), cfg,
               O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True), trace=trace)
    firsts = [i for i, r in enumerate(trace) if r["t"] == 0]
    assert [trace[i]["block"] for i in firsts] == list(range(nb))
    for i in firsts:
        assert not trace[i]["C"].any()
    assert any(r["C"].any() for r in trace if r["t"] > 0)


def _stable_suite_tpf(base, seeds, nb=2, P=3):
    """Mean TPF (T_i / F_i averaged over the suite) of the oracle's
    generate() on a scripted stable suite: every position keeps ONE target for
    the whole block (no flips) and its planted top logit rises monotonically,
    ramp 1.0 per iteration plus a U(0,1) jitter, from below the threshold
    (a0 ~ U[ln V - 3, ln V + 1], onset 0)."""
    W64, W = _weights()
    tpf = []
    for seed in seeds:
        sch = {}

        def hidden_of(n, st):
            k, t = st["block"], st["t"]
            if k not in sch:
                sch[k] = synth.PlantedSchedule(S, V, H, seed * 100 + k, ramp=1.0, flip_prob=0.0, onset_max=0)
            tgt, a = sch[k].targets_and_amplitudes(t)
            return O.bf16_bits_to_f64(sch[k].hidden(W[tgt], a)).reshape(1, S, H)

        cfg = O.GenConfig(prompt_len=P, S=S, mask_id=MASK, eos_id=EOS, tau_target=0.9, early_termination=False)
        out = O.generate(hidden_of, W64, None, None, _X0(1, P, nb, seed), cfg, base)
        T, F = int(out["T"][0]), out["F"]
        assert 1.0 <= T / F <= S                     # SPEC invariant: TPF in [1, S]
        tpf.append(T / F)
    return float(np.mean(tpf)), tpf


def test_credit_mean_tpf_exceeds_threshold_on_stable_suite():
    """SPEC S:542 (directional): on a suite whose under-threshold tokens are
    stable and whose confidences rise monotonically, credit decoding (P:306-327,
    the credit accumulated on the stable argmax raises its fused confidence)
    commits earlier than plain threshold decoding at the same tau, so its mean
    TPF is strictly higher; both decode the same targets."""
    seeds = range(6)
    thr, thr_each = _stable_suite_tpf(O.Params(decoder=O.DEC_THRESHOLD, tau=0.9), seeds)
    cred, cred_each = _stable_suite_tpf(O.Params(decoder=O.DEC_THRESHOLD, tau=0.9, use_credit=True), seeds)
    assert cred > thr, (cred_each, thr_each)
    assert all(c >= t for c, t in zip(cred_each, thr_each)), (cred_each, thr_each)
