"""Vetted multi-iteration trajectories for parity tests (test infrastructure).

The planted hidden states come from paper_2510_08666_b200.synth (no method
arithmetic); this helper then runs the ORACLE on the carried state and
re-draws any position that sits within 1e-3 of a decision boundary
(reading c19):
  * raw top-2 margin  p*(1) - p*(2) > 1e-3        (v* feeds the credit update)
  * fused top-2 margin p~(1) - p~(2) > 1e-3      (v~ is the committed id)
  * |p~ - threshold| > 1e-3 for every active threshold
  * |p~_s - p~_t| > 1e-3 among undecided positions with p~ <= the primary
    threshold (only those can compete in a fallback / run maximum).
Golden outputs are the oracle's; nothing here comes from the CUDA path.
"""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2510_08666_b200 import synth

MARGIN = 1e-3


def _offenders(f, res, C_after, mask_before, params: O.Params):
    """Return the set of flat positions (b*S+s) violating a margin."""
    B, S = mask_before.shape
    bad = set()
    for b in range(B):
        und = mask_before[b]
        if not und.any():
            continue
        fb = f[b]
        ft = O.credit_fuse(fb, C_after[b], params.c_alpha) if params.use_credit else fb
        pt = res["ptilde"][b]
        if params.decoder == O.DEC_THRESHOLD:
            thr, primary = [params.tau], params.tau
        else:
            thr, primary = [params.theta_hi, params.theta_lo], params.theta_hi
        for s in np.nonzero(und)[0]:
            for row in ((fb[s], ft[s]) if params.use_credit else (fb[s],)):
                top2 = np.partition(row, -2)[-2:]
                lse = row.max() + np.log(np.exp(row - row.max()).sum())
                if np.exp(top2[1] - lse) - np.exp(top2[0] - lse) <= MARGIN:
                    bad.add(b * S + s)
            if any(abs(pt[s] - t) <= MARGIN for t in thr):
                bad.add(b * S + s)
        low = [s for s in np.nonzero(und)[0] if pt[s] <= primary + MARGIN]
        for i, s in enumerate(low):
            for t in low[i + 1:]:
                if abs(pt[s] - pt[t]) <= MARGIN:
                    bad.add(b * S + t)
    return bad


def vetted_trajectory(W_u16, E_u16, B, S, seed, params_fn, max_iters=None,
                      use_credit_table=False, ramp=2.5, flip_prob=0.2, max_rounds=400):
    """Run a block from fully masked until done (or max_iters); returns
    (W64, E64, e_mask64, steps) where steps[t] = dict(h=u16 [B,S,H], params,
    state_before (mask, tokens, C), result (oracle))."""
    V, H = W_u16.shape
    M = B * S
    W64 = O.bf16_bits_to_f64(W_u16)
    E64 = O.bf16_bits_to_f64(E_u16)
    em64 = E64[synth.mask_id(V)] if E64.shape[0] == V else E64[0]  # e_mask only used with smoothing
    sch = synth.PlantedSchedule(M, V, H, seed, ramp=ramp, flip_prob=flip_prob)
    mask = np.ones((B, S), bool)
    tokens = np.full((B, S), synth.mask_id(V), dtype=np.int64)
    C = np.zeros((B, S, V)) if use_credit_table else None
    steps = []
    t = 0
    while mask.any() and (max_iters is None or t < max_iters):
        params = params_fn(t)
        tgt, a = sch.targets_and_amplitudes(t)
        h = sch.hidden(W_u16[tgt], a).reshape(B, S, H)
        redraws = np.zeros(M, dtype=int)
        for _round in range(max_rounds):
            h64 = O.bf16_bits_to_f64(h)
            f = np.stack([O.logits(h64[b], W64) for b in range(B)])
            res = O.step(h64, W64, E64, em64, mask, tokens, C, params, f=f)
            bad = _offenders(f, res, res["C"] if params.use_credit else None, mask, params)
            if not bad:
                break
            rows = np.array(sorted(bad))
            redraws[rows] += 1
            base = rows[redraws[rows] % 25 == 0]
            if len(base):
                sch.redraw_base(base)
                a[base] = sch.a0[base] + sch.ramp * np.maximum(0, t - sch.onset[base]) + 0.5
            hf = h.reshape(M, H)
            hf[rows] = sch.hidden(W_u16[tgt[rows]], a[rows])
            h = hf.reshape(B, S, H)
        else:
            raise RuntimeError("vetting did not converge")
        steps.append(dict(h=h.copy(), params=params,
                          mask=mask.copy(), tokens=tokens.copy(),
                          C=None if C is None else C.copy(), result=res))
        mask, tokens = res["mask"], res["tokens"]
        if params.use_credit:
            C = res["C"]
        t += 1
    return W64, E64, em64, steps


def vetted_generation(W_u16, E_u16, B, S, nblocks, prompt_len, seed, base: O.Params, cfg: O.GenConfig,
                      eos_at=(), ramp=2.5, flip_prob=0.1, max_rounds=400, onset_max=5):
    """A whole blockwise generation (Alg. 1) driven by planted hidden states,
    every iteration vetted against the decision margins (c19) on the oracle's
    carried state.  Block k draws from PlantedSchedule(seed*100 + k); eos_at =
    [(row, block, offset)] plants eos_id as that position's target.
    Returns (hidden [F, B*S, H] u16, X0 [B, L], oracle result)."""
    V, H = W_u16.shape
    M = B * S
    W64 = O.bf16_bits_to_f64(W_u16)
    E64 = O.bf16_bits_to_f64(E_u16)
    em64 = E64[cfg.mask_id]
    rng = np.random.default_rng(np.random.SeedSequence([seed, 4242]))
    L = prompt_len + nblocks * S
    X0 = np.full((B, L), cfg.mask_id, dtype=np.int64)
    X0[:, :prompt_len] = rng.integers(0, V - 2, size=(B, prompt_len))
    schedules = {}
    hidden = []

    def hidden_of(n, st):
        k, t = st["block"], st["t"]
        if k not in schedules:
            sch = synth.PlantedSchedule(M, V, H, seed * 100 + k, ramp=ramp, flip_prob=flip_prob,
                                        onset_max=onset_max)
            for (r, blk, off) in eos_at:
                if blk == k:
                    sch.tgt[r * S + off] = cfg.eos_id
            schedules[k] = sch
        sch = schedules[k]
        p, mask, tokens, C = st["params"], st["mask"], st["tokens"], st["C"]
        tgt, a = sch.targets_and_amplitudes(t)
        h = sch.hidden(W_u16[tgt], a).reshape(B, S, H)
        redraws = np.zeros(M, dtype=int)
        for _round in range(max_rounds):
            h64 = O.bf16_bits_to_f64(h)
            f = np.stack([O.logits(h64[b], W64) for b in range(B)])
            res = O.step(h64, W64, E64, em64, mask, tokens, C, p, f=f)
            bad = _offenders(f, res, res["C"] if p.use_credit else None, mask, p)
            if not bad:
                break
            rows = np.array(sorted(bad))
            redraws[rows] += 1
            base_rows = rows[redraws[rows] % 25 == 0]
            if len(base_rows):
                sch.redraw_base(base_rows)
                a[base_rows] = sch.a0[base_rows] + sch.ramp * np.maximum(0, t - sch.onset[base_rows]) + 0.5
            hf = h.reshape(M, H)
            hf[rows] = sch.hidden(W_u16[tgt[rows]], a[rows])
            h = hf.reshape(B, S, H)
        else:
            raise RuntimeError("vetting did not converge")
        assert n == len(hidden)
        hidden.append(h.reshape(M, H).copy())
        return O.bf16_bits_to_f64(h)

    out = O.generate(hidden_of, W64, E64, em64, X0, cfg, base)
    return np.stack(hidden), X0, out
