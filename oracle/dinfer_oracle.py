"""CPU ORACLE for dInfer's denoise-and-commit step (arXiv 2510.08666).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2510_08666_b200``) never imports it and has
no CPU fallback.  This module shares no code with the CUDA path: it decodes
bf16 itself, it imports nothing from the package, and the package imports
nothing from here.

What it is: the plain definition of one iteration of the inner ``while`` loop
of Algorithm 1 restricted to the decode side: given the
block's hidden states, it forms the logits, the decoder's credit
update / fuse (App. B.2), the threshold or hierarchical
(App. B.1) commit rule, the commit, and iteration
smoothing (App. A.1).  Everything is float64 numpy on inputs that
are already bf16-rounded (bf16 -> float64 is exact), written in the paper's
order and notation.  A library primitive (matmul, argmax, exp, log) is used
as a step; there is no blocking, fusion or reordering.

Readings of silent / ambiguous passages are the SURVEY.md §8(c) readings
c1..c20 plus c21..c27 for the §8(f) rows, restated in DESIGN.md "Readings";
each function names the ones it takes.

Beyond the step: the blockwise generation loop of Alg. 1
(`generate`, f1), the next iteration's model input (`next_input_embedding`,
f2), the vicinity KV-cache refresh on a synthetic attention layer
(`refresh_region`, `vicinity_step`, `attention`, f3) and the credit-fused
smoothing variant (`smooth_credit_fused`, f4).

Parity pins: every function is pinned by tests under ``tests/`` (marked
"not gpu") against worked examples, closed forms, brute force and
invariants.  Parity unpinned: whether the
hierarchical run rule (reading c8) is the paper's exact rule (the paper gives
no worked example), the concrete beta/gamma/alpha values (c6), and raw-vs-
fused p for smoothing (c13) -- these are readings, not derivations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEC_THRESHOLD = 0
DEC_HIERARCHICAL = 1


# ---------------------------------------------------------------------------
# bf16 decoding (own copy; the oracle shares no helper with the CUDA path)
# ---------------------------------------------------------------------------
def bf16_bits_to_f64(u16: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> exact float64 values."""
    u32 = np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u32.view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# Step 1. logits  (Alg. 1 line "logits <- M.Forward"; W_out is the
# LM head, not tied to W_emb)
# ---------------------------------------------------------------------------
def logits(h: np.ndarray, W: np.ndarray) -> np.ndarray:
    """f[s, v] = sum_k h[s, k] * W[v, k]   (h: [M, H], W: [V, H]) -> [M, V]."""
    return np.asarray(h, np.float64) @ np.asarray(W, np.float64).T


# ---------------------------------------------------------------------------
# Step 2. softmax statistics  (p = Softmax(f), v* = argmax_v p)
# ---------------------------------------------------------------------------
def softmax_stats(f: np.ndarray):
    """Per row: m = max_v f, v* = lowest argmax (reading c3), lse = log sum exp f,
    p* = softmax(f)[v*] = exp(f[v*] - lse).   Returns (m, vstar, lse, pstar)."""
    f = np.asarray(f, np.float64)
    m = f.max(axis=1)
    vstar = f.argmax(axis=1)                       # first occurrence = lowest id
    lse = m + np.log(np.exp(f - m[:, None]).sum(axis=1))
    pstar = np.exp(f[np.arange(f.shape[0]), vstar] - lse)
    return m, vstar.astype(np.int64), lse, pstar


def softmax(f: np.ndarray) -> np.ndarray:
    """p = Softmax(f) row-wise, temperature 1 ("without temperature scaling")."""
    f = np.asarray(f, np.float64)
    e = np.exp(f - f.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


# ---------------------------------------------------------------------------
# Step 3a. credit update, Eq. (credit-update-top1)
#   C_t[i, v] = beta * C_{t-1}[i, v] + p(v)^gamma   if v = v*
#             = beta * C_{t-1}[i, v]                otherwise
# applied to undecided positions only (reading c7); p and v* are the RAW
# model distribution's (reading c4).
# ---------------------------------------------------------------------------
def credit_update(C: np.ndarray, vstar: np.ndarray, pstar: np.ndarray,
                  undecided: np.ndarray, beta: float, gamma: float) -> np.ndarray:
    C = np.array(C, dtype=np.float64, copy=True)
    for i in range(C.shape[0]):
        if not undecided[i]:
            continue                      # decided rows are frozen (c7)
        C[i, :] = beta * C[i, :]
        C[i, vstar[i]] += pstar[i] ** gamma
    return C


# ---------------------------------------------------------------------------
# Step 3b. credit fuse, Eq. (logits-fuse)
#   f~[i, v] = f[i, v] + alpha * log(1 + C_t[i, v])
# then p~ = Softmax(f~) replaces p; the committed id is argmax f~ (c5).
# ---------------------------------------------------------------------------
def credit_fuse(f: np.ndarray, C: np.ndarray, alpha: float) -> np.ndarray:
    return np.asarray(f, np.float64) + alpha * np.log1p(np.asarray(C, np.float64))


def confidence(ftilde: np.ndarray):
    """(v~, p~, lse~): argmax of the (fused) logits (lowest id on ties) and its
    softmax probability."""
    m, v, lse, p = softmax_stats(ftilde)
    return v, p, lse


# ---------------------------------------------------------------------------
# Step 4a. threshold decoding (Fast-dLLM), "commits tokens whose
# confidence exceeds a preset threshold".  Reading c1: strict '>'.
# Reading c2: if nothing clears, commit the undecided position with the
# highest confidence (lowest index on ties).
# ---------------------------------------------------------------------------
def _clears(p, thr, inclusive: bool) -> bool:
    """Reading c1: "exceeds" is strict '>'; the SPEC's inclusive
    '>=' is the `inclusive` variant (DESIGN.md c1')."""
    return p >= thr if inclusive else p > thr


def threshold_decode(ptilde, undecided, tau: float, inclusive: bool = False) -> np.ndarray:
    S = len(undecided)
    A = np.zeros(S, dtype=bool)
    for s in range(S):
        if undecided[s] and _clears(ptilde[s], tau, inclusive):
            A[s] = True
    if not A.any():
        best = _fallback_argmax(ptilde, undecided)
        if best is not None:
            A[best] = True
    return A


def _fallback_argmax(ptilde, undecided):
    best = None
    for s in range(len(undecided)):
        if undecided[s] and (best is None or ptilde[s] > ptilde[best]):
            best = s                                # strict: lowest s on ties
    return best


def undecided_runs(undecided):
    """Maximal runs [first, last] of consecutive undecided positions."""
    runs, s, S = [], 0, len(undecided)
    while s < S:
        if undecided[s]:
            first = s
            while s + 1 < S and undecided[s + 1]:
                s += 1
            runs.append((first, s))
        s += 1
    return runs


# ---------------------------------------------------------------------------
# Step 4b. hierarchical decoding, P:119 and App. B.1 P:293-299.
#   "recursively partitions masked spans into smaller sub-regions ...
#    attempting to resolve at least one token in each region during every
#    forward pass whenever confidence permits"; positions near the
#   centre of each span are preferred.  Hyper-parameters: decoding
#   threshold 0.92, lower boundary 0.62.
# Readings c8/c9/c10: (a) commit every undecided s with p~ > theta_hi;
# (b) sub-regions = maximal runs of undecided positions at step start
#     (runs_after_hi=True: runs of the positions still undecided after (a),
#     variant A'); a run with no commit from (a) commits its max-p~ position
#     (ties: nearest the run centre, then lower index) if p~ > theta_lo;
# (c) nothing committed at all -> global argmax fallback (c2).
# The recursion happens across iterations: every commit splits its run.
# ---------------------------------------------------------------------------
def hierarchical_decode(ptilde, undecided, theta_hi: float, theta_lo: float,
                        runs_after_hi: bool = False, inclusive: bool = False) -> np.ndarray:
    S = len(undecided)
    A = np.zeros(S, dtype=bool)
    for s in range(S):                                            # (a)
        if undecided[s] and _clears(ptilde[s], theta_hi, inclusive):
            A[s] = True
    region_mask = [bool(undecided[s]) and not (runs_after_hi and A[s]) for s in range(S)]
    for first, last in undecided_runs(region_mask):               # (b)
        if any(A[first:last + 1]):
            continue
        best = None
        for s in range(first, last + 1):
            if best is None or _hier_better(s, best, ptilde, first, last):
                best = s
        if _clears(ptilde[best], theta_lo, inclusive):
            A[best] = True
    if not A.any():                                               # (c)
        best = _fallback_argmax(ptilde, undecided)
        if best is not None:
            A[best] = True
    return A


def _hier_better(s, t, ptilde, first, last) -> bool:
    """Is position s preferred over t inside run [first, last]?  Higher p~;
    then nearer the centre (first+last)/2 (compared as |2s-first-last|);
    then lower index."""
    if ptilde[s] != ptilde[t]:
        return ptilde[s] > ptilde[t]
    ds, dt = abs(2 * s - first - last), abs(2 * t - first - last)
    if ds != dt:
        return ds < dt
    return s < t


# ---------------------------------------------------------------------------
# Step 6. iteration smoothing, App. A.1
#   p_t[i] = softmax(z_t[i]); Delta e_t[i] = p_t[i] W_emb;
#   e_{t+1}[i] = e_mask + alpha_t * Delta e_t[i]   (masked positions only)
# Reading c13: raw softmax; c14: rows still undecided after this step's commit.
# ---------------------------------------------------------------------------
def smooth(f_rows: np.ndarray, E: np.ndarray, e_mask: np.ndarray, alpha_t: float) -> np.ndarray:
    p = softmax(f_rows)
    delta_e = p @ np.asarray(E, np.float64)
    return np.asarray(e_mask, np.float64)[None, :] + alpha_t * delta_e


# ---------------------------------------------------------------------------
# Credit-fused smoothing variant (the alternative of
# reading c13): the expected embedding under the distribution the decoder
# actually decides on, p~ = softmax(f~) with f~ = f + alpha * ln(1 + C)
# (Eq. logits-fuse), instead of the raw softmax(z) of P:278.
#   e_{t+1} = e_mask + alpha_t * softmax(f + c_alpha ln(1 + C)) W_emb
# C is the credit table after this iteration's update (the one the decision
# used).  c_alpha = 0 or C = 0 reduce it to smooth().
# ---------------------------------------------------------------------------
def smooth_credit_fused(f_rows: np.ndarray, C_rows: np.ndarray, E: np.ndarray, e_mask: np.ndarray,
                        alpha_t: float, c_alpha: float) -> np.ndarray:
    return smooth(credit_fuse(f_rows, C_rows, c_alpha), E, e_mask, alpha_t)


# ---------------------------------------------------------------------------
# Next iteration's model input (Fig. 3 / P:152):
# the embedding the model reads at iteration t+1 for each position of the
# block.  Decided positions feed their token's row of the input embedding
# W_emb (the ordinary lookup); positions still masked feed e_{t+1}, the
# smoothed embedding -- "iteration smoothing ... only on masked positions"
# (P:275), "retains logit-weighted embeddings" for the next iteration.
# Reading c24: without smoothing a masked position would feed e_mask; this
# output is defined for smoothing steps only (the CUDA path requires it).
# ---------------------------------------------------------------------------
def next_input_embedding(E: np.ndarray, tokens: np.ndarray, mask: np.ndarray,
                         smoothed: np.ndarray) -> np.ndarray:
    """tokens, mask: [B, S] after this step's commit; smoothed: [B, S, H]
    (e_{t+1}, valid where mask).  Returns [B, S, H] float64."""
    E = np.asarray(E, np.float64)
    B, S = tokens.shape
    out = np.empty((B, S, E.shape[1]))
    for b in range(B):
        for s in range(S):
            out[b, s] = smoothed[b, s] if mask[b, s] else E[tokens[b, s]]
    return out


def alpha_schedule(alpha_init: float, alpha_growth: float, alpha_preset: float, t: int) -> float:
    """alpha_t = min(alpha_init + alpha_growth * t, alpha_preset)."""
    return min(alpha_init + alpha_growth * t, alpha_preset)


def tau_schedule(target: float, t: int, decay_steps: int) -> float:
    """Decode threshold decaying from 1.0 toward `target`; reading c11:
    linear over `decay_steps` iterations of the block, constant afterwards."""
    if decay_steps <= 0:
        return target
    frac = min(t, decay_steps) / decay_steps
    return 1.0 - (1.0 - target) * frac


# ---------------------------------------------------------------------------
# The whole step (one iteration of Alg. 1's inner loop, decode side)
# ---------------------------------------------------------------------------
@dataclass
class Params:
    decoder: int = DEC_THRESHOLD
    tau: float = 0.9
    theta_hi: float = 0.92
    theta_lo: float = 0.62
    use_credit: bool = False
    c_alpha: float = 1.0
    c_beta: float = 0.9
    c_gamma: float = 0.5
    use_smooth: bool = False
    alpha_t: float = 0.1
    hier_runs_after_hi: bool = False
    smooth_credit_fused: bool = False   # f4: smooth with softmax(f~) instead of softmax(f)
    inclusive: bool = False             # c1': thresholds compare '>=' instead of '>'


def step(h, W, E, e_mask, mask, tokens, C, params: Params, f=None):
    """One denoise-and-commit iteration for B batch rows of a block of S.

    h: [B, S, H] float64 (bf16 values); W, E: [V, H]; e_mask: [H];
    mask: [B, S] bool (True = undecided); tokens: [B, S] int;
    C: [B, S, V] dense credit table or None (credit off);
    f (optional): precomputed logits [B, S, V] (reused by shard tests).
    Returns dict with new tokens / mask / C, committed, stats and smoothed
    (NaN rows where no smoothed embedding is produced).
    Order: credit update -> credit fuse -> decode -> commit ->
    smoothing capture.
    """
    B, S, H = h.shape
    tokens = np.array(tokens, copy=True)
    mask = np.array(mask, dtype=bool, copy=True)
    C_new = None if C is None else np.array(C, dtype=np.float64, copy=True)
    committed = np.zeros((B, S), dtype=bool)
    out_m = np.zeros((B, S)); out_lse = np.zeros((B, S))
    out_pt = np.zeros((B, S)); out_vt = np.zeros((B, S), dtype=np.int64)
    out_vstar = np.zeros((B, S), dtype=np.int64); out_pstar = np.zeros((B, S))
    smoothed = np.full((B, S, H), np.nan)
    for b in range(B):
        fb = logits(h[b], W) if f is None else np.asarray(f[b], np.float64)
        m, vstar, lse, pstar = softmax_stats(fb)
        und = mask[b].copy()
        if params.use_credit:
            C_new[b] = credit_update(C_new[b], vstar, pstar, und, params.c_beta, params.c_gamma)
            vt, pt, _ = confidence(credit_fuse(fb, C_new[b], params.c_alpha))
        else:
            vt, pt = vstar, pstar
        if not und.any():
            A = np.zeros(S, dtype=bool)           # empty row: defined no-op (§8b)
        elif params.decoder == DEC_THRESHOLD:
            A = threshold_decode(pt, und, params.tau, params.inclusive)
        else:
            A = hierarchical_decode(pt, und, params.theta_hi, params.theta_lo,
                                    params.hier_runs_after_hi, params.inclusive)
        for s in range(S):                         # commit
            if A[s]:
                tokens[b, s] = vt[s]
                mask[b, s] = False
        committed[b] = A
        out_m[b], out_lse[b], out_pt[b], out_vt[b] = m, lse, pt, vt
        out_vstar[b], out_pstar[b] = vstar, pstar
        if params.use_smooth:
            still = np.nonzero(mask[b])[0]
            if len(still):
                if params.smooth_credit_fused and params.use_credit:
                    smoothed[b, still] = smooth_credit_fused(fb[still], C_new[b][still], E, e_mask,
                                                             params.alpha_t, params.c_alpha)
                else:
                    smoothed[b, still] = smooth(fb[still], E, e_mask, params.alpha_t)
    return dict(tokens=tokens, mask=mask, C=C_new, committed=committed,
                m=out_m, lse=out_lse, ptilde=out_pt, vtilde=out_vt,
                vstar=out_vstar, pstar=out_pstar, smoothed=smoothed)


# ---------------------------------------------------------------------------
# Shard-merge mode (vocab split across G ranks).
# Each shard j reports (m_j, v*_j (global id), l_j = sum_{v in shard} e^{f-m_j},
# acc_j = sum_{v in shard} e^{f-m_j} E[v]); the merge is the exact identity
#   m = max_j m_j ; l = sum_j l_j e^{m_j - m} ; acc = sum_j acc_j e^{m_j - m};
#   v* = v*_j of the maximising shard (lowest id on ties).
# ---------------------------------------------------------------------------
def shard_record(f_shard: np.ndarray, v_offset: int, E_shard=None):
    f_shard = np.asarray(f_shard, np.float64)
    m = f_shard.max(axis=1)
    v = f_shard.argmax(axis=1) + v_offset
    w = np.exp(f_shard - m[:, None])
    l = w.sum(axis=1)
    acc = None if E_shard is None else w @ np.asarray(E_shard, np.float64)
    return dict(m=m, vstar=v, l=l, acc=acc)


def merge_records(records):
    m = np.max(np.stack([r["m"] for r in records]), axis=0)
    l = np.zeros_like(m)
    vstar = np.full(m.shape, np.iinfo(np.int64).max, dtype=np.int64)
    acc = None
    for r in records:                                  # fixed shard order
        scale = np.exp(r["m"] - m)
        l = l + r["l"] * scale
        hit = r["m"] == m
        vstar = np.where(hit, np.minimum(vstar, r["vstar"]), vstar)
        if r["acc"] is not None:
            acc = (0 if acc is None else acc) + r["acc"] * scale[:, None]
    lse = m + np.log(l)
    return dict(m=m, vstar=vstar, l=l, lse=lse, pstar=1.0 / l, acc=acc)


# ---------------------------------------------------------------------------
# The blockwise generation loop (Algorithm 1) around step(),
# with the schedules (App. A.1), per-block credit reset
# and EOS early termination.  SURVEY §8(f) row f1.
#
# Readings:
#   c11/c12  tau_t / alpha_t restart at t = 0 in every block; tau_t drives tau
#            (threshold) or theta_hi (hierarchical), theta_lo stays fixed.
#   c21      blocks are [prompt_len + k*S, prompt_len + (k+1)*S), left to
#            right; all B rows decode the same block in lockstep (a row with
#            no undecided position is a no-op, §8(b)); the block ends when no
#            row has an undecided position.  Positions of the generation
#            region that are not mask_id at block start count as decided.
#   c22      early termination: when row b's block contains eos_id after the
#            block completes, row b is finished -- every later block of row b
#            is filled with eos_id ("fills all remaining blocks with
#            EOS"); the block in which EOS appeared is decoded to completion
#            (P:174 makes the *remaining blocks* redundant, not the current
#            one).  The loop halts when every row is finished or the blocks
#            run out.
#   c23      T_b = number of generated tokens before the first eos_id of row
#            b, gen_len if none; F = number of forwards (iterations)
#            the loop ran -- shared by the B rows, which step in lockstep.
#   The model forward is outside the method's hot path: iteration n (global,
#   0-based) uses the hidden block hidden_of(n) supplied by the caller.
# ---------------------------------------------------------------------------
@dataclass
class GenConfig:
    prompt_len: int
    S: int
    mask_id: int
    eos_id: int
    early_termination: bool = True
    tau_target: float = 0.9      # decays from 1.0, reading c11
    tau_decay_steps: int = 0     # 0 = constant tau_target
    alpha_init: float = 0.1      # alpha_t = min(init + growth*t, preset)
    alpha_growth: float = 0.05
    alpha_preset: float = 0.3
    max_forwards: int = 1 << 30


def iteration_params(base: Params, cfg: GenConfig, t: int) -> Params:
    """The step parameters of block-local iteration t (schedules, c11/c12)."""
    p = Params(**vars(base))
    thr = tau_schedule(cfg.tau_target, t, cfg.tau_decay_steps)
    if p.decoder == DEC_THRESHOLD:
        p.tau = thr
    else:
        p.theta_hi = thr
    if p.use_smooth:
        p.alpha_t = alpha_schedule(cfg.alpha_init, cfg.alpha_growth, cfg.alpha_preset, t)
    return p


def generate(hidden_of, W, E, e_mask, X0, cfg: GenConfig, base: Params, dense_credit=True, trace=None):
    """Run Algorithm 1's block loop on token rows X0 [B, L].

    hidden_of(n, state) -> [B, S, H] float64 hidden states of global
    iteration n (the model stand-in); state = dict(block, t, tokens, mask, C,
    params) before the step.  Returns dict(X, F, T, truncated).  `trace`,
    when a list, receives per-iteration dicts (block, t, params, state
    before, step result)."""
    X = np.array(X0, dtype=np.int64, copy=True)
    B, L = X.shape
    S, P = cfg.S, cfg.prompt_len
    gen_len = L - P
    assert gen_len > 0 and gen_len % S == 0
    V = W.shape[0]
    nblocks = gen_len // S
    done = np.zeros(B, dtype=bool)
    F = 0
    truncated = False
    for k in range(nblocks):
        lo, hi = P + k * S, P + (k + 1) * S
        tokens = X[:, lo:hi].copy()
        for b in range(B):
            if done[b]:
                tokens[b][tokens[b] == cfg.mask_id] = cfg.eos_id     # c22: EOS fill
        mask = tokens == cfg.mask_id
        C = np.zeros((B, S, V)) if (base.use_credit and dense_credit) else None  # P:327 reset
        t = 0
        while mask.any():
            if F >= cfg.max_forwards:
                truncated = True
                break
            p = iteration_params(base, cfg, t)
            h = hidden_of(F, dict(block=k, t=t, tokens=tokens, mask=mask, C=C, params=p))
            res = step(h, W, E, e_mask, mask, tokens, C, p)
            if trace is not None:
                trace.append(dict(block=k, t=t, params=p, mask=mask.copy(), tokens=tokens.copy(),
                                  C=None if C is None else C.copy(), h=h, result=res))
            tokens, mask = res["tokens"], res["mask"]
            if C is not None:
                C = res["C"]
            F += 1
            t += 1
        X[:, lo:hi] = tokens
        if truncated:
            break
        if cfg.early_termination:
            done |= (tokens == cfg.eos_id).any(axis=1)
            if done.all():
                for b in range(B):                                   # c22: fill the rest
                    rest = X[b, hi:]
                    rest[rest == cfg.mask_id] = cfg.eos_id
                break
    T = np.full(B, gen_len, dtype=np.int64)
    for b in range(B):
        e = np.nonzero(X[b, P:] == cfg.eos_id)[0]
        if len(e):
            T[b] = e[0]
    return dict(X=X, F=F, T=T, truncated=truncated)


# ---------------------------------------------------------------------------
# Vicinity KV-cache refresh (§2.3, App. D
# P:368) on a synthetic single bidirectional attention layer -- the KV-cache
# manager of Algorithm 1 (K.ShouldUpdate / K.Update).
#
# Readings:
#   c25  refresh region: for block [start, end), iteration t of
#        the block: all positions [0, L) while t < warmup_times, else
#        [start - prefix_look, end + after_look) clipped to [0, L) (P:133
#        "recomputed for both masked tokens and their immediate neighbors";
#        looks 16, warmup 4).  The region is also the forward's query
#        region; positions outside it keep their cached K/V (stale).
#        A block's completion triggers a full refresh ("once a block is
#        fully decoded, a full cache update ensures global consistency").
#   c26  the layer: q = x Wq^T, k = x Wk^T, v = x Wv^T (nn.Linear layout
#        [out, in]); n_heads = H / d_head; per head o = softmax(q K^T /
#        sqrt(d_head)) V over all L cached positions (bidirectional: no mask).
#   c27  storage precision: q and the cached k, v are stored in bf16
#        (round to nearest even) as a bf16 model would; accumulation in fp64
#        here (fp32 on the GPU).
# ---------------------------------------------------------------------------
def refresh_region(L: int, start: int, end: int, t: int, prefix_look: int, after_look: int,
                   warmup_times: int, full: bool = False):
    """[lo, hi) of positions whose K/V (and queries) this forward recomputes."""
    if full or t < warmup_times:
        return 0, L
    return max(0, start - prefix_look), min(L, end + after_look)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """float64 -> nearest bf16 value (ties to even), returned as float64.
    bf16 keeps 8 significand bits: x = m 2^e with m in [0.5, 1) (frexp), so
    the bf16 value is round(m 2^8) 2^(e-8) (np.round ties to even).  Normal
    range only (the layer's values are far from bf16 under/overflow)."""
    m, e = np.frexp(np.asarray(x, np.float64))
    return np.round(m * 256.0) * np.exp2(e - 8.0)


def attention(Q: np.ndarray, K: np.ndarray, V: np.ndarray, n_heads: int) -> np.ndarray:
    """Bidirectional multi-head attention: Q [R, H], K, V [L, H] -> [R, H]."""
    R, H = Q.shape
    d = H // n_heads
    out = np.empty((R, H))
    for hh in range(n_heads):
        sl = slice(hh * d, (hh + 1) * d)
        s = Q[:, sl] @ K[:, sl].T / math.sqrt(d)
        out[:, sl] = softmax(s) @ V[:, sl]
    return out


def vicinity_step(X, Wq, Wk, Wv, Kc, Vc, start: int, end: int, t: int, n_heads: int,
                  prefix_look: int = 16, after_look: int = 16, warmup_times: int = 4, full: bool = False):
    """One forward of the attention layer under vicinity refresh.
    X: [L, H] layer input (all positions, this iteration); Kc, Vc: [L, H]
    cached keys / values (bf16 values as float64).  Returns dict(lo, hi, O
    [hi-lo, H] for the query rows lo..hi-1, K, V = updated caches)."""
    L = X.shape[0]
    lo, hi = refresh_region(L, start, end, t, prefix_look, after_look, warmup_times, full)
    X = np.asarray(X, np.float64)
    K = np.array(Kc, np.float64, copy=True)
    Vn = np.array(Vc, np.float64, copy=True)
    K[lo:hi] = round_bf16(X[lo:hi] @ np.asarray(Wk, np.float64).T)      # K.Update on the region
    Vn[lo:hi] = round_bf16(X[lo:hi] @ np.asarray(Wv, np.float64).T)
    Q = round_bf16(X[lo:hi] @ np.asarray(Wq, np.float64).T)
    return dict(lo=lo, hi=hi, O=attention(Q, K, Vn, n_heads), K=K, V=Vn)
