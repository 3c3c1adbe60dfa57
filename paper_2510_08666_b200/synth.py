"""Seeded synthetic inputs shared by the tests and bench.py.

This module holds NONE of the method's arithmetic: no logits, softmax,
credit, selection or smoothing.  It only draws random numbers, rounds them to
bf16 and plants hidden states.  Both the CUDA path (via bench/tests) and the
CPU oracle (via tests) consume its arrays; neither side imports the other.

Recipe (paper shapes from BASELINE.json configs):
  * W_vocab[V, H] = bf16(N(0, 1/H)),  E[V, H] = bf16(N(0, 1)); drawn in
    1024-row blocks, each from SeedSequence([seed, block]), so any vocab shard
    can be produced alone and identically on every rank.
  * mask_id = V-1 (e_mask = E[V-1]), eos = V-2: synthetic ids ("standard
    mask embedding"; the paper gives no ids).
  * hidden states are planted: h_s = a_s * W[tgt_s] / ||W[tgt_s]||^2 + n,
    n ~ N(0, (0.3/sqrt(H))^2), so that the top logit is ~a_s and the top
    probability is ~sigmoid(a_s - ln V).  Per position: target tgt ~ U[0, V-2),
    onset ~ U{0..5}, base a0 ~ U[ln V - 3, ln V + 1]; at iteration t
    a = a0 + ramp * max(0, t - onset) + U(0, 1), and with probability
    flip_prob the target is replaced for that one iteration by a random token.
"""
from __future__ import annotations

import math

import numpy as np

ROW_BLOCK = 1024


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern (uint16), round-to-nearest-even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    bias = np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    return ((u + bias) >> np.uint32(16)).astype(np.uint16)


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def _normal_rows(seed: int, row_begin: int, row_end: int, H: int, std: float) -> np.ndarray:
    """Rows [row_begin, row_end) of a [V, H] N(0, std^2) matrix, as bf16 bits."""
    out = np.empty((row_end - row_begin, H), dtype=np.uint16)
    b0, b1 = row_begin // ROW_BLOCK, (row_end - 1) // ROW_BLOCK
    for blk in range(b0, b1 + 1):
        rng = np.random.default_rng(np.random.SeedSequence([seed, blk]))
        x = rng.standard_normal((ROW_BLOCK, H), dtype=np.float32)
        x *= np.float32(std)
        lo, hi = max(row_begin, blk * ROW_BLOCK), min(row_end, (blk + 1) * ROW_BLOCK)
        out[lo - row_begin:hi - row_begin] = bf16_round(x[lo - blk * ROW_BLOCK:hi - blk * ROW_BLOCK])
    return out


def make_W(V: int, H: int, seed: int = 1, rows: tuple | None = None) -> np.ndarray:
    """LM head W_vocab[V, H] (nn.Linear layout) = bf16(N(0, 1/H)); optional row range."""
    r0, r1 = rows if rows is not None else (0, V)
    return _normal_rows(seed, r0, r1, H, 1.0 / math.sqrt(H))


def make_E(V: int, H: int, seed: int = 2, rows: tuple | None = None) -> np.ndarray:
    """Input embedding W_emb[V, H] = bf16(N(0, 1))  (not tied to W_vocab)."""
    r0, r1 = rows if rows is not None else (0, V)
    return _normal_rows(seed, r0, r1, H, 1.0)


def mask_id(V: int) -> int:
    return V - 1


def eos_id(V: int) -> int:
    return V - 2


def shard_range(V: int, rank: int, world: int) -> tuple:
    """Contiguous vocab rows owned by `rank` (V divisible by world)."""
    assert V % world == 0
    n = V // world
    return rank * n, (rank + 1) * n


class PlantedSchedule:
    """Per-position planted-confidence schedule for M = B*S positions."""

    def __init__(self, M: int, V: int, H: int, seed: int, ramp: float = 2.5,
                 flip_prob: float = 0.2, onset_max: int = 5, a0_lo: float = -3.0,
                 a0_hi: float = 1.0, noise: float = 0.3):
        self.M, self.V, self.H = M, V, H
        self.ramp, self.flip_prob, self.noise = ramp, flip_prob, noise
        self.rng = np.random.default_rng(np.random.SeedSequence([seed, 7777]))
        lnV = math.log(V)
        self.tgt = self.rng.integers(0, V - 2, size=M)
        self.onset = self.rng.integers(0, onset_max + 1, size=M)
        self.a0 = self.rng.uniform(lnV + a0_lo, lnV + a0_hi, size=M)
        self.a0_lo, self.a0_hi = lnV + a0_lo, lnV + a0_hi

    def targets_and_amplitudes(self, t: int):
        """(tgt[M], a[M]) for iteration t (fresh draws for jitter and flips)."""
        a = self.a0 + self.ramp * np.maximum(0, t - self.onset) + self.rng.uniform(0, 1, size=self.M)
        tgt = self.tgt.copy()
        flip = self.rng.uniform(0, 1, size=self.M) < self.flip_prob
        tgt[flip] = self.rng.integers(0, self.V - 2, size=int(flip.sum()))
        return tgt, a

    def redraw_base(self, rows):
        rows = np.asarray(rows)
        self.a0[rows] = self.rng.uniform(self.a0_lo, self.a0_hi, size=len(rows))

    def hidden(self, W_target_rows: np.ndarray, a: np.ndarray, rows=None) -> np.ndarray:
        """Planted h for the given positions: W_target_rows[k] = W[tgt[k]] (bf16 bits)."""
        w = bf16_to_f32(W_target_rows).astype(np.float32)
        n2 = (w.astype(np.float64) ** 2).sum(axis=1)
        a = np.asarray(a, np.float64)
        h = (a / n2)[:, None] * w
        h = h + self.rng.normal(0.0, self.noise / math.sqrt(self.H), size=h.shape)
        return bf16_round(h.astype(np.float32))


def planted_hidden(W: np.ndarray, M: int, seed: int, t: int = 0, **kw) -> np.ndarray:
    """Convenience: one [M, H] planted hidden block at iteration t (no vetting)."""
    V, H = W.shape
    sch = PlantedSchedule(M, V, H, seed, **kw)
    tgt, a = None, None
    for tt in range(t + 1):
        tgt, a = sch.targets_and_amplitudes(tt)
    return sch.hidden(W[tgt], a)
