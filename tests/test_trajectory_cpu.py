"""Generator + oracle integration on the tiny config (BASELINE configs[0]):
the vetted planted trajectory finishes a block of 32 in a handful of
iterations (TPF in the paper's 2.3-7.1 range) and every recorded
iteration keeps all decision margins (reading c19)."""
import numpy as np

import oracle as O
from paper_2510_08666_b200 import synth
from tests.trajectory import vetted_trajectory, _offenders


def _tiny():
    V, H = 1024, 256
    return synth.make_W(V, H, 1), synth.make_E(V, H, 2)


def test_tiny_threshold_trajectory():
    W, E = _tiny()
    _, _, _, steps = vetted_trajectory(W, E, 1, 32, seed=0,
                                       params_fn=lambda t: O.Params(decoder=O.DEC_THRESHOLD, tau=0.9))
    assert 2 <= len(steps) <= 16
    assert not steps[-1]["result"]["mask"].any()
    n = [int(s["result"]["committed"].sum()) for s in steps]
    assert sum(n) == 32 and min(n) >= 1


def test_tiny_hier_credit_smooth_trajectory():
    W, E = _tiny()
    pf = lambda t: O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=O.tau_schedule(0.92, t, 4),
                            theta_lo=0.62, use_credit=True, use_smooth=True,
                            alpha_t=O.alpha_schedule(0.1, 0.05, 0.3, t))
    W64, E64, em, steps = vetted_trajectory(W, E, 2, 32, seed=1, params_fn=pf, use_credit_table=True)
    assert not steps[-1]["result"]["mask"].any()
    for st in steps:
        h64 = O.bf16_bits_to_f64(st["h"])
        f = np.stack([O.logits(h64[b], W64) for b in range(2)])
        assert not _offenders(f, st["result"], st["result"]["C"], st["mask"], st["params"])
