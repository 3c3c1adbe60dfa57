"""GPU parity of the device-resident generation loop (dinfer_generate, Alg. 1
with schedules, per-block credit reset and EOS early termination; SURVEY
§8(f) f1) against the oracle's generate() on margin-vetted planted
trajectories.  Token rows X, T_b and the forward count F must match exactly."""
import numpy as np
import pytest

import oracle as O
from paper_2510_08666_b200 import synth
from tests.gpu_harness import gpu_params, to_dev_bf16
from tests.trajectory import vetted_generation

pytestmark = pytest.mark.gpu

V, H, S = 1024, 256, 32


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2510_08666_b200 import build
    build.build()
    return torch


def _gen_cfg(ocfg: O.GenConfig, L):
    from paper_2510_08666_b200 import make_gen_config
    return make_gen_config(L, ocfg.prompt_len, ocfg.mask_id, ocfg.eos_id, ocfg.early_termination, ocfg.tau_target,
                           ocfg.tau_decay_steps, ocfg.alpha_init, ocfg.alpha_growth, ocfg.alpha_preset,
                           min(ocfg.max_forwards, 1 << 30))


def _run(torch, B, nblocks, P, seed, base, ocfg, eos_at, K=16, repeats=1, **sched):
    from paper_2510_08666_b200 import Context
    W, E = synth.make_W(V, H, 1), synth.make_E(V, H, 2)
    hid, X0, ref = vetted_generation(W, E, B, S, nblocks, P, seed, base, ocfg, eos_at=eos_at, **sched)
    ctx = Context(B, S, H, K, V)
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[ocfg.mask_id])
    hsrc = to_dev_bf16(hid)
    X = torch.from_numpy(X0.astype(np.int32)).cuda()
    out = torch.zeros(B + 2, dtype=torch.int32, device="cuda")
    for r in range(repeats):  # graph reuse: same pointers, same configuration
        X.copy_(torch.from_numpy(X0.astype(np.int32)))
        out.zero_()
        ctx.generate(_gen_cfg(ocfg, X0.shape[1]), gpu_params(base), Wd, Ed, emd, hsrc, X, out)
        ctx.sync()
        torch.cuda.synchronize()
        got = X.cpu().numpy()
        o = out.cpu().numpy()
        bad = np.argwhere(got != ref["X"])
        assert len(bad) == 0, f"repeat {r}: X differs at {bad[:8].tolist()} (F ref {ref['F']}, gpu {o[B]})"
        assert o[B] == ref["F"], (o, ref["F"])
        assert list(o[:B]) == list(ref["T"]), (o, ref["T"])
        assert o[B + 1] == int(ref["truncated"])
    return ref


def test_generate_hier_credit_smooth_early_termination(torch_cuda):
    base = O.Params(decoder=O.DEC_HIERARCHICAL, theta_lo=0.62, use_credit=True, use_smooth=True)
    cfg = O.GenConfig(prompt_len=5, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.9, tau_decay_steps=3,
                      alpha_init=0.1, alpha_growth=0.05, alpha_preset=0.3)
    ref = _run(torch_cuda, 2, 4, 5, 1, base, cfg, eos_at=[(0, 1, 9), (1, 2, 3)], repeats=2)
    assert ref["F"] < 4 * S and (ref["X"][:, -S:] == V - 2).all()   # early termination exercised


def test_generate_threshold_full_run(torch_cuda):
    base = O.Params(decoder=O.DEC_THRESHOLD)
    cfg = O.GenConfig(prompt_len=0, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.85, tau_decay_steps=0,
                      early_termination=False)
    _run(torch_cuda, 1, 3, 0, 4, base, cfg, eos_at=[(0, 0, 20)])


def test_generate_credit_no_smooth_rows_finish_apart(torch_cuda):
    base = O.Params(decoder=O.DEC_THRESHOLD, use_credit=True)
    cfg = O.GenConfig(prompt_len=7, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.8, tau_decay_steps=2)
    _run(torch_cuda, 3, 3, 7, 5, base, cfg, eos_at=[(1, 0, 30)])


def test_generate_max_forwards_truncates(torch_cuda):
    base = O.Params(decoder=O.DEC_HIERARCHICAL, use_smooth=True)
    cfg = O.GenConfig(prompt_len=2, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.9, max_forwards=5)
    ref = _run(torch_cuda, 2, 3, 2, 6, base, cfg, eos_at=[])
    assert ref["truncated"] and ref["F"] == 5


def test_generate_on_the_fused_kernel(torch_cuda, monkeypatch):
    """The generation graph around K12 (forced: the tiny vocabulary would pick
    K1 -> K2), hierarchical + credit + smoothing with early termination: the
    loop must match the oracle token for token."""
    monkeypatch.setenv("DINFER_FUSED", "2")
    base = O.Params(decoder=O.DEC_HIERARCHICAL, theta_lo=0.62, use_credit=True, use_smooth=True)
    cfg = O.GenConfig(prompt_len=3, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.9, tau_decay_steps=3,
                      alpha_init=0.1, alpha_growth=0.05, alpha_preset=0.3)
    _run(torch_cuda, 2, 3, 3, 7, base, cfg, eos_at=[(1, 1, 5)], repeats=2)



def test_generate_credit_tpf_exceeds_threshold(torch_cuda):
    """SPEC S:542 directional check, on the GPU loop: a stable suite (fixed
    targets, confidence rising monotonically: ramp 1.0, onset 0, no flips),
    every forward margin-vetted against the oracle.  X, T_b and F match the
    oracle exactly for both decoders, and credit decoding's mean TPF
    (T_i / F_i over the suite) strictly exceeds threshold
    decoding's at the same tau."""
    cfg = O.GenConfig(prompt_len=3, S=S, mask_id=V - 1, eos_id=V - 2, tau_target=0.9, early_termination=False)
    tpf = {}
    for name, base in (("threshold", O.Params(decoder=O.DEC_THRESHOLD)),
                       ("credit", O.Params(decoder=O.DEC_THRESHOLD, use_credit=True))):
        per = []
        for seed in range(3):
            ref = _run(torch_cuda, 1, 2, 3, 20 + seed, base, cfg, eos_at=[], ramp=1.0, flip_prob=0.0, onset_max=0)
            per.append(ref["T"][0] / ref["F"])
        tpf[name] = float(np.mean(per))
    assert tpf["credit"] > tpf["threshold"], tpf
