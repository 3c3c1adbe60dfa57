"""Drive the CUDA path (through the C ABI) on the same seeded inputs as the
oracle and compare element by element.  Test infrastructure."""
from __future__ import annotations

import numpy as np

import oracle as O

TOL_REL = 2e-3          # north_star: lse / smoothed within 2e-3 relative
TOL_CREDIT_REL = 1e-4   # credit values: fp32 functions of p* (DESIGN.md c17)


def to_dev_bf16(u16):
    import torch
    return torch.from_numpy(np.ascontiguousarray(u16).view(np.int16)).view(torch.bfloat16).cuda()


class GpuState:
    """Device-side decode state + outputs for one context."""

    def __init__(self, B, S, H, K, mask_id):
        import torch
        self.B, self.S, self.H, self.K = B, S, H, K
        dev = "cuda"
        self.mask = torch.ones((B, S), dtype=torch.uint8, device=dev)
        self.tokens = torch.full((B, S), mask_id, dtype=torch.int32, device=dev)
        self.cids = torch.full((B, S, K), -1, dtype=torch.int32, device=dev)
        self.cval = torch.zeros((B, S, K), dtype=torch.float32, device=dev)
        self.committed = torch.zeros((B, S), dtype=torch.uint8, device=dev)
        self.smoothed = torch.full((B, S, H), float("nan"), dtype=torch.float32, device=dev)
        self.stats = torch.zeros((B, S, 4), dtype=torch.float32, device=dev)

    def load(self, mask, tokens):
        import torch
        self.mask.copy_(torch.from_numpy(np.asarray(mask, np.uint8)))
        self.tokens.copy_(torch.from_numpy(np.asarray(tokens, np.int32)))

    def snapshot(self):
        st = self.stats.cpu().numpy()
        return dict(mask=self.mask.cpu().numpy().astype(bool), tokens=self.tokens.cpu().numpy().astype(np.int64),
                    committed=self.committed.cpu().numpy().astype(bool), cids=self.cids.cpu().numpy(),
                    cval=self.cval.cpu().numpy(), smoothed=self.smoothed.cpu().numpy(),
                    m=st[..., 0], lse=st[..., 1], ptilde=st[..., 2], vtilde=st[..., 3].view(np.int32))


def gpu_params(p: O.Params):
    from paper_2510_08666_b200 import make_params
    return make_params(decoder=p.decoder, tau=p.tau, theta_hi=p.theta_hi, theta_lo=p.theta_lo,
                       hier_runs_after_hi=p.hier_runs_after_hi, use_credit=p.use_credit, c_alpha=p.c_alpha,
                       c_beta=p.c_beta, c_gamma=p.c_gamma, use_smooth=p.use_smooth, alpha_t=p.alpha_t,
                       smooth_credit_fused=p.smooth_credit_fused, inclusive=p.inclusive)


def compare(out, gold, mask_before, params: O.Params, where="", exclude=()):
    """Element-by-element parity of one step.  Integer / decision state is
    bit-exact; floating outputs within the stated tolerances.  `exclude`:
    positions (b, s) whose own top-2 margin is within 1e-3 (reading c19) --
    their v~ / p~ / credit slots are not compared (every decision still is)."""
    B, S = mask_before.shape
    und_all = np.array(mask_before, bool)
    mask_before = und_all.copy()
    for b, s in exclude:
        mask_before[b, s] = False
    np.testing.assert_array_equal(out["committed"], gold["committed"], err_msg=f"committed {where}")
    np.testing.assert_array_equal(out["mask"], gold["mask"], err_msg=f"mask {where}")
    np.testing.assert_array_equal(out["tokens"], gold["tokens"], err_msg=f"tokens {where}")
    for key in ("m", "lse"):
        ref = gold[key]
        err = np.abs(out[key] - ref) / np.maximum(1.0, np.abs(ref))
        assert err.max() <= TOL_REL, f"{key} rel err {err.max():.3g} {where}"
    und = mask_before
    np.testing.assert_array_equal(out["vtilde"][und], gold["vtilde"][und], err_msg=f"vtilde {where}")
    perr = np.abs(out["ptilde"][und] - gold["ptilde"][und])
    assert perr.size == 0 or perr.max() <= TOL_REL, f"ptilde abs err {perr.max():.3g} {where}"
    if params.use_credit:
        C = gold["C"]
        for b in range(B):
            for s in range(S):
                if not und[b, s]:
                    continue
                got = {int(i): float(v) for i, v in zip(out["cids"][b, s], out["cval"][b, s]) if i >= 0}
                nz = np.nonzero(C[b, s])[0]
                want = {int(v): float(C[b, s, v]) for v in nz}
                assert set(got) == set(want), f"credit ids b{b} s{s} {sorted(got)} vs {sorted(want)} {where}"
                for v in want:
                    assert abs(got[v] - want[v]) <= TOL_CREDIT_REL * max(1.0, abs(want[v])), \
                        f"credit val b{b} s{s} v{v} {got[v]} vs {want[v]} {where}"
    if params.use_smooth:
        still = gold["mask"] & und_all
        for b in range(B):
            for s in np.nonzero(still[b])[0]:
                ref = gold["smoothed"][b, s]
                got = out["smoothed"][b, s]
                rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                assert rel <= TOL_REL, f"smoothed normwise rel {rel:.3g} b{b} s{s} {where}"


TOL_EMB_REL = TOL_REL + 2.0 ** -9  # bf16 model input: + one bf16 rounding (DESIGN.md c24)


def bf16_round_bits(x):
    """fp32 -> bf16 bit patterns, round to nearest even (test-side reference)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def compare_embed(emb_bits, out, gold, E_bits, where=""):
    """Next-iteration input (f2): decided rows are W_emb[token] bit for bit;
    masked rows are bf16(e_{t+1}) -- the GPU's own fp32 smoothed row rounded
    to nearest (bit-exact) and within TOL_EMB_REL of the oracle's fp64 row."""
    B, S = gold["mask"].shape
    oracle_emb = O.next_input_embedding(O.bf16_bits_to_f64(E_bits), gold["tokens"], gold["mask"], gold["smoothed"])
    for b in range(B):
        for s in range(S):
            if not gold["mask"][b, s]:
                np.testing.assert_array_equal(emb_bits[b, s], E_bits[gold["tokens"][b, s]],
                                              err_msg=f"emb decided row b{b} s{s} {where}")
            else:
                np.testing.assert_array_equal(emb_bits[b, s], bf16_round_bits(out["smoothed"][b, s]),
                                              err_msg=f"emb masked row = bf16(smoothed) b{b} s{s} {where}")
                got = O.bf16_bits_to_f64(emb_bits[b, s])
                ref = oracle_emb[b, s]
                rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                assert rel <= TOL_EMB_REL, f"emb normwise rel {rel:.3g} b{b} s{s} {where}"


def replay(ctx, W_dev, E_dev, em_dev, steps, B, S, H, K, V, on_step=None, E_bits=None):
    """Feed every vetted iteration's hidden states to the CUDA path, carrying
    the GPU's OWN decode state, and compare with the oracle's golden result.
    With E_bits (host bf16 [V, H]) the step also writes the next-iteration
    input embedding (dinfer_step_embed), checked by compare_embed."""
    import torch
    from paper_2510_08666_b200 import synth
    st = GpuState(B, S, H, K, synth.mask_id(V))
    emb = None
    if E_bits is not None:
        emb = torch.full((B, S, H), -1, dtype=torch.int16, device="cuda")
    for t, step in enumerate(steps):
        p = step["params"]
        hid = to_dev_bf16(step["h"].reshape(B * S, H))
        args = (hid, W_dev, E_dev if p.use_smooth else None, em_dev if p.use_smooth else None, st.mask, st.tokens,
                st.cids if p.use_credit else None, st.cval if p.use_credit else None, gpu_params(p),
                st.committed, st.smoothed if p.use_smooth else None, st.stats)
        if emb is not None:
            emb.fill_(-1)  # 0xFFFF (NaN) everywhere: every row must be written
            ctx.step_embed(*args, emb)
        else:
            ctx.step(*args)
        torch.cuda.synchronize()
        ctx.sync()
        out = st.snapshot()
        compare(out, step["result"], step["mask"], p, where=f"iter {t}")
        if emb is not None:
            compare_embed(emb.cpu().numpy().view(np.uint16), out, step["result"], E_bits, where=f"iter {t}")
        if on_step is not None:
            on_step(t, out)
    return st
