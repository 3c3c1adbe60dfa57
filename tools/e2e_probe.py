"""Break down dinfer_step_host's end-to-end time at the bench (MoE) shape:
device-only step, copies alone, the host call (graph / plain), host wall time."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_08666_b200 import Context, make_params, synth  # noqa: E402

V, H, S, K = 157184, 2048, 32, 32
dev = torch.device("cuda")
W = torch.randn(V, H, device=dev, dtype=torch.bfloat16) * (H ** -0.5)
E = torch.randn(V, H, device=dev, dtype=torch.bfloat16)
em = E[V - 1].contiguous()
p = make_params(decoder="hierarchical", use_credit=True, use_smooth=True, alpha_t=0.1, c_gamma=0.5)
ctx = Context(1, S, H, K, V)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
hid = pin(np.random.default_rng(0).standard_normal((S, H)).astype(np.float32)).to(torch.bfloat16).pin_memory()
mask, tok = pin(np.ones((1, S), np.uint8)), pin(np.full((1, S), V - 1, np.int32))
cids, cval = pin(np.full((1, S, K), -1, np.int32)), pin(np.zeros((1, S, K), np.float32))
com, sts, sm = pin(np.zeros((1, S), np.uint8)), pin(np.zeros((1, S, 4), np.float32)), pin(np.zeros((1, S, H), np.float32))


def timed(fn, n=50, warm=5):
    ev = []
    wall = []
    for i in range(warm + n):
        mask.fill_(1); tok.fill_(V - 1); cids.fill_(-1); cval.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        t1 = time.perf_counter()
        if i >= warm:
            ev.append(e0.elapsed_time(e1) * 1e3)
            wall.append((t1 - t0) * 1e6)
    return f"event {np.median(ev):7.1f} us   wall {np.median(wall):7.1f} us"


hd = torch.empty((S, H), device=dev, dtype=torch.bfloat16)
smd = torch.empty((1, S, H), device=dev, dtype=torch.float32)
m_d, t_d = torch.ones((1, S), dtype=torch.uint8, device=dev), torch.full((1, S), V - 1, dtype=torch.int32, device=dev)
c_d, v_d = torch.full((1, S, K), -1, dtype=torch.int32, device=dev), torch.zeros((1, S, K), device=dev)
co_d, st_d = torch.zeros((1, S), dtype=torch.uint8, device=dev), torch.zeros((1, S, 4), device=dev)


def dev_step():
    m_d.fill_(1); t_d.fill_(V - 1); c_d.fill_(-1); v_d.zero_()
    ctx.step(hd, W, E, em, m_d, t_d, c_d, v_d, p, co_d, smd, st_d)


def copies():
    hd.copy_(hid, non_blocking=True)
    sm.copy_(smd, non_blocking=True)


print("device step   ", timed(dev_step))
print("copies only   ", timed(copies))
print("step_host     ", timed(lambda: ctx.step_host(hid, W, E, em, mask, tok, cids, cval, p, com, sm, sts)))
ctx.set_timing(True)
print("host+timing   ", timed(lambda: ctx.step_host(hid, W, E, em, mask, tok, cids, cval, p, com, sm, sts)))
ctx.set_timing(False)
