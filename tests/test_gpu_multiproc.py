"""Two processes on one GPU exchange per-rank records over torch.distributed
(gloo) exactly as the NCCL allgather would: rank r runs dinfer_step_local on
its vocab shard, the records are all-gathered in rank order, every rank runs
dinfer_step_combine and must end with the identical state, equal to the
oracle's unsharded step.  (NCCL itself needs >= 2 GPUs; this covers the
multi-process protocol of the sharded path on the single-GPU box.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2510_08666_b200 import Context, synth
    from tests.gpu_harness import GpuState, compare, gpu_params, to_dev_bf16
    from tests.trajectory import vetted_trajectory

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        V, H, B, S, K = 2048, 256, 1, 32, 32
        W, E = synth.make_W(V, H, 1), synth.make_E(V, H, 2)
        pf = lambda t: O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=O.tau_schedule(0.92, t, 4), use_credit=True,
                                use_smooth=True, alpha_t=0.2)
        _, _, _, steps = vetted_trajectory(W, E, B, S, 40, pf, max_iters=4, use_credit_table=True)
        v0, v1 = synth.shard_range(V, rank, world)
        ctx = Context(B, S, H, K, V, V_local=v1 - v0, v_offset=v0, world=world, rank=rank)
        Wd, Ed = to_dev_bf16(W[v0:v1]), to_dev_bf16(E[v0:v1])
        emd = to_dev_bf16(E[synth.mask_id(V)])
        words = ctx.record_words(True)
        rec = torch.zeros(words, dtype=torch.float32, device="cuda")
        st = GpuState(B, S, H, K, synth.mask_id(V))
        ok = True
        for t, step in enumerate(steps):
            gp = gpu_params(step["params"])
            ctx.step_local(to_dev_bf16(step["h"].reshape(B * S, H)), Wd, Ed, st.mask, st.cids, gp, rec)
            torch.cuda.synchronize()
            parts = [torch.zeros(words, dtype=torch.float32) for _ in range(world)]
            dist.all_gather(parts, rec.cpu())
            recs = torch.stack(parts).cuda()
            ctx.step_combine(recs, emd, st.mask, st.tokens, st.cids, st.cval, gp, st.committed, st.smoothed,
                             st.stats)
            torch.cuda.synchronize()
            ctx.sync()
            snap = st.snapshot()
            compare(snap, step["result"], step["mask"], step["params"], where=f"rank {rank} iter {t}")
        out[rank] = {k: snap[k] for k in ("tokens", "mask", "cids", "cval", "smoothed", "lse")}
        out[f"ok{rank}"] = ok
    finally:
        dist.destroy_process_group()


def _worker_p2p(rank, world, port, out):
    """Full dinfer_step on each rank's vocab shard with the records exchanged
    IN-KERNEL over peer memory (CUDA IPC; both processes share the one GPU,
    whose time-slicing interleaves their kernels)."""
    import torch
    import torch.distributed as dist

    import oracle as O
    from paper_2510_08666_b200 import Context, synth
    from tests.gpu_harness import GpuState, compare, gpu_params, to_dev_bf16
    from tests.trajectory import vetted_trajectory

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        V, H, B, S, K = 4096, 256, 1, 32, 32
        W, E = synth.make_W(V, H, 1), synth.make_E(V, H, 2)
        pf = lambda t: O.Params(decoder=O.DEC_HIERARCHICAL, theta_hi=O.tau_schedule(0.92, t, 4), use_credit=True,
                                use_smooth=True, alpha_t=O.alpha_schedule(0.1, 0.05, 0.3, t))
        _, _, _, steps = vetted_trajectory(W, E, B, S, 41, pf, max_iters=5, use_credit_table=True)
        v0, v1 = synth.shard_range(V, rank, world)
        ctx = Context(B, S, H, K, V, V_local=v1 - v0, v_offset=v0, world=world, rank=rank)
        handles = [None] * world
        dist.all_gather_object(handles, ctx.exchange_handle())
        ctx.exchange_open(b"".join(handles))
        Wd, Ed = to_dev_bf16(W[v0:v1]), to_dev_bf16(E[v0:v1])
        emd = to_dev_bf16(E[synth.mask_id(V)])
        st = GpuState(B, S, H, K, synth.mask_id(V))
        for t, step in enumerate(steps):
            ctx.step(to_dev_bf16(step["h"].reshape(B * S, H)), Wd, Ed, emd, st.mask, st.tokens, st.cids, st.cval,
                     gpu_params(step["params"]), st.committed, st.smoothed, st.stats)
            torch.cuda.synchronize()
            ctx.sync()
            snap = st.snapshot()
            compare(snap, step["result"], step["mask"], step["params"], where=f"p2p rank {rank} iter {t}")
        out[rank] = {k: snap[k] for k in ("tokens", "mask", "cids", "cval", "smoothed", "lse")}
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_exchange_records_over_peer_memory():
    """The product's multi-GPU exchange (dinfer_exchange_open): rank records
    pushed into each other's gather buffers by the record-finalize kernel,
    epoch flags awaited by K34; both ranks end bit-identical and equal to the
    unsharded oracle along a whole trajectory."""
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_p2p, args=(2, _port(), out), nprocs=2, join=True)
    for k in ("tokens", "mask", "cids", "cval", "lse"):
        assert np.array_equal(out[0][k], out[1][k]), k
    assert np.array_equal(np.nan_to_num(out[0]["smoothed"]), np.nan_to_num(out[1]["smoothed"]))


def test_two_processes_exchange_records_over_gloo():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    for k in ("tokens", "mask", "cids", "cval", "lse"):
        assert np.array_equal(out[0][k], out[1][k]), k
    assert np.array_equal(np.nan_to_num(out[0]["smoothed"]), np.nan_to_num(out[1]["smoothed"]))


def test_step_is_cuda_graph_capturable():
    """dinfer_step enqueues only kernels on the ctx stream (no host sync, no
    allocation): capture it into a CUDA graph and replay == eager."""
    import torch

    import oracle as O
    from paper_2510_08666_b200 import Context, synth
    from tests.gpu_harness import GpuState, gpu_params, to_dev_bf16
    V, H, B, S, K = 4096, 512, 1, 32, 16
    W, E = synth.make_W(V, H, 1), synth.make_E(V, H, 2)
    h = to_dev_bf16(synth.planted_hidden(W, B * S, seed=41))
    Wd, Ed, emd = to_dev_bf16(W), to_dev_bf16(E), to_dev_bf16(E[V - 1])
    p = gpu_params(O.Params(decoder=O.DEC_HIERARCHICAL, use_credit=True, use_smooth=True))
    s = torch.cuda.Stream()
    ctx = Context(B, S, H, K, V, stream=s.cuda_stream)
    eager, graphed = GpuState(B, S, H, K, V - 1), GpuState(B, S, H, K, V - 1)
    with torch.cuda.stream(s):
        ctx.step(h, Wd, Ed, emd, eager.mask, eager.tokens, eager.cids, eager.cval, p, eager.committed,
                 eager.smoothed, eager.stats)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.step(h, Wd, Ed, emd, graphed.mask, graphed.tokens, graphed.cids, graphed.cval, p, graphed.committed,
                 graphed.smoothed, graphed.stats)
    for _ in range(2):  # replay twice from the same initial state
        graphed.mask.fill_(1)
        graphed.tokens.fill_(V - 1)
        graphed.cids.fill_(-1)
        graphed.cval.zero_()
        g.replay()
        torch.cuda.synchronize()
        a, b = eager.snapshot(), graphed.snapshot()
        for k in ("committed", "tokens", "mask", "cids", "cval", "m", "lse", "ptilde"):
            assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(np.nan_to_num(a["smoothed"]), np.nan_to_num(b["smoothed"]))
