"""World-size-2 (gloo, CPU) tests of the host side of the vocab-sharded path:
the NCCL unique-id bootstrap over torch.distributed, per-rank shard
generation, and the record allgather + combine data flow (using the oracle's
shard-merge mode): every rank ends with the identical,
unsharded result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2510_08666_b200 import synth
from paper_2510_08666_b200.dist import broadcast_unique_id, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = broadcast_unique_id("cpu")
        V, H, M = 1024, 64, 16
        v0, v1 = shard_range(V, rank, world)
        W_shard = synth.make_W(V, H, 1, rows=(v0, v1))
        E_shard = synth.make_E(V, H, 2, rows=(v0, v1))
        W_full = synth.make_W(V, H, 1)
        h = O.bf16_bits_to_f64(synth.planted_hidden(W_full, M, seed=4))
        f = O.logits(h, O.bf16_bits_to_f64(W_shard))
        rec = O.shard_record(f, v0, O.bf16_bits_to_f64(E_shard))
        packed = torch.from_numpy(np.concatenate([rec["m"], rec["vstar"].astype(np.float64), rec["l"],
                                                  rec["acc"].ravel()]))
        gathered = [torch.zeros_like(packed) for _ in range(world)]
        dist.all_gather(gathered, packed)
        recs = []
        for g in gathered:
            a = g.numpy()
            recs.append(dict(m=a[:M], vstar=a[M:2 * M].astype(np.int64), l=a[2 * M:3 * M],
                             acc=a[3 * M:].reshape(M, H)))
        merged = O.merge_records(recs)
        out[rank] = dict(uid=uid, shard_equal=bool(np.array_equal(W_shard, W_full[v0:v1])),
                         vstar=merged["vstar"], lse=merged["lse"], sm=merged["acc"] / merged["l"][:, None])
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_shards_and_combine():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert len(r0["uid"]) == 128 and r0["uid"] == r1["uid"]
    assert r0["shard_equal"] and r1["shard_equal"]
    # replicated state: bit-identical on both ranks
    assert np.array_equal(r0["vstar"], r1["vstar"]) and np.array_equal(r0["lse"], r1["lse"])
    assert np.array_equal(r0["sm"], r1["sm"])
    # and equal to the unsharded definition
    V, H, M = 1024, 64, 16
    W = O.bf16_bits_to_f64(synth.make_W(V, H, 1))
    E = O.bf16_bits_to_f64(synth.make_E(V, H, 2))
    h = O.bf16_bits_to_f64(synth.planted_hidden(synth.make_W(V, H, 1), M, seed=4))
    f = O.logits(h, W)
    m, vs, lse, ps = O.softmax_stats(f)
    assert np.array_equal(r0["vstar"], vs)
    np.testing.assert_allclose(r0["lse"], lse, rtol=1e-13)
    np.testing.assert_allclose(r0["sm"], O.softmax(f) @ E, rtol=1e-10, atol=1e-12)


def test_shard_generation_is_rank_independent():
    V, H = 5000 * 8, 32
    full = synth.make_W(V, H, 1)
    for world in (2, 4, 8):
        for r in range(world):
            a, b = shard_range(V, r, world)
            assert np.array_equal(synth.make_W(V, H, 1, rows=(a, b)), full[a:b])
