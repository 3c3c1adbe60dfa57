#!/usr/bin/env python
"""Benchmark of the fused denoise-and-commit step (dInfer, arXiv 2510.08666).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                  [--config moe|8b|8b-bs64|tiny] [--shard-sim G]

Workload (BASELINE.json metric: "denoise-step positions/sec and HBM GB/s
fraction, LLaDA-MoE shape bs1, 1/2/4/8 B200"): configs[2], LLaDA-MoE shape
H=2048, V=157184, block S=32, batch 1, hierarchical + credit decoding +
iteration smoothing; for N > 1 the vocabulary is sharded over the N GPUs
(configs[3]) and the ranks read each other's records in place over NVLink once
the producing kernel raises their flags (peer-memory exchange; NCCL allgather
fallback).  A
step = one dinfer_step on the first iteration of a block (all 32 positions
undecided, fresh credit): K12 (vocab projection + softmax statistics +
smoothing contraction; when sharded it also builds the rank's record -- the
accumulator added into one fp32 record with L2 reductions -- and raises the
exchange flags) then K34 (combine, credit, selection, commit, smoothing
output; when sharded it reads the peers' records in place).
Synthetic seeded weights and planted hidden states (paper_2510_08666_b200.synth).
The headline times K back-to-back steps (each a block's first iteration,
params.block_start) under one event pair; every step reads weights the L2 does
not hold (1.29 GB per step at N=1; for shards smaller than 3x the L2 the loop
rotates over enough weight copies).  The same steps timed one at a time with
the L2 flushed before each are reported under "l2_flushed", and the steps
replayed from one CUDA graph under "graph_replay".

--shard-sim G (N=1 only, measurement): one rank of a G-way vocab shard on one
GPU (V_local = V/G; every "peer" is its own exchange buffer, so K34 reads the
rank's record G times -- dinfer_exchange_loopback), i.e. the per-rank step of
configs[3] minus the NVLink latency; its decisions are not meaningful.

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
reference arm of this tier) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "denoise-step positions/sec and HBM GB/s fraction, LLaDA-MoE shape bs1, 1/2/4/8 B200"
UNIT = "positions/s"
# BASELINE.json configs.  The default (the metric's workload) is "moe".
CONFIGS = {
    "moe": dict(B=1, S=32, H=2048, V=157184, K=32, decoder="hierarchical", credit=True, smooth=True,
                workload="LLaDA-MoE shape bs1 block32 hierarchical+credit+smoothing (BASELINE configs[2]; "
                         "vocab-sharded configs[3] for N>1)"),
    "8b": dict(B=1, S=32, H=4096, V=126464, K=32, decoder="threshold", credit=False, smooth=False,
               workload="LLaDA-8B shape bs1 block32 threshold decoding (BASELINE configs[1])"),
    "8b-bs64": dict(B=64, S=64, H=4096, V=126464, K=8, decoder="threshold", credit=False, smooth=False,
                    workload="LLaDA-8B shape bs64 block64 threshold decoding, compute-bound (BASELINE configs[4])"),
    "tiny": dict(B=1, S=32, H=256, V=1024, K=32, decoder="threshold", credit=False, smooth=False,
                 workload="tiny synthetic block32 hidden256 vocab1024 threshold 0.9 (BASELINE configs[0])"),
}
B = S = H = V = K = None
CFG = None
WORKLOAD = None


def set_config(name):
    global B, S, H, V, K, CFG, WORKLOAD
    CFG = dict(CONFIGS[name], name=name)
    B, S, H, V, K = CFG["B"], CFG["S"], CFG["H"], CFG["V"], CFG["K"]
    WORKLOAD = CFG["workload"]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def peaks_sustained():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops_sustained"])
    except Exception:
        return 1400.0


def ncu_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def report(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ oracle (CPU) arm
def oracle_run(n_steps: int, n_warm: int, rows: int, budget_s: float | None = None, threads: int | None = None):
    """Time the CPU oracle (as it stands) on `rows` positions of the workload
    per step, with the BLAS pools limited to `threads` (None: all host cores).
    Returns (seconds per step list, threads used)."""
    import oracle as O
    from paper_2510_08666_b200 import synth
    from threadpoolctl import threadpool_info, threadpool_limits
    W_u16 = synth.make_W(V, H, 1)
    W = O.bf16_bits_to_f64(W_u16)
    E = O.bf16_bits_to_f64(synth.make_E(V, H, 2)) if CFG["smooth"] else W[:1]
    h = O.bf16_bits_to_f64(synth.planted_hidden(W_u16, S, seed=0))[:rows].reshape(1, rows, H)
    del W_u16
    em = E[synth.mask_id(V)] if CFG["smooth"] else None
    p = O.Params(decoder=O.DEC_HIERARCHICAL if CFG["decoder"] == "hierarchical" else O.DEC_THRESHOLD,
                 tau=0.9, theta_hi=0.92, theta_lo=0.62, use_credit=CFG["credit"], use_smooth=CFG["smooth"],
                 alpha_t=0.1)
    times = []
    with threadpool_limits(limits=threads):
        cores = max((d.get("num_threads", 1) for d in threadpool_info()), default=1)
        for i in range(n_warm + n_steps):
            mask = np.ones((1, rows), bool)
            tok = np.full((1, rows), V - 1)
            C = np.zeros((1, rows, V)) if CFG["credit"] else None
            t0 = time.perf_counter()
            O.step(h, W, E, em, mask, tok, C, p)
            dt = time.perf_counter() - t0
            if i >= n_warm:
                times.append(dt)
            if budget_s is not None and i >= n_warm and sum(times) > budget_s:
                break
    return times, cores


def bench_config(world: int, Vl: int, exchange: str, partition: str, weight_copies: int, shard_sim: int = 0):
    """The `config` object of both arms (same keys, so the driver can match them)."""
    G = shard_sim or world
    step_bytes = Vl * H * 2 * (2 if CFG["smooth"] else 1)
    if shard_sim:
        par = f"one rank of a {shard_sim}-way vocab shard on one GPU (loopback record exchange; measurement)"
    elif world > 1:
        par = f"vocab-sharded x{world} (" + ("in-kernel peer-memory record exchange" if exchange == "p2p"
                                              else "NCCL allgather") + ")"
    else:
        par = "single GPU"
    return {"workload": WORKLOAD, "name": CFG["name"], "B": B, "S": S, "H": H, "V": V, "K": K,
            "decoder": CFG["decoder"], "credit": CFG["credit"], "smooth": CFG["smooth"], "vocab_shards": G,
            "V_local": Vl, "parallelism": par, "exchange": exchange, "partition": partition,
            "l2": (f"no flush: every step reads weights the L2 does not hold ({step_bytes / 1e9:.2f} GB of W/E per "
                   f"step per GPU, {weight_copies} weight cop{'y' if weight_copies == 1 else 'ies'} rotated, "
                   f"vs 126 MB L2); K back-to-back block-start steps under one event pair")}


def default_partition(balance: bool) -> str:
    return ("calibrated for back-to-back steps (dinfer_balance, 4 steps)" if CFG["smooth"] and balance
            else "even")


def weight_copies_for(shard_bytes: int, l2_bytes: int = 126 * 1024 * 1024) -> int:
    """Copies of the weight shard rotated by the headline loop so that each
    step reads bytes the L2 cannot hold: >= 3x the L2 in total."""
    return max(1, min(4, math.ceil(3 * l2_bytes / max(1, shard_bytes))))


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    rows = 8  # bounded sample: 8 of the 32 positions per step (cost ~ linear in rows)
    times, cores = oracle_run(args.steps, args.warmup, rows)
    sec = sum(times) / len(times)
    value = rows / sec
    G = args.gpus
    Vl = V // G
    cfg = bench_config(G, Vl, "p2p" if G > 1 else "none", default_partition(args.balance),
                       weight_copies_for(Vl * H * 2 * (2 if CFG["smooth"] else 1)))
    cfg["oracle"] = "host cores (numpy fp64 oracle, whole vocabulary)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{rows} of {B * S} positions per step, full vocab {V}, fp64 numpy oracle step "
                                   f"({CFG['decoder']}, credit={CFG['credit']}, smoothing={CFG['smooth']})"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def gpu_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2510_08666_b200 import Context, build, make_params, synth

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.shard_sim and world != 1:
        raise SystemExit("--shard-sim is a single-GPU measurement")
    # BENCH_SAME_DEVICE=1 (test hook): every rank on cuda:0 with a gloo process
    # group, so the N > 1 code path can run on a one-GPU box (--exchange p2p)
    same_dev = os.environ.get("BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2510_08666_b200 import dinfer as _d
    _d.lib()

    # ---- synthetic inputs: this rank's vocab shard of W and E
    G = args.shard_sim or world  # vocab shards
    v0, v1 = synth.shard_range(V, rank, G)
    Vl = v1 - v0
    smooth, credit = CFG["smooth"], CFG["credit"]
    W_u16 = synth.make_W(V, H, 1, rows=(v0, v1))
    Wfull_rows = synth.make_W(V, H, 1) if G > 1 else W_u16  # planted hidden needs W[target] rows
    hid_u16 = synth.planted_hidden(Wfull_rows, B * S, seed=0)
    del Wfull_rows

    def dev_bf16(u):
        return torch.from_numpy(np.ascontiguousarray(u).view(np.int16)).view(torch.bfloat16).cuda()

    hid = dev_bf16(hid_u16)
    shard_bytes = Vl * H * 2 * (2 if smooth else 1)
    R = weight_copies_for(shard_bytes, torch.cuda.get_device_properties(local).L2_cache_size)
    Wd = [dev_bf16(W_u16)]
    Ed = [dev_bf16(synth.make_E(V, H, 2, rows=(v0, v1)))] if smooth else [None]
    for _ in range(R - 1):  # identical copies at other addresses (L2-cold rotation)
        Wd.append(Wd[0].clone())
        Ed.append(Ed[0].clone() if smooth else None)
    emd = dev_bf16(synth.make_E(V, H, 2, rows=(V - 1, V))[0]) if smooth else None
    del W_u16

    stream = torch.cuda.Stream()
    nid = None
    if world > 1 and args.exchange != "p2p":  # the NCCL communicator (allgather / fallback)
        from paper_2510_08666_b200.dist import broadcast_unique_id
        nid = broadcast_unique_id("cpu" if same_dev else "cuda")
    ctx = Context(B, S, H, K, V, V_local=Vl, v_offset=v0, world=G, rank=rank, stream=stream.cuda_stream,
                  nccl_id=nid, smooth_capable=smooth)
    exchange = "none"
    if args.shard_sim:
        ctx.exchange_loopback()
        exchange = "loopback"
    elif world > 1:
        # the product's exchange: K34 reads every rank's record in place over NVLink P2P
        # once the producing kernel raised that rank's flag (CUDA IPC handles shared via
        # torch.distributed); the NCCL allgather stays as the fallback / --exchange nccl
        exchange = "nccl"
        if args.exchange in ("auto", "p2p"):
            from paper_2510_08666_b200 import DInferError
            handles = [None] * world
            dist.all_gather_object(handles, ctx.exchange_handle())
            try:
                ctx.exchange_open(b"".join(handles))
                ok = 1
            except DInferError as e:
                if args.exchange == "p2p":
                    raise
                print(f"[bench] peer-memory exchange unavailable ({e}); using the NCCL allgather", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device="cpu" if same_dev else "cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag[0]) == 1:
                exchange = "p2p"
            elif ok:
                raise SystemExit("peer-memory exchange opened on some ranks only")
    p = make_params(decoder=CFG["decoder"], tau=0.9, theta_hi=0.92, theta_lo=0.62, use_credit=credit,
                    use_smooth=smooth, alpha_t=0.1)

    dev = "cuda"
    M = B * S
    mask = torch.ones((B, S), dtype=torch.uint8, device=dev)
    tokens = torch.full((B, S), V - 1, dtype=torch.int32, device=dev)
    cids = torch.full((B, S, K), -1, dtype=torch.int32, device=dev)
    cval = torch.zeros((B, S, K), dtype=torch.float32, device=dev)
    committed = torch.zeros((B, S), dtype=torch.uint8, device=dev)
    smoothed = torch.zeros((B, S, H), dtype=torch.float32, device=dev) if smooth else None
    stats = torch.zeros((B, S, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def reset_and_flush():
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
            mask.fill_(1)
            tokens.fill_(V - 1)
            cids.fill_(-1)
            cval.zero_()

    p_bs = make_params(decoder=CFG["decoder"], tau=0.9, theta_hi=0.92, theta_lo=0.62, use_credit=credit,
                       use_smooth=smooth, alpha_t=0.1, block_start=True, mask_id=V - 1)

    def one_step(c=0):
        ctx.step(hid, Wd[c], Ed[c], emd, mask, tokens, cids if credit else None, cval if credit else None, p,
                 committed, smoothed, stats)

    def block_start_step(c=0):  # a block's first iteration: the state inputs are not read (params.block_start)
        ctx.step(hid, Wd[c], Ed[c], emd, mask, tokens, cids if credit else None, cval if credit else None, p_bs,
                 committed, smoothed, stats)

    # calibrated vocab partition (K12): measured per-SM streaming rates -> slab split
    partition = "even"
    if args.balance and smooth:
        from paper_2510_08666_b200 import DInferError
        try:
            ctx.balance(hid, Wd[0], Ed[0], emd, p, iters=4, mode="back_to_back")
            partition = default_partition(True)
        except DInferError:
            pass
    # warm-up: every kernel of every timed loop runs here first (CUDA loads
    # modules lazily on first launch: a first launch inside a timed loop would
    # be charged to it), the back-to-back sequence W times, then W flushed steps
    for i in range(max(args.warmup, R)):
        block_start_step(i % R)
    for _ in range(args.warmup):
        reset_and_flush()
        one_step()
    ctx.sync()
    torch.cuda.synchronize()
    # the same back-to-back steps as one CUDA graph (R steps per replay)
    graph = None
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for c in range(R):
                block_start_step(c)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001 -- reported, not fatal
        print(f"[bench] graph capture failed: {e}", file=sys.stderr)
        graph = None

    # ---- timed region.
    # Loop A (headline): K back-to-back steps, each a block's first iteration
    # (params.block_start: all positions undecided, credit slots empty), bracketed
    # by one event pair, rotating over R weight copies (R x shard >= 3x L2).
    # Loop A2: the same K steps one at a time with L2 flushed before each
    # (outside the events): no overlap with the previous step.
    # Loop A3: the steps replayed from one CUDA graph.
    # Loop B: as A with the library's per-kernel events on (these serialise the
    # PDL overlap between kernels, so B's per-kernel times are upper bounds)
    # and a stream sync per step to read them -> roofline per kernel.
    ea = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    eg = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    evb = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phase_acc = {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    wall0 = time.perf_counter()
    n_graph = 0
    with sampler:
        ea[0].record(stream)
        for i in range(args.steps):
            block_start_step(i % R)
        ea[1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        for i in range(args.steps):
            reset_and_flush()
            evs[i][0].record(stream)
            one_step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        if graph is not None:
            reps = max(1, args.steps // R)
            eg[0].record(stream)
            with torch.cuda.stream(stream):
                for _ in range(reps):
                    graph.replay()
            eg[1].record(stream)
            n_graph = reps * R
            torch.cuda.synchronize()
        ctx.set_timing(True)
        for i in range(args.steps):
            evb[i][0].record(stream)
            block_start_step(i % R)
            evb[i][1].record(stream)
            ph = ctx.get_timing()  # syncs the stream (outside the event pair)
            for k_, v_ in ph.items():
                phase_acc[k_] = phase_acc.get(k_, 0.0) + v_
        ctx.set_timing(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ctx.sync()
    ms = ea[0].elapsed_time(ea[1]) / args.steps
    ms_graph = eg[0].elapsed_time(eg[1]) / n_graph if n_graph else float("nan")
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms_fl = sum(step_ms) / len(step_ms)
    ms_b = sum(a.elapsed_time(b) for a, b in evb) / len(evb)
    phases = {k_: v_ / args.steps for k_, v_ in phase_acc.items()}
    if world > 1:
        t = torch.tensor([ms, ms_fl, ms_b, ms_graph] + [phases[k_] for k_ in sorted(phases)], dtype=torch.float64,
                         device="cpu" if same_dev else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_fl, ms_b, ms_graph = float(t[0]), float(t[1]), float(t[2]), float(t[3])
        for j, k_ in enumerate(sorted(phases)):
            phases[k_] = float(t[4 + j])

    # ---- e2e: the public host-buffer call (H2D of hidden + state, D2H of state + outputs)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hid_h = pin(hid_u16.view(np.int16))
    mask_h, tok_h = pin(np.ones((B, S), np.uint8)), pin(np.full((B, S), V - 1, np.int32))
    cids_h, cval_h = pin(np.full((B, S, K), -1, np.int32)), pin(np.zeros((B, S, K), np.float32))
    com_h, st_h = pin(np.zeros((B, S), np.uint8)), pin(np.zeros((B, S, 4), np.float32))
    sm_h = pin(np.zeros((B, S, H), np.float32)) if smooth else None
    # dinfer_step_host's packed state block (include/dinfer.h): params(32 B) | mask | tokens |
    # credit ids | credit values | committed | stats; uploaded up to `committed`, read back whole
    al = lambda x: (x + 15) & ~15
    o_com = al(32 + M) + 4 * M + 8 * M * K
    h2d = M * H * 2 + o_com
    d2h = al(o_com + M) + 16 * M + (4 * M * H if smooth else 0)
    e2e_steps = max(3, min(args.steps, 50))
    e2e_ms = []
    for i in range(args.warmup + e2e_steps):
        # a new block each call (host state reset)
        mask_h.fill_(1); tok_h.fill_(V - 1); cids_h.fill_(-1); cval_h.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        # the public host-buffer API: copies in, step, results back in host memory
        # (e1 follows the result copies on the stream), then the unpacking wait
        ctx.step_host_async(hid_h, Wd[i % R], Ed[i % R], emd, mask_h, tok_h, cids_h if credit else None,
                            cval_h if credit else None, p, com_h, sm_h, st_h)
        e1.record(stream)
        e1.synchronize()
        ctx.step_host_wait()
        if i >= args.warmup:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e = sum(e2e_ms) / len(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cpu" if same_dev else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t[0])
    launches = ctx.launches_per_step(p)
    geom = ctx.geometry()

    if rank == 0:
        hbm, tflops, peak_kind = peaks()
        tflops_sus = peaks_sustained()
        k1_bytes = Vl * H * 2 + M * H * 2
        k2_bytes = (Vl * H * 2 + M * H * 4) if smooth else 0
        k1_ms, k2_ms = phases.get("k1_vocab_proj", 0.0), phases.get("k2_smooth_mix", 0.0)
        if smooth and geom.get("fused"):  # K12: W and E streams in one kernel (timed in the K1 phase slot)
            dom, dom_bytes, dom_ms = "k12_proj_smooth", k1_bytes + k2_bytes, k1_ms
        else:
            dom, dom_bytes, dom_ms = ("k1_vocab_proj", k1_bytes, k1_ms) if k1_ms >= k2_ms else \
                ("k2_smooth_mix", k2_bytes, k2_ms)
        shards = args.shard_sim or world  # traffic captures of a vocab shard are keyed "<config>-g<G>"
        tkey = CFG["name"] + (f"-g{shards}" if shards > 1 else "")
        traffic = ncu_traffic().get(f"{tkey}/" + (dom if M <= 256 else "k1b_vocab_proj_dense"))
        step_bytes = k1_bytes + k2_bytes
        if M > 256:  # compute-bound regime (BASELINE configs[4]): tensor roofline of K1b
            flops = 2.0 * M * H * Vl
            achieved = flops / (dom_ms * 1e-3) / 1e12
            roof = {"bound": "tensor", "kernel": "k1b_vocab_proj_dense", "achieved": achieved, "peak": tflops_sus,
                    "unit": "TFLOP/s", "frac": achieved / tflops_sus, "traffic": traffic, "peak_kind":
                    peak_kind + " sustained (kernel timed inside a ms-long step)", "burst_peak": tflops,
                    "algorithmic_flops_per_launch": flops, "ms_per_launch": dom_ms}
        else:
            achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
            roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                    "algorithmic_bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms}
        cpu = None
        if world == 1 and not args.no_cpu_baseline and not args.shard_sim:
            rows = 8
            times, cores = oracle_run(100, 1, rows, budget_s=args.cpu_budget)
            sec = sum(times) / len(times)
            times1, _ = oracle_run(100, 0, rows, budget_s=args.cpu_budget / 2, threads=1)
            sec1 = sum(times1) / len(times1)
            cpu = {"value": rows / sec, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{len(times)} oracle steps of {rows} of {B * S} positions (full vocab {V}, fp64 numpy; "
                             f"{sum(times):.1f} s of CPU work)",
                   "one_thread": {"value": rows / sec1, "unit": UNIT, "cores": 1,
                                  "sample": f"{len(times1)} oracle steps of {rows} positions, BLAS limited to 1 "
                                            f"thread ({sum(times1):.1f} s)"}}
        value = M / (ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": bench_config(world, Vl, exchange, partition, R, args.shard_sim),
            "e2e": {"value": M / (e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e, "api": "dinfer_step_host_async + dinfer_step_host_wait",
                    "timing": "per call: CUDA events around the call's copies + kernels on the ctx stream, "
                              "host wait between calls"},
            "gpu_launches": launches * args.steps,
            "roofline": roof,
            "step_roofline": None if M > 256 else {"bytes": step_bytes, "achieved_gbs": step_bytes / (ms * 1e-3) / 1e9,
                              "frac": step_bytes / (ms * 1e-3) / 1e9 / hbm},
            "phases_ms": phases,
            "l2_flushed": {"ms_per_step": ms_fl, "value": M / (ms_fl * 1e-3),
                           "note": "the same steps one at a time, L2 flushed (256 MiB write) before each, "
                                   "per-step event pairs (no overlap with the previous step)",
                           "ms_per_step_min": min(step_ms), "ms_per_step_max": max(step_ms),
                           "ms_per_step_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)]},
            "graph_replay": None if not n_graph else {
                "ms_per_step": ms_graph, "value": M / (ms_graph * 1e-3),
                "note": f"the back-to-back block-start steps captured once into a CUDA graph ({R} per graph), "
                        f"{n_graph} steps replayed under one event pair"},
            "ms_per_step_with_kernel_events": ms_b,
            "geometry": geom,
            "clocks": sampler.report(),
            "wall_s_timed_loop": wall,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--config", default="moe", choices=sorted(CONFIGS))
    ap.add_argument("--balance", action="store_true",
                    help="calibrate the K12 vocab partition first (dinfer_balance); the default even partition "
                         "measured as fast or faster with the round-2 W tiles (214.0-215.0 vs 215.1-216.2 us)")
    ap.add_argument("--no-balance", action="store_true", help="(default; kept for old command lines)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "p2p", "nccl"],
                    help="N>1 record exchange: peer memory (auto: if every rank can open it) or NCCL allgather")
    ap.add_argument("--shard-sim", type=int, default=0, choices=[0, 2, 4, 8],
                    help="measurement: one rank of a G-way vocab shard on one GPU (loopback exchange)")
    args = ap.parse_args()
    set_config(args.config)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
