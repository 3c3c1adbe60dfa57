"""Thin ctypes binding of libdinfer.so (include/dinfer.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  torch tensors are passed by data pointer; torch is used for device
memory, streams and torch.distributed (plumbing).  There is no CPU fallback:
if libdinfer.so is missing, importing the binding's entry points raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_float, c_int32, c_int64, c_size_t, c_uint8, c_uint16, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdinfer.so")
if os.environ.get("DINFER_LIB"):  # measurement only: A/B against another in-tree build (tools/ab_lib.sh)
    LIB_PATH = os.path.abspath(os.environ["DINFER_LIB"])

DEC_THRESHOLD = 0
DEC_HIERARCHICAL = 1
PHASES = ("k1_vocab_proj", "k2_smooth_mix", "rec_finalize", "c1_allgather", "k34_select_smooth", "unused")

STATUS = {0: "ok", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_CUDA", 4: "ERR_NCCL", 5: "ERR_NOMEM",
          6: "ERR_UNSUPPORTED", 7: "ERR_DEVICE"}


class DInferError(RuntimeError):
    def __init__(self, status: int, what: str):
        detail = lib().dinfer_last_error().decode() if status in (3, 4) else ""
        super().__init__(f"{what}: {STATUS.get(status, status)} ({lib().dinfer_strerror(status).decode()})"
                         + (f" [{detail}]" if detail else ""))
        self.status = status


class Shape(ctypes.Structure):
    _fields_ = [("B", c_int32), ("S", c_int32), ("H", c_int32), ("K", c_int32), ("V_total", c_int64),
                ("V_local", c_int64), ("v_offset", c_int64), ("world", c_int32), ("rank", c_int32),
                ("smooth_capable", c_int32)]


class Params(ctypes.Structure):
    _fields_ = [("decoder", c_int32), ("tau", c_float), ("theta_hi", c_float), ("theta_lo", c_float),
                ("hier_runs_after_hi", c_int32), ("use_credit", c_int32), ("c_alpha", c_float),
                ("c_beta", c_float), ("c_gamma", c_float), ("use_smooth", c_int32), ("alpha_t", c_float),
                ("smooth_credit_fused", c_int32), ("block_start", c_int32), ("mask_id", c_int32),
                ("inclusive", c_int32)]


class GenConfig(ctypes.Structure):
    """dinfer_gen_config (include/dinfer.h): the block loop of Algorithm 1."""
    _fields_ = [("L", c_int32), ("prompt_len", c_int32), ("mask_id", c_int32), ("eos_id", c_int32),
                ("early_termination", c_int32), ("tau_target", c_float), ("tau_decay_steps", c_int32),
                ("alpha_init", c_float), ("alpha_growth", c_float), ("alpha_preset", c_float),
                ("max_forwards", c_int32)]


def make_gen_config(L, prompt_len, mask_id, eos_id, early_termination=True, tau_target=0.9, tau_decay_steps=0,
                    alpha_init=0.1, alpha_growth=0.05, alpha_preset=0.3, max_forwards=1 << 30) -> GenConfig:
    return GenConfig(int(L), int(prompt_len), int(mask_id), int(eos_id), int(bool(early_termination)),
                     float(tau_target), int(tau_decay_steps), float(alpha_init), float(alpha_growth),
                     float(alpha_preset), int(max_forwards))


class Geometry(ctypes.Structure):
    _fields_ = [(n, c_int32) for n in ("k1_grid", "k1_stages", "k1_h_resident", "k1_smem", "k2_grid", "k2_hw",
                                        "k2_groups", "k2_stages", "k2_smem", "num_sms", "fused",
                                        "fused_smem")]


class KvShape(ctypes.Structure):
    """dinfer_kv_shape (include/dinfer.h): vicinity KV-cache refresh layer."""
    _fields_ = [(n, c_int32) for n in ("L", "H", "d_head", "prefix_look", "after_look", "warmup_times")]


_LIB = None


def lib():
    """Load libdinfer.so (raises if it was not built -- no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built (python -m paper_2510_08666_b200.build)")
    L = ctypes.CDLL(LIB_PATH)
    P, S = c_void_p, c_int32
    sig = {
        "dinfer_get_unique_id": (S, [P]),
        "dinfer_create": (S, [POINTER(Shape), P, P, POINTER(c_void_p)]),
        "dinfer_destroy": (None, [P]),
        "dinfer_set_stream": (S, [P, P]),
        "dinfer_step": (S, [P, P, P, P, P, P, P, P, P, POINTER(Params), P, P, P]),
        "dinfer_step_host": (S, [P, P, P, P, P, P, P, P, P, POINTER(Params), P, P, P]),
        "dinfer_step_embed": (S, [P, P, P, P, P, P, P, P, P, POINTER(Params), P, P, P, P]),
        "dinfer_step_host_async": (S, [P, P, P, P, P, P, P, P, P, POINTER(Params), P, P, P]),
        "dinfer_step_host_wait": (S, [P]),
        "dinfer_record_words": (c_size_t, [P, S]),
        "dinfer_step_local": (S, [P, P, P, P, P, P, POINTER(Params), P]),
        "dinfer_step_combine": (S, [P, P, P, P, P, P, P, POINTER(Params), P, P, P]),
        "dinfer_credit_reset": (S, [P, P, P]),
        "dinfer_block_reset": (S, [P, P, P, P, P, S]),
        "dinfer_alpha_schedule": (c_float, [c_float, c_float, c_float, S]),
        "dinfer_tau_schedule": (c_float, [c_float, S, S]),
        "dinfer_sync": (S, [P]),
        "dinfer_strerror": (ctypes.c_char_p, [S]),
        "dinfer_last_error": (ctypes.c_char_p, []),
        "dinfer_set_timing": (S, [P, S]),
        "dinfer_get_timing": (S, [P, POINTER(c_float), S]),
        "dinfer_launches_per_step": (S, [P, POINTER(Params)]),
        "dinfer_get_geometry": (S, [P, POINTER(Geometry)]),
        "dinfer_get_trace": (S, [P, P, S]),
        "dinfer_generate": (S, [P, POINTER(GenConfig), POINTER(Params), P, P, P, P, c_int64, P, P]),
        "dinfer_balance": (S, [P, P, P, P, P, POINTER(Params), S, S]),
        "dinfer_balance_reset": (S, [P]),
        "dinfer_exchange_handle": (S, [P, P]),
        "dinfer_exchange_open": (S, [P, P]),
        "dinfer_exchange_loopback": (S, [P]),
        "dinfer_kv_create": (S, [POINTER(KvShape), P, POINTER(c_void_p)]),
        "dinfer_kv_destroy": (None, [P]),
        "dinfer_kv_region": (S, [POINTER(KvShape), S, S, S, S, POINTER(c_int32), POINTER(c_int32)]),
        "dinfer_kv_step": (S, [P, P, P, P, P, P, P, S, S, S, S, P, POINTER(c_int32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    _LIB = L
    return L


def _ptr(t):
    if t is None:
        return None
    return c_void_p(t.data_ptr())


def _expect(t, name: str, dtypes, numel: int, device: str, at_least: bool = False):
    """Argument marshalling guard: the C ABI takes bare pointers and cannot
    check sizes, so a wrong dtype, a strided view, the wrong device or a short
    buffer would be silent garbage or an out-of-bounds device access.  None is
    passed through (the library checks which pointers may be NULL)."""
    if t is None:
        return
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype not in dtypes:
        raise TypeError(f"{name}: dtype {t.dtype}, expected one of {[str(d) for d in dtypes]}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if t.numel() < numel or (t.numel() != numel and not at_least):
        raise ValueError(f"{name}: {t.numel()} elements, expected {'at least ' if at_least else ''}{numel}")
    if device == "cuda" and not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if device == "cpu" and t.is_cuda:
        raise ValueError(f"{name}: must be a host (CPU) tensor")


def _dt():
    import torch
    return dict(bf16=(torch.bfloat16, torch.int16), u8=(torch.uint8, torch.bool), i32=(torch.int32,),
                f32=(torch.float32,))


def _check(status: int, what: str):
    if status != 0:
        raise DInferError(status, what)


def make_params(decoder=DEC_THRESHOLD, tau=0.9, theta_hi=0.92, theta_lo=0.62, hier_runs_after_hi=False,
                use_credit=False, c_alpha=1.0, c_beta=0.9, c_gamma=0.5, use_smooth=False, alpha_t=0.1,
                smooth_credit_fused=False, block_start=False, mask_id=0, inclusive=False) -> Params:
    if isinstance(decoder, str):
        decoder = {"threshold": DEC_THRESHOLD, "hierarchical": DEC_HIERARCHICAL}[decoder]
    return Params(int(decoder), float(tau), float(theta_hi), float(theta_lo), int(bool(hier_runs_after_hi)),
                  int(bool(use_credit)), float(c_alpha), float(c_beta), float(c_gamma), int(bool(use_smooth)),
                  float(alpha_t), int(bool(smooth_credit_fused)), int(bool(block_start)), int(mask_id),
                  int(bool(inclusive)))


def alpha_schedule(init: float, growth: float, preset: float, t: int) -> float:
    return float(lib().dinfer_alpha_schedule(init, growth, preset, int(t)))


def tau_schedule(target: float, t: int, decay_steps: int) -> float:
    return float(lib().dinfer_tau_schedule(target, int(t), int(decay_steps)))


def get_unique_id() -> bytes:
    buf = (c_uint8 * 128)()
    _check(lib().dinfer_get_unique_id(buf), "dinfer_get_unique_id")
    return bytes(buf)


class Context:
    """One dInfer step context (workspace + stream [+ NCCL communicator])."""

    def __init__(self, B: int, S: int, H: int, K: int, V_total: int, V_local: int | None = None,
                 v_offset: int = 0, world: int = 1, rank: int = 0, smooth_capable: bool = True,
                 stream=None, nccl_id: bytes | None = None):
        V_local = V_total // world if V_local is None else V_local
        self.shape = Shape(B, S, H, K, V_total, V_local, v_offset, world, rank, int(bool(smooth_capable)))
        if stream is None:
            import torch
            stream = torch.cuda.current_stream().cuda_stream
        self._stream = stream
        idbuf = None if nccl_id is None else (c_uint8 * 128).from_buffer_copy(nccl_id)
        h = c_void_p()
        _check(lib().dinfer_create(ctypes.byref(self.shape), idbuf, c_void_p(stream), ctypes.byref(h)),
               "dinfer_create")
        self._h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            lib().dinfer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_step(self, dev, hidden, W, E, e_mask, mask, tokens, credit_ids, credit_val, committed, smoothed,
                    stats, emb=None):
        d = _dt()
        sh = self.shape
        M = sh.B * sh.S
        _expect(hidden, "hidden", d["bf16"], M * sh.H, dev)
        _expect(W, "W_vocab", d["bf16"], sh.V_local * sh.H, "cuda")
        _expect(E, "E", d["bf16"], sh.V_local * sh.H, "cuda")
        _expect(e_mask, "e_mask", d["bf16"], sh.H, "cuda")
        _expect(mask, "mask", d["u8"], M, dev)
        _expect(tokens, "tokens", d["i32"], M, dev)
        _expect(credit_ids, "credit_ids", d["i32"], M * sh.K, dev)
        _expect(credit_val, "credit_val", d["f32"], M * sh.K, dev)
        _expect(committed, "committed", d["u8"], M, dev)
        _expect(smoothed, "smoothed", d["f32"], M * sh.H, dev)
        _expect(stats, "stats", d["f32"], M * 4, dev)
        _expect(emb, "emb", d["bf16"], M * sh.H, "cuda")

    def set_stream(self, stream):
        self._stream = stream
        _check(lib().dinfer_set_stream(self._h, c_void_p(stream)), "dinfer_set_stream")

    # -- the step
    def step(self, hidden, W, E, e_mask, mask, tokens, credit_ids, credit_val, params: Params, committed,
             smoothed=None, stats=None):
        self._check_step("cuda", hidden, W, E, e_mask, mask, tokens, credit_ids, credit_val, committed, smoothed,
                         stats)
        _check(lib().dinfer_step(self._h, _ptr(hidden), _ptr(W), _ptr(E), _ptr(e_mask), _ptr(mask), _ptr(tokens),
                                 _ptr(credit_ids), _ptr(credit_val), ctypes.byref(params), _ptr(committed),
                                 _ptr(smoothed), _ptr(stats)), "dinfer_step")

    BALANCE_MODES = {"after_forward": 0, "back_to_back": 1}

    def balance(self, hidden, W, E, e_mask, params: Params, iters: int = 4, mode: str = "after_forward"):
        """Calibrate the K12 vocab partition to this GPU's per-SM rates
        (dinfer_balance) for steps that follow a model forward
        ("after_forward") or each other directly ("back_to_back")."""
        self._check_step("cuda", hidden, W, E, e_mask, None, None, None, None, None, None, None)
        _check(lib().dinfer_balance(self._h, _ptr(hidden), _ptr(W), _ptr(E), _ptr(e_mask), ctypes.byref(params),
                                    int(iters), self.BALANCE_MODES[mode]), "dinfer_balance")

    def balance_reset(self):
        _check(lib().dinfer_balance_reset(self._h), "dinfer_balance_reset")

    def exchange_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's gather buffer (peer-memory exchange)."""
        buf = (ctypes.c_uint8 * 64)()
        _check(lib().dinfer_exchange_handle(self._h, buf), "dinfer_exchange_handle")
        return bytes(buf)

    def exchange_open(self, handles: bytes):
        """Open every rank's gather buffer (world x 64 bytes, rank order): dinfer_step
        then exchanges the records over peer memory instead of NCCL."""
        buf = (ctypes.c_uint8 * len(handles)).from_buffer_copy(handles)
        _check(lib().dinfer_exchange_open(self._h, buf), "dinfer_exchange_open")

    def exchange_loopback(self):
        """Measurement only: run as one rank of a `world`-way shard on one GPU
        (records stored into all of this GPU's own slots; results not meaningful)."""
        _check(lib().dinfer_exchange_loopback(self._h), "dinfer_exchange_loopback")

    def step_embed(self, hidden, W, E, e_mask, mask, tokens, credit_ids, credit_val, params: Params, committed,
                   smoothed, stats, emb):
        """dinfer_step + the next iteration's bf16 input embedding `emb` [B,S,H]."""
        self._check_step("cuda", hidden, W, E, e_mask, mask, tokens, credit_ids, credit_val, committed, smoothed,
                         stats, emb)
        _check(lib().dinfer_step_embed(self._h, _ptr(hidden), _ptr(W), _ptr(E), _ptr(e_mask), _ptr(mask),
                                       _ptr(tokens), _ptr(credit_ids), _ptr(credit_val), ctypes.byref(params),
                                       _ptr(committed), _ptr(smoothed), _ptr(stats), _ptr(emb)), "dinfer_step_embed")

    def block_reset(self, mask, tokens, credit_ids, credit_val, mask_id: int):
        """Block start on the device (mask = 1, tokens = mask_id, credit slots empty)."""
        _check(lib().dinfer_block_reset(self._h, _ptr(mask), _ptr(tokens), _ptr(credit_ids), _ptr(credit_val),
                                        int(mask_id)), "dinfer_block_reset")

    def step_host_async(self, hidden_h, W, E, e_mask, mask_h, tokens_h, credit_ids_h, credit_val_h, params: Params,
                        committed_h, smoothed_h=None, stats_h=None):
        """dinfer_step_host without the final wait (see step_host_wait)."""
        self._check_step("cpu", hidden_h, W, E, e_mask, mask_h, tokens_h, credit_ids_h, credit_val_h, committed_h,
                         smoothed_h, stats_h)
        self._pending = (hidden_h, mask_h, tokens_h, credit_ids_h, credit_val_h, committed_h, smoothed_h, stats_h)
        _check(lib().dinfer_step_host_async(self._h, _ptr(hidden_h), _ptr(W), _ptr(E), _ptr(e_mask), _ptr(mask_h),
                                            _ptr(tokens_h), _ptr(credit_ids_h), _ptr(credit_val_h),
                                            ctypes.byref(params), _ptr(committed_h), _ptr(smoothed_h),
                                            _ptr(stats_h)), "dinfer_step_host_async")

    def step_host_wait(self):
        _check(lib().dinfer_step_host_wait(self._h), "dinfer_step_host_wait")
        self._pending = None

    def step_host(self, hidden_h, W, E, e_mask, mask_h, tokens_h, credit_ids_h, credit_val_h, params: Params,
                  committed_h, smoothed_h=None, stats_h=None):
        self._check_step("cpu", hidden_h, W, E, e_mask, mask_h, tokens_h, credit_ids_h, credit_val_h, committed_h,
                         smoothed_h, stats_h)
        _check(lib().dinfer_step_host(self._h, _ptr(hidden_h), _ptr(W), _ptr(E), _ptr(e_mask), _ptr(mask_h),
                                      _ptr(tokens_h), _ptr(credit_ids_h), _ptr(credit_val_h), ctypes.byref(params),
                                      _ptr(committed_h), _ptr(smoothed_h), _ptr(stats_h)), "dinfer_step_host")

    def generate(self, cfg: GenConfig, base: Params, W, E, e_mask, hidden_src, X, out):
        """Device-resident block loop (Alg. 1) over X [B, L] int32; hidden_src
        [iters, B*S, H] bf16 is the model stand-in; out int32 [B + 2] receives
        T_b, F, truncated.  Asynchronous on the ctx stream."""
        iters = int(hidden_src.shape[0])
        d, sh = _dt(), self.shape
        _expect(hidden_src, "hidden_src", d["bf16"], iters * sh.B * sh.S * sh.H, "cuda")
        _expect(X, "X", d["i32"], sh.B * int(cfg.L), "cuda")
        _expect(out, "out", d["i32"], sh.B + 2, "cuda")
        _expect(W, "W_vocab", d["bf16"], sh.V_local * sh.H, "cuda")
        _expect(E, "E", d["bf16"], sh.V_local * sh.H, "cuda")
        _expect(e_mask, "e_mask", d["bf16"], sh.H, "cuda")
        _check(lib().dinfer_generate(self._h, ctypes.byref(cfg), ctypes.byref(base), _ptr(W), _ptr(E), _ptr(e_mask),
                                     _ptr(hidden_src), iters, _ptr(X), _ptr(out)), "dinfer_generate")

    def record_words(self, use_smooth: bool) -> int:
        return int(lib().dinfer_record_words(self._h, int(bool(use_smooth))))

    def step_local(self, hidden, W, E, mask, credit_ids, params: Params, record):
        self._check_step("cuda", hidden, W, E, None, mask, None, credit_ids, None, None, None, None)
        _expect(record, "record", _dt()["f32"], self.record_words(bool(params.use_smooth)), "cuda", at_least=True)
        _check(lib().dinfer_step_local(self._h, _ptr(hidden), _ptr(W), _ptr(E), _ptr(mask), _ptr(credit_ids),
                                       ctypes.byref(params), _ptr(record)), "dinfer_step_local")

    def step_combine(self, records, e_mask, mask, tokens, credit_ids, credit_val, params: Params, committed,
                     smoothed=None, stats=None):
        self._check_step("cuda", None, None, None, e_mask, mask, tokens, credit_ids, credit_val, committed, smoothed,
                         stats)
        _expect(records, "records", _dt()["f32"], self.shape.world * self.record_words(bool(params.use_smooth)),
                "cuda", at_least=True)
        _check(lib().dinfer_step_combine(self._h, _ptr(records), _ptr(e_mask), _ptr(mask), _ptr(tokens),
                                         _ptr(credit_ids), _ptr(credit_val), ctypes.byref(params),
                                         _ptr(committed), _ptr(smoothed), _ptr(stats)), "dinfer_step_combine")

    def credit_reset(self, credit_ids, credit_val):
        _check(lib().dinfer_credit_reset(self._h, _ptr(credit_ids), _ptr(credit_val)), "dinfer_credit_reset")

    def sync(self):
        _check(lib().dinfer_sync(self._h), "dinfer_sync")

    # -- instrumentation
    def set_timing(self, enable: bool):
        _check(lib().dinfer_set_timing(self._h, int(bool(enable))), "dinfer_set_timing")

    def get_timing(self) -> dict:
        buf = (c_float * len(PHASES))()
        _check(lib().dinfer_get_timing(self._h, buf, len(PHASES)), "dinfer_get_timing")
        return {n: float(v) for n, v in zip(PHASES, buf)}

    def launches_per_step(self, params: Params) -> int:
        return int(lib().dinfer_launches_per_step(self._h, ctypes.byref(params)))

    def trace(self):
        """Per-CTA globaltimer stamps of the last step (DINFER_TRACE=1), as
        (k1 [grid,5], k2 [grid,5], k34 [64,5]) numpy arrays (4 stamps in ns + SM id; K34
        blocks that did not run stay 0), or None."""
        import numpy as np
        n = int(lib().dinfer_get_trace(self._h, None, 0))
        if n == 0:
            return None
        buf = np.zeros(n, dtype=np.uint64)
        lib().dinfer_get_trace(self._h, c_void_p(buf.ctypes.data), n)
        g = self.geometry()
        n1, n2 = 5 * g["k1_grid"], 5 * g["k2_grid"]
        k1 = buf[:n1].reshape(-1, 5)
        k2 = buf[n1:n1 + n2].reshape(-1, 5)
        k34 = buf[n1 + n2:n1 + n2 + 5 * 64].reshape(-1, 5)
        return k1, k2, k34  # K1, K2, K34 (first 64 blocks)

    def geometry(self) -> dict:
        g = Geometry()
        _check(lib().dinfer_get_geometry(self._h, ctypes.byref(g)), "dinfer_get_geometry")
        return {n: getattr(g, n) for n, _ in Geometry._fields_}


class VicinityKV:
    """Vicinity KV-cache refresh on a synthetic attention layer (dinfer_kv_*):
    marshalling only."""

    def __init__(self, L, H, d_head=128, prefix_look=16, after_look=16, warmup_times=4, stream=None):
        self.shape = KvShape(L, H, d_head, prefix_look, after_look, warmup_times)
        h = c_void_p()
        _check(lib().dinfer_kv_create(ctypes.byref(self.shape), c_void_p(stream) if stream else None,
                                      ctypes.byref(h)), "dinfer_kv_create")
        self._h = h

    def region(self, start, end, t, full=False):
        lo, hi = c_int32(), c_int32()
        lib().dinfer_kv_region(ctypes.byref(self.shape), start, end, t, int(bool(full)), ctypes.byref(lo),
                               ctypes.byref(hi))
        return lo.value, hi.value

    def step(self, X, Wq, Wk, Wv, Kc, Vc, start, end, t, out, full=False):
        lohi = (c_int32 * 2)()
        _check(lib().dinfer_kv_step(self._h, _ptr(X), _ptr(Wq), _ptr(Wk), _ptr(Wv), _ptr(Kc), _ptr(Vc), start, end,
                                    t, int(bool(full)), _ptr(out), lohi), "dinfer_kv_step")
        return lohi[0], lohi[1]

    def close(self):
        if getattr(self, "_h", None):
            lib().dinfer_kv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
