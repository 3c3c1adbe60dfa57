"""C-ABI library checks that need no GPU: libdinfer.so loads, exports every
symbol include/dinfer.h declares, validates shapes synchronously, and its host
schedule helpers agree with the oracle's schedules."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from paper_2510_08666_b200 import build, dinfer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return dinfer.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dinfer.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dinfer_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("dinfer_create", "dinfer_step", "dinfer_step_host", "dinfer_step_local", "dinfer_step_combine",
                 "dinfer_credit_reset", "dinfer_alpha_schedule", "dinfer_tau_schedule", "dinfer_sync",
                 "dinfer_destroy", "dinfer_strerror", "dinfer_get_unique_id"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    for name in declared_functions():
        assert hasattr(L, name), name


def test_library_is_sm100a_with_tcgen05_and_tma():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", dinfer.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in out, mnem


def test_kernels_do_not_spill():
    """Every kernel keeps its state in registers: no local-memory stack (a
    spill is a dependent L1/L2 round trip on the latency-bound K34 path)."""
    import re
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", dinfer.LIB_PATH], capture_output=True,
                         text=True).stdout
    funcs = re.findall(r"Function (\S+):\n\s*REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
    assert len(funcs) >= 5, out[:500]
    for name, reg, stack, local in funcs:
        assert int(stack) == 0 and int(local) == 0, (name, reg, stack, local)


def test_schedules_match_oracle(L):
    for t in range(12):
        assert dinfer.alpha_schedule(0.1, 0.05, 0.3, t) == pytest.approx(O.alpha_schedule(0.1, 0.05, 0.3, t), abs=1e-7)
        for D in (0, 1, 4, 7):
            assert dinfer.tau_schedule(0.8, t, D) == pytest.approx(O.tau_schedule(0.8, t, D), abs=1e-7)


def _create(L, **kw):
    shp = dict(B=1, S=32, H=256, K=8, V_total=1024, V_local=1024, v_offset=0, world=1, rank=0, smooth_capable=1)
    shp.update(kw)
    s = dinfer.Shape(*[shp[n] for n, _ in dinfer.Shape._fields_])
    h = ctypes.c_void_p()
    return L.dinfer_create(ctypes.byref(s), None, None, ctypes.byref(h))


@pytest.mark.parametrize("bad", [dict(H=200), dict(V_local=1020, V_total=1020), dict(S=0), dict(K=0),
                                 dict(world=2, V_total=1024), dict(rank=1), dict(S=2000)])
def test_create_rejects_bad_shapes_synchronously(L, bad):
    assert _create(L, **bad) == 2  # DINFER_ERR_SHAPE, before touching the device


def test_create_rejects_large_M(L):
    assert _create(L, B=64, S=64) == 6  # UNSUPPORTED: M > 256 (compute-bound regime not in this path)


def test_null_args(L):
    assert L.dinfer_create(None, None, None, None) == 1
    assert L.dinfer_step(None, *([None] * 12)) == 1
    assert L.dinfer_sync(None) == 1
    assert L.dinfer_strerror(0) == b"ok"


def test_kv_region_helper_matches_oracle(L):
    """The host refresh-region helper of the vicinity KV cache (f3) against the
    oracle's refresh_region, incl. warmup, clipping and full refresh."""
    import ctypes
    from paper_2510_08666_b200.dinfer import KvShape
    rng = np.random.default_rng(5)
    for _ in range(200):
        Ls = int(rng.integers(32, 400))
        pre, aft, warm = (int(x) for x in rng.integers(0, 40, 3))
        start = int(rng.integers(0, Ls - 1)); end = int(rng.integers(start + 1, Ls + 1))
        t = int(rng.integers(0, 8)); full = bool(rng.random() < 0.2)
        s = KvShape(Ls, 256, 128, pre, aft, warm % 6)
        lo, hi = ctypes.c_int32(), ctypes.c_int32()
        n = L.dinfer_kv_region(ctypes.byref(s), start, end, t, int(full), ctypes.byref(lo), ctypes.byref(hi))
        want = O.refresh_region(Ls, start, end, t, pre, aft, warm % 6, full)
        assert (lo.value, hi.value) == want and n == want[1] - want[0]


def test_binding_rejects_bad_tensors_before_the_abi():
    """The ctypes binding checks dtype, contiguity, device and element count
    against the ctx shape before handing bare pointers to the C ABI (ADVICE
    r1): a wrong buffer must raise, not become silent garbage."""
    import torch
    from paper_2510_08666_b200.dinfer import _dt, _expect
    d = _dt()
    _expect(torch.zeros(64, dtype=torch.int32), "tokens", d["i32"], 64, "cpu")
    with pytest.raises(TypeError):
        _expect(torch.zeros(64, dtype=torch.int64), "tokens", d["i32"], 64, "cpu")
    with pytest.raises(ValueError):
        _expect(torch.zeros(63, dtype=torch.int32), "tokens", d["i32"], 64, "cpu")
    with pytest.raises(ValueError):
        _expect(torch.zeros(8, 16, dtype=torch.int32).t(), "tokens", d["i32"], 128, "cpu")
    with pytest.raises(ValueError):
        _expect(torch.zeros(64, dtype=torch.int32), "tokens", d["i32"], 64, "cuda")
    _expect(torch.zeros(70, dtype=torch.float32), "records", d["f32"], 64, "cpu", at_least=True)
    with pytest.raises(TypeError):
        _expect(np.zeros(64, np.int32), "tokens", d["i32"], 64, "cpu")
    _expect(None, "E", d["bf16"], 10, "cuda")


def test_params_struct_matches_header():
    """dinfer_params field order / count in the binding equals include/dinfer.h."""
    src = open(os.path.join(ROOT, "include", "dinfer.h")).read()
    body = re.search(r"typedef struct \{([^}]*)\} dinfer_params;", src).group(1)
    names = re.findall(r"(\w+)\s*[,;]", re.sub(r"/\*.*?\*/", "", body, flags=re.S))
    assert names == [n for n, _ in dinfer.Params._fields_]


def test_library_links_no_cublas():
    """Every contraction of the path (vocab projection, smoothing mix, the
    vicinity layer's projections and attention) is a hand-written tcgen05
    kernel: libdinfer.so has no cuBLAS dependency."""
    import subprocess
    build.build()
    out = subprocess.run(["readelf", "-d", dinfer.LIB_PATH], capture_output=True, text=True).stdout
    assert "NEEDED" in out and "cublas" not in out.lower(), out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", dinfer.LIB_PATH], capture_output=True,
                          text=True).stdout
    fn = [blk for blk in sass.split("Function : ") if blk.split("\n")[0].find("kv_proj_tc") >= 0]
    assert len(fn) == 1 and "UTCHMMA" in fn[0] and "UTMALDG" in fn[0]
