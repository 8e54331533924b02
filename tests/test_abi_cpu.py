"""CPU-side checks of the boundary: the library builds for sm_100a, loads, and exports every
symbol include/hopf.h declares; host-side argument validation; the seeded generators."""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hopf.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hopf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1605_01799_b200 import build
    return build.build()


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols()
    for s in ("hopf_eval_diag", "hopf_eval_dense", "hopf_eval_union", "hopf_dense_plan_create",
              "hopf_dense_plan_destroy", "hopf_strerror"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", str(libpath)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hopf_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    L = ctypes.CDLL(str(libpath))
    for s in declared_symbols():
        assert hasattr(L, s)


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", str(libpath)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_host_validation_without_gpu(libpath):
    """Argument validation happens before any CUDA call (return codes of include/hopf.h)."""
    L = ctypes.CDLL(str(libpath))
    L.hopf_strerror.restype = ctypes.c_char_p
    L.hopf_last_error.restype = ctypes.c_char_p
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    L.hopf_eval_diag.argtypes = [i64, i32, vp, vp, vp, vp, f32, ctypes.c_int, vp, f32, i32, f32,
                                 vp, vp, vp, vp]
    assert L.hopf_eval_diag(-1, 4, None, None, None, None, 0, 0, None, 1, 10, 1e-8,
                            None, None, None, None) == -1
    assert L.hopf_eval_diag(10, 0, None, None, None, None, 0, 0, None, 1, 10, 1e-8,
                            None, None, None, None) == -1
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 7, None, 1, 10, 1e-8,
                            None, None, None, None) == -1           # unknown H
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 1, None, 1, 10, 1e-8,
                            None, None, None, None) == -1           # WL1 without w
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 0, None, -1, 10, 1e-8,
                            None, None, None, None) == -1           # lambda <= 0
    assert L.hopf_eval_diag(0, 4, None, None, None, None, 0, 0, None, 1, 10, 1e-8,
                            None, None, None, None) == 0            # M == 0: no-op
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 0, None, 1, 10, 1e-8,
                            None, None, None, None) == -1           # NULL pointers
    assert b"pointer" in L.hopf_last_error()
    assert L.hopf_strerror(-2) == b"unsupported shape"
    L.hopf_dense_plan_create.argtypes = [i32, vp, vp, f32, ctypes.POINTER(vp)]
    h = vp()
    Q = np.eye(7)
    lam = np.ones(7)
    assert L.hopf_dense_plan_create(7, Q.ctypes.data, lam.ctypes.data, 1.0, ctypes.byref(h)) == -2


def test_python_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    import paper_1605_01799_b200 as hb
    monkeypatch.setattr(hb, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(hb, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        hb.lib()


def test_generators_are_shard_invariant():
    from paper_1605_01799_b200 import inputs
    wl = inputs.config("c3", M=20000)
    X, t = inputs.points(wl)
    for r0, r1 in ((0, 1), (4095, 4097), (5000, 13000), (19999, 20000)):
        Xs, ts = inputs.points(wl, r0, r1)
        assert np.array_equal(Xs, X[r0:r1]) and np.array_equal(ts, t[r0:r1])
    assert X.dtype == np.float32 and abs(X.std() - 1.0) < 0.01
    assert t.min() >= 0.0 and t.max() <= 2.0


def test_config_laws():
    from paper_1605_01799_b200 import inputs
    c2 = inputs.config("c2")
    assert c2.n == 100 and c2.M == 10 ** 6 and c2.h == "wl1"
    assert c2.D.min() >= 0.5 and c2.D.max() <= 2.0 and c2.w.min() >= 0.5 and c2.w.max() <= 1.5
    c4 = inputs.config("c4")
    assert np.allclose(c4.Q @ c4.Q.T, np.eye(256), atol=1e-12)
    assert c4.Lam.min() >= 0.1 and c4.Lam.max() <= 10
    c5 = inputs.config("c5")
    assert c5.K == 16 and c5.n == 64 and np.all(c5.Dk >= 0.25) and np.all(c5.Dk <= 4.0)


def test_host_validation_next_entry_points(libpath):
    """NEXT entry points (union / maxh / distance / normsq / diag_A / ELL / LINF kinds): argument
    validation before any CUDA call."""
    L = ctypes.CDLL(str(libpath))
    L.hopf_last_error.restype = ctypes.c_char_p
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    L.hopf_eval_diag.argtypes = [i64, i32, vp, vp, vp, vp, f32, ctypes.c_int, vp, f32, i32, f32,
                                 vp, vp, vp, vp]
    # ELL needs w; LINF does not (NULL pointers then fail on X)
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 3, None, 1, 10, 1e-8,
                            None, None, None, None) == -1
    assert b"w is required" in L.hopf_last_error()
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 4, None, 1, 10, 1e-8,
                            None, None, None, None) == -1
    assert b"pointer" in L.hopf_last_error()
    assert L.hopf_eval_diag(10, 4, None, None, None, None, 0, 5, None, 1, 10, 1e-8,
                            None, None, None, None) == -1           # unknown H
    L.hopf_eval_normsq.argtypes = [i64, i32, vp, vp, ctypes.c_int, f32, ctypes.c_int, vp, f32, i32,
                                   f32, vp, vp, vp, vp]
    assert L.hopf_eval_normsq(10, 4, None, None, 2, 0, 0, None, 1, 10, 1e-8, None, None, None,
                              None) == -1                          # unknown J
    assert L.hopf_eval_normsq(10, 4, None, None, 0, 0, 3, None, 1, 10, 1e-8, None, None, None,
                              None) == -1                          # ELL not available
    assert L.hopf_eval_normsq(10, 600, None, None, 0, 0, 0, None, 1, 10, 1e-8, None, None, None,
                              None) == -2                          # n > 512
    assert L.hopf_eval_normsq(0, 4, None, None, 0, 0, 0, None, 1, 10, 1e-8, None, None, None,
                              None) == 0                           # M == 0
    L.hopf_eval_diag_A.argtypes = [i64, i32, vp, vp, vp, vp, f32, vp, vp, f32, i32, f32, vp, vp,
                                   vp, vp]
    assert L.hopf_eval_diag_A(10, 200, None, None, None, None, 0, None, None, 1, 10, 1e-8, None,
                              None, None, None) == -2              # n > 128
    assert L.hopf_eval_diag_A(10, 16, None, None, None, None, 0, None, None, 1, 10, 1e-8, None,
                              None, None, None) == -1              # NULL Q / Lam
    assert L.hopf_eval_diag_A(10, 16, None, None, None, None, 0, None, None, 1, 0, 1e-8, None,
                              None, None, None) == -1              # max_iter < 1
    L.hopf_eval_union.argtypes = [i64, i32, i32, vp, vp, vp, vp, vp, ctypes.c_int, vp, f32, i32,
                                  f32, vp, vp, vp, vp, vp, vp, vp]
    for h in (3, 4):   # ELL / LINF unions are not instantiated: rejected before the launch
        rc = L.hopf_eval_union(10, 8, 2, 1, 1, 1, 1, 1, h, 1, 1.0, 10, 1e-8, 1, 1, 1, None, None,
                               None, None)
        assert rc == -2, rc
    L.hopf_eval_maxh.argtypes = [i64, i32, vp, vp, vp, vp, f32, i32, vp, vp, vp, f32, i32, f32, vp,
                                 vp, vp, vp, vp]
    kinds = np.array([0, 3], np.int32)
    a = np.array([1.0, 1.0], np.float32)
    assert L.hopf_eval_maxh(10, 4, 1, 1, 1, None, 0, 2, kinds.ctypes.data, a.ctypes.data, None,
                            1.0, 10, 1e-8, 1, 1, 1, None, None) == -1   # ELL member without W
    a[1] = 0.0
    kinds[1] = 0
    assert L.hopf_eval_maxh(10, 4, 1, 1, 1, None, 0, 2, kinds.ctypes.data, a.ctypes.data, None,
                            1.0, 10, 1e-8, 1, 1, 1, None, None) == -1   # a_i <= 0


@pytest.mark.parametrize("cfg", ["c1", "c3", "c5", "t5", "t4a", "c2h", "c5d"])
def test_bench_reference_arm_contract(cfg):
    """`bench.py --impl reference` (the fp64 oracle on host cores) prints one JSON line with the
    contract's keys, on a tiny sample (no GPU needed)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--config", cfg, "--cpu-sample", "16"],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"].startswith(cfg)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
