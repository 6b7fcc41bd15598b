"""ctypes binding of the plain-C dense Alg 1 restatement (TEST INFRASTRUCTURE ONLY).

``oracle/c/rplu_oracle.c`` restates dense_pivots.py:129-209 for real float64
(and float32) residuals with the reference's sequential row-mass and CDF sums; this module
gives it the same call shape as ``rplu_oracle.eliminate_real``.  It is the
checker for the full-size configs (C3 32768^2 x 512 pivots: a fused,
row-parallel update + next-step mass pass instead of numpy's three passes
and an n x m temporary).  Built by ``oracle/Makefile``; a missing library
raises (tests that need it fail loudly rather than skip).
"""

import ctypes
import os

import numpy as np

from .rplu_oracle import uniform_stream

__all__ = ["available", "eliminate_c", "replay_c", "library_path"]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "liboracle_c.so")
_lib = None
_RULES = {"rplu": 0, "c2plu": 1, "cplu": 2}


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise RuntimeError(f"{library_path} not built (make -C oracle)")
        lib = ctypes.CDLL(library_path)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        for fn in (lib.oracle_dense_f64, lib.oracle_dense_f32):
            fn.argtypes = [P, i64, i64, i64, ctypes.c_int, P, i64, P,
                           ctypes.c_double, ctypes.c_int, P, P, P, P, P, P]
            fn.restype = ctypes.c_int
        _lib = lib
    return _lib


def available():
    return os.path.exists(library_path)


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _run(R, tag, steps, uniforms, forced, stop_tol, threads, margins):
    lib = _load()
    n, m = R.shape
    k = max(steps, 1)
    piv = np.zeros(2 * k, dtype=np.int64)
    Lt = np.zeros((k, n), dtype=R.dtype)
    U = np.zeros((k, m), dtype=R.dtype)
    resid = np.zeros(steps + 1)
    mg = np.full(k, np.inf) if margins else None
    out = np.zeros(5, dtype=np.int64)
    uni = uniforms if uniforms is not None else np.zeros(1)
    fp = None if forced is None else np.ascontiguousarray(forced, dtype=np.int64).ravel()
    fn = lib.oracle_dense_f32 if R.dtype == np.float32 else lib.oracle_dense_f64
    st = fn(_ptr(R), n, m, steps, _RULES[tag], _ptr(uni), 0 if uniforms is None else uni.size,
            _ptr(fp), float(stop_tol), int(threads or os.cpu_count() or 1),
            _ptr(piv), _ptr(Lt), _ptr(U), _ptr(resid), _ptr(mg), _ptr(out))
    if st == -1:
        raise ZeroDivisionError(f"pivot at step {int(out[4])} has exactly zero value "
                                "after resampling")
    if st == -2:
        raise ValueError(f"steps {steps} out of range [0, {min(n, m)}]")
    if st:
        raise RuntimeError(f"oracle_dense failed ({st})")
    done = int(out[0])
    return dict(pivots=[(int(piv[2 * t]), int(piv[2 * t + 1])) for t in range(done)],
                L=Lt[:done].T, U=U[:done], resid_fro=resid[:done + 1], residual=R,
                steps=done, clean_early_stop=bool(out[2]), tol_stop=bool(out[3]),
                uniforms_consumed=int(out[1]),
                margins=None if mg is None else mg[:done])


def eliminate_c(A, tag, steps, seed=None, gen=None, stop_tol=0.0, margins=False, threads=None,
                copy=True, dtype=np.float64):
    """dense_pivots.py:129-209 on a real copy of A (``copy=False``
    eliminates a C-contiguous A of ``dtype`` in place); same result dict as
    ``eliminate_real`` plus ``uniforms_consumed``.  ``dtype=np.float32`` runs
    the same steps with float32 residual arithmetic (float64 masses), the
    C3-fp32 restatement."""
    if tag not in _RULES:
        raise ValueError(f"unknown pivot rule {tag!r}")
    R = np.array(A, dtype=dtype, order="C") if copy else np.ascontiguousarray(A, dtype)
    uniforms = None
    if tag == "rplu":
        g = gen if gen is not None else uniform_stream(seed)
        # bulk draws equal scalar draws; 4 per step covers
        # a resample at every step
        uniforms = g.random(4 * max(steps, 1))
    return _run(R, tag, steps, uniforms, None, stop_tol, threads, margins)


def replay_c(A, pivots, threads=None, dtype=np.float64):
    """Forced-pivot replay (dense_pivots.py:185-191 with given pivots) in
    ``dtype``; the float64 replay of fp32 pivots measures the fp32 factors'
    distance from exact-pivot float64 arithmetic."""
    R = np.array(A, dtype=dtype, order="C")
    forced = np.array(pivots, dtype=np.int64).reshape(-1, 2)
    return _run(R, "rplu", len(forced), None, forced, 0.0, threads, False)


def structured_eliminate_c(x, y, G, B, rule, rank, seed=None, gen=None, stop_tol=0.0,
                           keep_steps=False, threads=None):
    """cauchy.py:177-256 (plan=None) in C (oracle/c/cauchy_oracle.c): same
    result dict as ``rplu_oracle.structured_eliminate`` (row / column
    indices, bound maxes / sums, stop flags, kept (c, r, a) steps, final
    G / B, margins of the draws) plus ``uniforms_consumed``."""
    lib = _load()
    if not hasattr(lib, "_cauchy_typed"):
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_cauchy.argtypes = [P, P, P, P, i64, i64, ctypes.c_int, i64, ctypes.c_int, P,
                                      i64, ctypes.c_double, ctypes.c_int, P, P, P, P, P, P, P,
                                      P, P]
        lib.oracle_cauchy.restype = ctypes.c_int
        lib._cauchy_typed = True
    if rule not in ("rplu", "c2plu"):
        raise ValueError(f"unknown structured rule {rule!r}")
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128).ravel())
    y = np.ascontiguousarray(np.asarray(y, dtype=np.complex128).ravel())
    Gc = np.array(G, dtype=np.complex128, order="C")
    Bt = np.array(np.asarray(B, dtype=np.complex128).T, order="C")   # m x p
    n, p = Gc.shape
    m = Bt.shape[0]
    k = max(rank, 1)
    uniforms = np.zeros(1)
    if rule == "rplu":
        g = gen if gen is not None else uniform_stream(seed)
        uniforms = g.random(3 * k)
    rows = np.zeros(k, dtype=np.int64)
    cols = np.zeros(k, dtype=np.int64)
    bmax = np.zeros(k)
    bsum = np.zeros(k)
    mg = np.full(k, np.inf)
    R = np.zeros((k, m), dtype=np.complex128) if keep_steps else None
    C = np.zeros((k, n), dtype=np.complex128) if keep_steps else None
    av = np.zeros(k, dtype=np.complex128) if keep_steps else None
    out = np.zeros(5, dtype=np.int64)
    st = lib.oracle_cauchy(_ptr(x), _ptr(y), _ptr(Gc), _ptr(Bt), n, m, p, rank,
                           0 if rule == "rplu" else 1, _ptr(uniforms),
                           uniforms.size if rule == "rplu" else 0, float(stop_tol),
                           int(threads or os.cpu_count() or 1), _ptr(rows), _ptr(cols),
                           _ptr(bmax), _ptr(bsum), _ptr(mg), _ptr(R), _ptr(C), _ptr(av),
                           _ptr(out))
    if st == -1:
        raise ZeroDivisionError(f"pivot at step {int(out[4])} is numerically zero")
    if st == -2:
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    if st:
        raise RuntimeError(f"oracle_cauchy failed ({st})")
    done = int(out[0])
    nb = done + (1 if (out[2] or out[3]) else 0)
    res = dict(row_indices=[int(v) for v in rows[:done]], col_indices=[int(v) for v in cols[:done]],
               bound_maxes=list(bmax[:nb]), bound_sums=list(bsum[:nb]), tol_stop=bool(out[2]),
               degenerate_stop=bool(out[3]), margins=mg[:done], uniforms_consumed=int(out[1]),
               G=Gc, B=Bt.T.copy(), steps=[])
    if keep_steps:
        res["steps"] = [(C[t].copy(), R[t].copy(), complex(av[t])) for t in range(done)]
    return res
