"""Error evaluation of a low-rank approximation on the device.

Restates the reference's sweep error measures (``cli.py:86-99``,
``cli.py:151-157``, ``cli.py:200-206``, ``core.py:66-76``) on HBM-resident
factors:

* ``lu_error(A, L, U)`` — ||A - L U||_F / ||A||_F (a17): the K11 kernel
  (``rplu_lu_error``, ``csrc/lu_error.cu``) accumulates L U tile by tile on
  the FP64 tensor cores (DMMA) and folds the subtraction, the square and
  both Frobenius sums into its epilogue — no panel of L U or A - L U is ever
  written.  ``lu_error_sq`` returns the raw sums and the kernel time.
* ``cur_error(A, fact)`` — ||A - C W^{-1} R||_F for a CUR factorization
  (cli.py:163-169 with _cur_dense :200-206): C^T = A[:, J]^T and
  W^{-1} A[I, :] (device core solve) through the same kernel.
* ``residual_spectral(A, L, U, seed, iters=20)`` — the reference's power
  iteration on R = A - L U (``_residual_spectral``, cli.py:86-99): the start
  vector is ``RngState(seed).complex_normal(m)`` normalized, then ``iters``
  steps of w = R^H (R v), est = ||w||, v = w / est; returns sqrt(est).  R is
  applied as A v - L (U v), never formed; real factors stay real (the
  complex iterate is applied as two real vectors).
* ``truncated_svd_error(A, k)`` — the optimal rank-k errors from the
  singular values (cuSOLVER via torch), for the error ratios of the sweeps.
"""

import ctypes

import numpy as np
import torch

from . import _device, _ffi
from .rng import RngState

__all__ = ["lu_error", "lu_error_sq", "cur_error", "residual_spectral", "truncated_svd_error"]

_DT = {torch.float32: _ffi.RPLU_F32, torch.float64: _ffi.RPLU_F64,
       torch.complex128: _ffi.RPLU_C128}


def _dev(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(dev)
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def _operands(A, L, U, dev=None):
    """Device A, Lt = L^T (k x n) and U (k x m) in one common dtype, each
    moved / converted once: complex128 if any is complex, float32 if all are
    float32, else float64."""
    dev = dev or (A.device if isinstance(A, torch.Tensor) and A.is_cuda else
                  _device.require_cuda())
    At, Lt, Ut = _dev(A, dev), _dev(L, dev), _dev(U, dev)
    dts = {At.dtype, Lt.dtype, Ut.dtype}
    if any(t.is_complex for t in dts):
        dt = torch.complex128
    elif dts == {torch.float32}:
        dt = torch.float32
    else:
        dt = torch.float64
    At = At.to(dt)
    if At.stride(1) != 1:
        At = At.contiguous()
    Lt = Lt.to(dt).T            # k x n view; contiguous when L came from eliminate
    if Lt.stride(1) != 1:
        Lt = Lt.contiguous()
    Ut = Ut.to(dt)
    if Ut.stride(1) != 1:
        Ut = Ut.contiguous()
    return At, Lt, Ut


def _kernel(At, Xt, Y):
    n, m = At.shape
    k = Xt.shape[0]
    if Xt.shape[1] != n or Y.shape != (k, m):
        raise ValueError(f"factor shapes {tuple(Xt.shape)} / {tuple(Y.shape)} do not match "
                         f"A {tuple(At.shape)}")
    c = _device.ctx(At.device)
    out = (ctypes.c_double * 2)()
    ms = ctypes.c_double(0.0)
    kx = max(k, 0)
    _ffi.check(c._lib.rplu_lu_error(
        c.handle, _DT[At.dtype], ctypes.c_void_p(At.data_ptr()), At.stride(0), n, m,
        ctypes.c_void_p(Xt.data_ptr() if kx else 0), Xt.stride(0) if kx else n,
        ctypes.c_void_p(Y.data_ptr() if kx else 0), Y.stride(0) if kx else m, kx, out,
        ctypes.byref(ms), _device.stream_handle(At.device)))
    return float(out[0]), float(out[1]), float(ms.value)


def lu_error_sq(A, L, U):
    """(||A - L U||_F^2, ||A||_F^2, product-kernel ms) through K11."""
    At, Lt, Ut = _operands(A, L, U)
    return _kernel(At, Lt, Ut)


def lu_error(A, L, U):
    """||A - L U||_F / ||A||_F (cli.py:151-157), fused on the tensor cores."""
    e, a, _ = lu_error_sq(A, L, U)
    return float(np.sqrt(e) / np.sqrt(a)) if a > 0 else 0.0


def cur_error(A, fact):
    """(||A - C W^{-1} R||_F, ||A||_F) for a CUR factorization over a dense
    A (cli.py:163-169, _cur_dense :200-206): C = A[:, J], R = A[I, :]."""
    dev = A.device if isinstance(A, torch.Tensor) and A.is_cuda else _device.require_cuda()
    At = _dev(A, dev)
    if not At.is_complex():
        At = At.to(torch.float64)
    if fact.rank == 0:
        e, a, _ = _kernel(At, At.new_zeros((0, At.shape[0])), At.new_zeros((0, At.shape[1])))
        return float(np.sqrt(e)), float(np.sqrt(a))
    I = torch.as_tensor(list(fact.row_indices), dtype=torch.int64, device=dev)
    J = torch.as_tensor(list(fact.col_indices), dtype=torch.int64, device=dev)
    Ct = At[:, J].T.contiguous()                      # k x n
    Rr = At[I, :]                                     # k x m
    Y = fact.core_solve_block(Rr)                     # W^{-1} R, k x m
    dt = torch.complex128 if (At.is_complex() or Y.is_complex()) else torch.float64
    e, a, _ = _kernel(At.to(dt).contiguous(), Ct.to(dt), Y.to(dt).contiguous())
    return float(np.sqrt(e)), float(np.sqrt(a))


def residual_spectral(A, L, U, seed, iters=20):
    """Power-iteration estimate of ||A - L U||_2 (cli.py:86-99)."""
    At, Lt, Ut = _operands(A, L, U)
    if At.dtype == torch.float32:
        At, Lt, Ut = At.double(), Lt.double(), Ut.double()
    Lm = Lt.T
    real = not At.is_complex()
    rng = RngState(seed)
    v0 = rng.complex_normal(At.shape[1])
    v0 = v0 / np.linalg.norm(v0)
    v = torch.from_numpy(v0).to(At.device)
    k = Lm.shape[1]

    def lin(x):          # R x
        return At @ x - (Lm @ (Ut @ x) if k else 0)

    def lin_h(y):        # R^H y
        return At.conj().T @ y - (Ut.conj().T @ (Lm.conj().T @ y) if k else 0)

    def both(fn, z):
        if real:         # real operator on a complex vector: two real applies
            return torch.complex(fn(z.real.contiguous()), fn(z.imag.contiguous()))
        return fn(z)

    est = 0.0
    for _ in range(iters):
        w = both(lin_h, both(lin, v))
        est = float(torch.linalg.norm(w))
        if est == 0.0:
            return 0.0
        v = w / est
    return float(np.sqrt(est))


def truncated_svd_error(A, k):
    """Optimal rank-k errors (sqrt(sum of trailing sigma^2), sigma_{k+1}) (core.py:66-76)."""
    At = _dev(A, A.device if isinstance(A, torch.Tensor) and A.is_cuda else
              _device.require_cuda())
    r = min(At.shape)
    if not 0 <= k <= r:
        raise ValueError(f"rank {k} out of range [0, {r}]")
    s = torch.linalg.svdvals(At.to(torch.complex128 if torch.is_complex(At) else torch.float64))
    tail = s[k:]
    return float(torch.sqrt((tail ** 2).sum())), (float(s[k]) if k < r else 0.0)
