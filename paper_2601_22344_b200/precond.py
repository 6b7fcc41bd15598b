"""SMW preconditioning of B + (low rank) and restarted GMRES on the B200 —
drop-in for ``rplu.precond`` (pkg/src/rplu/precond.py), SURVEY §8(f4).

The preconditioner applies (B + A[:, J] U A[I, :])^{-1} through the
Sherman-Morrison-Woodbury identity with the k x k inner matrix
W + A[I, :] B^{-1} A[:, J] (W = A[I, J], the CUR core of ``cur_build``).
B200 differences:

* for device operators (``DenseMatrix``, ``GaussianKernelOperator``) the two
  operator touches of an apply are k-restricted: A[I, :] u is the
  generated-entry GEMV of the k selected rows (K7 on the gathered row points)
  and A[:, J] q the K8 restricted product — O((n + m) k) instead of the
  reference's two full O(nm) applies (precond.py:48-55);
* the inner LU is cuSOLVER's (torch.linalg.lu_factor) on the device;
* GMRES keeps the Krylov basis in HBM ((restart + 1) x n complex128, one
  contiguous row per basis vector) and runs each modified Gram-Schmidt
  Arnoldi step as ONE cooperative kernel (``rplu_mgs_arnoldi``); only the
  (j + 2)-entry Hessenberg column crosses to the host for the Givens
  rotations, which stay on the host in the reference's scalar order.

Operators and B^{-1}: device accessors are applied on the device; a callable
is treated as a host (numpy) callable, as in the reference, unless it
carries ``on_device = True`` (see :func:`device_callable`), in which case it
receives and returns CUDA tensors.  Host arrays become device matrices.
"""

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import torch

from . import _device, _ffi
from .accessors import DenseMatrix, MatrixAccessor, foreign_dense_array, is_host_accessor

__all__ = ["SmwPreconditioner", "smw_build", "gmres", "GmresResult", "device_callable"]

INNER_CONDITION_LIMIT = 1e15   # precond.py:21


def device_callable(fn):
    """Mark ``fn`` as taking and returning CUDA complex128 tensors."""
    fn.on_device = True
    return fn


def _host_fn(fn, dev):
    def call(v):
        out = fn(v.cpu().numpy())
        return torch.from_numpy(np.ascontiguousarray(np.asarray(out, dtype=np.complex128))).to(dev)
    return call


def _c128(v, dev):
    if isinstance(v, torch.Tensor):
        return v.to(device=dev, dtype=torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=np.complex128))).to(dev)


class _DeviceLinear:
    """Device view of an operator accessor: full apply plus the k-restricted
    row / column products the SMW apply needs."""

    def __init__(self, A, dev):
        from .operators import GaussianKernelOperator
        self.dev = dev
        self.gauss = A if isinstance(A, GaussianKernelOperator) else None
        self.dense = None
        self.host = None
        if self.gauss is None:
            if isinstance(A, DenseMatrix):
                self.dense = A.tensor
            elif isinstance(A, torch.Tensor) and A.is_cuda:
                self.dense = A
            elif foreign_dense_array(A) is not None:   # the reference's rplu.DenseMatrix
                self.dense = _c128(foreign_dense_array(A), dev)
            elif is_host_accessor(A):
                self.host = A        # reference semantics: full applies through the accessor
            else:
                self.dense = _c128(A, dev)
        self.shape = tuple(A.shape)
        self._rows_op = None

    def _real_op(self, fn, v):
        if v.is_complex():
            return torch.complex(fn(v.real.contiguous()), fn(v.imag.contiguous()))
        return fn(v)

    def apply(self, v):
        if self.gauss is not None:
            return self._real_op(self.gauss.apply_dev, v)
        if self.dense is not None:
            if self.dense.is_complex():
                return self.dense @ v.to(self.dense.dtype)
            return self._real_op(lambda x: self.dense @ x.to(self.dense.dtype), v)
        return _c128(self.host.apply(v.cpu().numpy()), self.dev)

    def column(self, j):
        """A[:, j] (the reference applies A to a unit vector, precond.py:86)."""
        if self.gauss is not None:
            return self.gauss.line_dev(1, int(j)).to(torch.complex128)
        if self.dense is not None:
            return self.dense[:, int(j)].to(torch.complex128)
        e = np.zeros(self.shape[1], dtype=np.complex128)
        e[int(j)] = 1.0
        return _c128(self.host.apply(e), self.dev)

    def rows_apply(self, I, u):
        """(A u)[I] without the full product."""
        if self.gauss is not None:
            if self._rows_op is None or self._rows_op[0] != tuple(I):
                from .operators import GaussianKernelOperator
                sel = torch.as_tensor(list(I), dtype=torch.int64, device=self.dev)
                sub = GaussianKernelOperator(self.gauss.P[sel], self.gauss.Q, self.gauss.h,
                                             device=self.dev)
                self._rows_op = (tuple(I), sub)
            return self._real_op(self._rows_op[1].apply_dev, u)
        if self.dense is not None:
            sel = torch.as_tensor(list(I), dtype=torch.int64, device=self.dev)
            rows = self.dense[sel]
            if rows.is_complex():
                return rows @ u.to(rows.dtype)
            return self._real_op(lambda x: rows @ x.to(rows.dtype), u)
        return self.apply(u)[torch.as_tensor(list(I), dtype=torch.int64, device=self.dev)]

    def cols_apply(self, J, q):
        """A[:, J] q (the reference scatters q and applies A, precond.py:24-27)."""
        sel = torch.as_tensor(list(J), dtype=torch.int64, device=self.dev)
        if self.gauss is not None:
            f = lambda x: self.gauss.restricted_dev(1, sel, x)  # noqa: E731
            return self._real_op(f, q)
        if self.dense is not None:
            cols = self.dense[:, sel]
            if cols.is_complex():
                return cols @ q.to(cols.dtype)
            return self._real_op(lambda x: cols @ x.to(cols.dtype), q)
        v = torch.zeros(self.shape[1], dtype=torch.complex128, device=self.dev)
        v[sel] = q
        return self.apply(v)


def _as_dev_fn(op, dev):
    """Device apply for an operator, preconditioner, callable or array
    (precond.py:109-118)."""
    if isinstance(op, SmwPreconditioner):
        return op.apply_dev
    if isinstance(op, (MatrixAccessor, torch.Tensor)) or foreign_dense_array(op) is not None \
            or (is_host_accessor(op) and not callable(op)):
        return _DeviceLinear(op, dev).apply
    if callable(op):
        return op if getattr(op, "on_device", False) else _host_fn(op, dev)
    return _DeviceLinear(np.asarray(op, dtype=np.complex128), dev).apply


class SmwPreconditioner:
    """Applies (B + A[:, J] U A[I, :])^{-1} with two B-solves and two
    k-restricted operator products (precond.py:30-58).  Reentrant: apply
    only reads the cached device factors."""

    def __init__(self, b_inv_apply, A, fact, inner_lu, device=None):
        self._dev = _device.require_cuda(device)
        self._b_inv = _as_dev_fn(b_inv_apply, self._dev)
        self._A = A
        self._lin = _DeviceLinear(A, self._dev)
        self._fact = fact
        if inner_lu is not None and isinstance(inner_lu[0], np.ndarray):
            # scipy.linalg.lu_factor output: 0-based pivots -> LAPACK 1-based
            inner_lu = (_c128(inner_lu[0], self._dev),
                        torch.as_tensor(np.asarray(inner_lu[1]) + 1, dtype=torch.int32,
                                        device=self._dev))
        self._inner_lu = inner_lu

    @property
    def rank(self):
        return self._fact.rank if self._fact is not None else 0

    def apply_dev(self, v):
        u = self._b_inv(_c128(v, self._dev))
        if self.rank == 0:
            return u
        s = self._lin.rows_apply(self._fact.row_indices, u)       # R_k B^{-1} v
        LU, piv = self._inner_lu
        q = torch.linalg.lu_solve(LU, piv, s[:, None])[:, 0]
        corr = self._b_inv(self._lin.cols_apply(self._fact.col_indices, q))
        return u - corr

    def apply(self, v):
        if isinstance(v, torch.Tensor):
            return self.apply_dev(v)
        return self.apply_dev(v).cpu().numpy()

    def __call__(self, v):
        return self.apply(v)


def smw_build(b_inv_apply, A, fact, device=None):
    """Assemble the preconditioner for P = B + A[:, J] U A[I, :]
    (precond.py:61-94): inner = A[I, J] + A[I, :] B^{-1} A[:, J], built one
    selected column at a time, condition-checked and LU-factorised on the
    device.  A singular inner matrix raises LinAlgError."""
    n, m = A.shape
    if n != m:
        raise ValueError("the preconditioned system must be square")
    dev = _device.require_cuda(device)
    k = fact.rank
    if k == 0:
        return SmwPreconditioner(b_inv_apply, A, fact, None, device=dev)
    pre = SmwPreconditioner(b_inv_apply, A, fact, None, device=dev)
    lin, binv = pre._lin, pre._b_inv
    G = torch.empty((k, k), dtype=torch.complex128, device=dev)
    for t, j in enumerate(fact.col_indices):
        G[:, t] = lin.rows_apply(fact.row_indices, binv(lin.column(j)))
    W = fact._W if isinstance(getattr(fact, "_W", None), torch.Tensor) else \
        _c128(fact.core_matrix(), dev)
    inner = W.to(device=dev, dtype=torch.complex128) + G
    cond = float(torch.linalg.cond(inner))
    if not np.isfinite(cond) or cond > INNER_CONDITION_LIMIT:
        raise np.linalg.LinAlgError(
            f"inner SMW matrix has condition {cond:.2e}; reduce the CUR rank")
    pre._inner_lu = torch.linalg.lu_factor(inner)
    return pre


@dataclass
class GmresResult:
    x: np.ndarray
    residuals: np.ndarray      # relative residual after each inner step
    iterations: int
    converged: bool
    stagnated: bool = False


def _norm(v):
    return float(torch.linalg.vector_norm(v))


def gmres(K, b, M_inv=None, restart=20, tol=1e-10, max_restarts=200, x0=None, device=None):
    """Right-preconditioned restarted GMRES with modified Gram-Schmidt
    (precond.py:129-192).  ``x`` is returned as a numpy array (a CUDA tensor
    when ``b`` is one)."""
    if restart < 1:
        raise ValueError("restart must be >= 1")
    dev = b.device if isinstance(b, torch.Tensor) and b.is_cuda else _device.require_cuda(device)
    as_torch = isinstance(b, torch.Tensor)
    apply_k = _as_dev_fn(K, dev)
    apply_m = (lambda v: v) if M_inv is None else _as_dev_fn(M_inv, dev)
    bd = _c128(b, dev).reshape(-1)
    n = bd.numel()
    x = torch.zeros(n, dtype=torch.complex128, device=dev) if x0 is None else \
        _c128(x0, dev).reshape(-1).clone()
    out = (lambda v: v) if as_torch else (lambda v: v.cpu().numpy())
    bnorm = _norm(bd)
    if bnorm == 0.0:
        return GmresResult(out(x * 0.0), np.zeros(0), 0, True)

    c = _device.ctx(dev)
    stream = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    history = []
    best_x, best_res = x.clone(), np.inf
    total_iters = 0
    # every basis row is written before it is read (row j+1 by the Arnoldi
    # kernel, or zeroed below when H[j+1, j] == 0), so no fill pass is needed
    V = torch.empty((restart + 1, n), dtype=torch.complex128, device=dev)
    hcol = torch.zeros(restart + 2, dtype=torch.complex128, device=dev)

    for _ in range(max_restarts):
        r = bd - apply_k(x)
        beta = _norm(r)
        if beta / bnorm <= tol:
            return GmresResult(out(x), np.array(history), total_iters, True)
        cycle_start = beta / bnorm
        H = np.zeros((restart + 1, restart), dtype=np.complex128)
        cs = np.zeros(restart, dtype=np.complex128)
        sn = np.zeros(restart, dtype=np.complex128)
        g = np.zeros(restart + 1, dtype=np.complex128)
        V[0] = r * (1.0 / beta)           # r / beta (numpy: times 1/beta)
        g[0] = beta
        j_done = 0
        for j in range(restart):
            w = _c128(apply_k(apply_m(V[j])), dev).reshape(-1).clone()
            _ffi.check(c._lib.rplu_mgs_arnoldi(c.handle, V.data_ptr(), n, j, w.data_ptr(),
                                               V[j + 1].data_ptr(), hcol.data_ptr(), stream))
            H[:j + 2, j] = hcol[:j + 2].cpu().numpy()
            if not H[j + 1, j].real > 0:     # lucky breakdown: the reference's V[:, j+1] stays 0
                V[j + 1].zero_()
            for t in range(j):
                tmp = cs[t] * H[t, j] + sn[t] * H[t + 1, j]
                H[t + 1, j] = -np.conj(sn[t]) * H[t, j] + np.conj(cs[t]) * H[t + 1, j]
                H[t, j] = tmp
            denom = np.sqrt(np.abs(H[j, j]) ** 2 + np.abs(H[j + 1, j]) ** 2)
            if denom == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j] = np.conj(H[j, j]) / denom
                sn[j] = np.conj(H[j + 1, j]) / denom
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            total_iters += 1
            j_done = j + 1
            rel = float(np.abs(g[j + 1])) / bnorm
            history.append(rel)
            if rel <= tol:
                break
        y = scipy.linalg.solve_triangular(H[:j_done, :j_done], g[:j_done])
        yd = torch.from_numpy(y).to(dev)
        x = x + apply_m(V[:j_done].T @ yd)
        true_rel = _norm(bd - apply_k(x)) / bnorm
        if true_rel < best_res:
            best_res, best_x = true_rel, x.clone()
        if true_rel <= tol:
            return GmresResult(out(x), np.array(history), total_iters, True)
        if cycle_start - true_rel < 1e-14 * cycle_start:
            warnings.warn("GMRES stagnated within one restart cycle; "
                          "returning the best iterate", stacklevel=2)
            return GmresResult(out(best_x), np.array(history), total_iters, False,
                               stagnated=True)
    return GmresResult(out(best_x), np.array(history), total_iters, False)
