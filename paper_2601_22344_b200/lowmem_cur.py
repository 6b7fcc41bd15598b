"""Low-memory CUR-form RPLU (Alg 2) on the B200 — drop-in for
``rplu.lowmem_cur`` (pkg/src/rplu/lowmem_cur.py).

Same signature, rules (rplu-cur / c2plu-cur), uniform consumption (row draw
then column draw; one extra row draw on a degenerate residual row,
:252-263), stop rules, clamp/rebuild semantics (:280-292) and returned
``(CurFactorization, CurBuildInfo)``.  Storage stays O(k^2 + n + m): the
index sets, the k x k core and a handful of length-n/m device vectors.

Per step the device work is one full generated GEMV g = A l (K7) plus
k-restricted products A[I,:]^T w / A[:,J] w (K8), single rows/columns, the
row-norm downdate (K9) and the two inverse-CDF draws (K2) — instead of the
reference's 4 applies of A and 2 of A^T (bench.py:91-100 ledger).  The core
keeps the reference's QR representation, refactored on the device
(cuSOLVER geqrf via torch) at each extension; ``core_mode='inverse'``
keeps the block-inverse update with its QR fallback (:106-125).
"""

import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from .operators import as_device_operator
from .rng import UniformBlock, sample_index

__all__ = ["CurFactorization", "CurBuildInfo", "cur_build", "core_extend",
           "residual_column", "residual_row", "CUR_RULES"]

CUR_RULES = ("rplu-cur", "c2plu-cur")
SIGMA_DEGENERATE = 1e-14       # lowmem_cur.py:37
CLAMP_REBUILD_FRACTION = 0.01  # lowmem_cur.py:40


def _t(v, like):
    if isinstance(v, torch.Tensor):
        return v.to(device=like.device, dtype=like.dtype)
    return torch.as_tensor(np.asarray(v), device=like.device).to(like.dtype)


class CurFactorization:
    """Skeleton indices plus a stable solver for the core A[I, J]
    (lowmem_cur.py:43-133), kept on the device."""

    def __init__(self, mode="qr", device=None, dtype=torch.float64):
        if mode not in ("qr", "inverse"):
            raise ValueError(f"unknown core mode {mode!r}")
        self.row_indices = []
        self.col_indices = []
        self.mode = mode
        self.fell_back = False
        dev = torch.device("cuda") if device is None else device
        self._W = torch.zeros((0, 0), dtype=dtype, device=dev)
        self._Q = self._R = None
        self._U = torch.zeros((0, 0), dtype=dtype, device=dev)

    @property
    def rank(self):
        return len(self.row_indices)

    def core_matrix(self):
        return self._W.cpu().numpy().copy()

    def _solve(self, v, transpose):
        dev_in = isinstance(v, torch.Tensor)
        vt = _t(v, self._W)
        if self.rank == 0:
            out = torch.zeros(0, dtype=self._W.dtype, device=self._W.device)
        elif self.mode == "inverse":
            out = (self._U.T @ vt) if transpose else (self._U @ vt)
        elif transpose:   # W^T x = v  ->  x = conj(Q) R^{-T} v   (:81-88)
            y = torch.linalg.solve_triangular(self._R.T, vt[:, None], upper=False)[:, 0]
            out = self._Q.conj() @ y
        else:             # W x = v    ->  x = R^{-1} Q^H v       (:72-79)
            out = torch.linalg.solve_triangular(self._R, (self._Q.conj().T @ vt)[:, None],
                                                upper=True)[:, 0]
        return out if dev_in else out.cpu().numpy()

    @classmethod
    def from_core(cls, rows, cols, W, mode="qr", fell_back=False):
        """A factorization of a core A[I, J] built by the device loop: the
        reference's representation (QR of W, or W^{-1} in inverse mode)
        computed once instead of at every extension."""
        f = cls(mode=mode, device=W.device, dtype=W.dtype)
        f.row_indices = [int(i) for i in rows]
        f.col_indices = [int(j) for j in cols]
        f._W = W
        f.fell_back = bool(fell_back)
        if fell_back:
            f.mode = "qr"
        if len(f.row_indices):
            if f.mode == "inverse":
                f._U = torch.linalg.inv(W)
            else:
                f._Q, f._R = torch.linalg.qr(W)
        return f

    def core_solve(self, v):
        """Solve A[I, J] x = v."""
        return self._solve(v, False)

    def core_solve_block(self, B):
        """Solve A[I, J] X = B for a k x c device block in one call (the
        rebuild and the CUR error evaluation; no per-column host round trip)."""
        Bt = B.to(device=self._W.device, dtype=torch.promote_types(B.dtype, self._W.dtype))
        if self.rank == 0:
            return Bt[:0]
        if self.mode == "inverse":
            return self._U.to(Bt.dtype) @ Bt
        Q, R = self._Q.to(Bt.dtype), self._R.to(Bt.dtype)
        return torch.linalg.solve_triangular(R, Q.conj().T @ Bt, upper=True)

    def core_solve_t(self, v):
        """Solve A[I, J]^T x = v (plain transpose)."""
        return self._solve(v, True)

    def extended(self, i_new, j_new, w, z, omega):
        """Grow by one pivot: w = A[I, j_new], z = A[i_new, J], omega = A[i_new, j_new]."""
        k = self.rank
        out = CurFactorization.__new__(CurFactorization)
        out.row_indices = self.row_indices + [int(i_new)]
        out.col_indices = self.col_indices + [int(j_new)]
        out.fell_back = self.fell_back
        out.mode = self.mode
        dt = self._W.dtype
        if isinstance(omega, complex) and not torch.is_complex(self._W):
            dt = torch.complex128
        W = torch.zeros((k + 1, k + 1), dtype=dt, device=self._W.device)
        W[:k, :k] = self._W
        if k:
            W[:k, k] = _t(w, W)
            W[k, :k] = _t(z, W)
        W[k, k] = omega
        out._W = W
        out._Q, out._R = self._Q, self._R
        out._U = self._U.to(dt)
        if out.mode == "inverse":
            U = out._U
            wt = _t(w, W) if k else None
            zt = _t(z, W) if k else None
            Uw = U @ wt if k else torch.zeros(0, dtype=dt, device=W.device)
            zU = U.T @ zt if k else torch.zeros(0, dtype=dt, device=W.device)
            sigma = omega - (complex((zt @ Uw).item()) if k else 0.0)
            guard = abs(omega) + (float(torch.linalg.norm(zt)) * float(torch.linalg.norm(Uw))
                                  if k else 0.0)
            if abs(sigma) <= SIGMA_DEGENERATE * max(guard, 1e-300):
                out.mode = "qr"
                out.fell_back = True
                warnings.warn("degenerate pivot complement in block-inverse update; core fell "
                              "back to QR", stacklevel=2)
            else:
                if not torch.is_complex(W):
                    sigma = sigma.real
                Un = torch.zeros((k + 1, k + 1), dtype=dt, device=W.device)
                Un[:k, :k] = U + torch.outer(Uw, zU) / sigma
                Un[:k, k] = -Uw / sigma
                Un[k, :k] = -zU / sigma
                Un[k, k] = 1.0 / sigma
                out._U = Un
                return out
        out._Q, out._R = torch.linalg.qr(W)
        return out


def core_extend(fact, w, z, omega, i_new=-1, j_new=-1):
    """Return the factorization grown by one pivot (lowmem_cur.py:136-139)."""
    return fact.extended(i_new, j_new, w, z, omega)


@dataclass
class CurBuildInfo:
    """History summary of a CUR build (lowmem_cur.py:142-151) plus device
    diagnostics (near-boundary draws, uniforms consumed, K7 timings)."""

    total_sq_norms: list = field(default_factory=list)
    clamped: list = field(default_factory=list)
    rebuilds: int = 0
    degenerate_stop: bool = False
    tol_stop: bool = False
    row_norms: np.ndarray = None
    near_boundary_draws: int = 0
    uniforms_consumed: int = 0
    gemv_ms: list = field(default_factory=list)


class _Stream:
    """Uniform stream with exact consumption accounting."""

    def __init__(self, rng, cap):
        self.block = UniformBlock(rng, cap) if rng is not None else None
        self.used = 0

    def next(self):
        u = float(self.block.values[self.used])
        self.used += 1
        return u

    def commit(self):
        if self.block is not None:
            self.block.commit(self.used)


def _sel(idx, dev):
    return torch.tensor(idx, dtype=torch.int64, device=dev)


def _residual_col_dev(op, fact, j):
    c = op.line_dev(1, j)
    I = _sel(fact.row_indices, op.device)
    y = fact.core_solve(c[I]) if fact.rank else torch.zeros(0, dtype=c.dtype, device=c.device)
    return c - op.restricted_dev(1, _sel(fact.col_indices, op.device), y), c


def _residual_row_dev(op, fact, i):
    r = op.line_dev(0, i)
    J = _sel(fact.col_indices, op.device)
    z = fact.core_solve_t(r[J]) if fact.rank else torch.zeros(0, dtype=r.dtype, device=r.device)
    return r - op.restricted_dev(0, _sel(fact.row_indices, op.device), z), r


def residual_column(A, fact, j):
    """Column j of the residual A - A[:, J] U A[I, :] (lowmem_cur.py:190-194)."""
    op = as_device_operator(A)
    return _residual_col_dev(op, fact, j)[0].cpu().numpy()


def residual_row(A, fact, i):
    """Row i of the residual (lowmem_cur.py:197-201)."""
    op = as_device_operator(A)
    return _residual_row_dev(op, fact, i)[0].cpu().numpy()


def _rebuild_row_norms(op, fact, nrow, chunk=256):
    """Recompute maintained norms from m residual columns (lowmem_cur.py:204-209),
    column-blocked with a device GEMM for the CUR correction."""
    n, m = op.shape
    nrow.zero_()
    I = _sel(fact.row_indices, op.device)
    J = _sel(fact.col_indices, op.device)
    CJ = op.block_cols_dev(0, m)[:, J] if m <= chunk else torch.stack(
        [op.line_dev(1, j) for j in fact.col_indices], dim=1)
    for j0 in range(0, m, chunk):
        j1 = min(j0 + chunk, m)
        blk = op.block_cols_dev(j0, j1)
        X = fact.core_solve_block(blk[I, :])      # one k x chunk solve
        res = blk - CJ @ X
        nrow += (res.real ** 2 + (res.imag ** 2 if torch.is_complex(res) else 0)).sum(1)


def cur_build(A, rule, rank, stop_tol=0.0, rng=None, core_mode="qr", *, time_gemv=False):
    """Build a rank-``rank`` CUR skeleton from device applies (lowmem_cur.py:212-300).

    ``A`` must be a device operator (GaussianKernelOperator or DenseMatrix);
    host-callable operators raise CapabilityError.  Returns
    ``(CurFactorization, CurBuildInfo)``.
    """
    if rule not in CUR_RULES:
        raise ValueError(f"unknown CUR rule {rule!r}")
    if rule == "rplu-cur" and rng is None:
        raise ValueError("rplu-cur needs an RngState")
    if hasattr(A, "require"):
        A.require("apply", "adjoint_apply", "row_norms")
    op = as_device_operator(A)
    n, m = op.shape
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    if core_mode not in ("qr", "inverse"):
        raise ValueError(f"unknown core mode {core_mode!r}")
    if not torch.is_complex(torch.empty(0, dtype=op.dtype)) and rank <= 8192:
        return _cur_build_device(op, rule, rank, stop_tol, rng, core_mode, time_gemv)
    return _cur_build_torch(op, rule, rank, stop_tol, rng, core_mode, time_gemv)


def _cur_build_device(op, rule, rank, stop_tol, rng, core_mode, time_gemv):
    """The whole loop in ``rplu_mf_run`` (csrc/mf.cu): one host
    synchronisation per step, device draws, device core (LU in selection
    order), device rebuild.  Real operators: the Gaussian kernel and real
    dense matrices."""
    import ctypes

    from . import _device, _ffi
    from .operators import _GaussDeviceOp
    n, m = op.shape
    dev = op.device
    info = CurBuildInfo()
    stream = _Stream(rng if rule == "rplu-cur" else None, 3 * max(rank, 1))
    if isinstance(op, _GaussDeviceOp):
        g = op.g
        kind, P, Q, h, Ad, lda = _ffi.MF_GAUSS3D, g.P.data_ptr(), g.Q.data_ptr(), g.h, None, 0
        keep = (g.P, g.Q)
    else:
        At = op.t.to(torch.float64)
        if At.stride(1) != 1:
            At = At.contiguous()
        kind, P, Q, h, Ad, lda = _ffi.MF_DENSE, None, None, 0.0, At.data_ptr(), At.stride(0)
        keep = (At,)
    k1 = max(rank, 1)
    rows = np.zeros(k1, dtype=np.int64)
    cols = np.zeros(k1, dtype=np.int64)
    totals = np.zeros(rank + 1)
    clamped = np.zeros(k1, dtype=np.int64)
    core = np.zeros(k1 * k1)
    nrow = torch.empty(n, dtype=torch.float64, device=dev)
    uni = stream.block.values if stream.block is not None else None
    args = _ffi.MfArgs(
        op_kind=kind, rule=_ffi.RULE_IDS["rplu" if rule == "rplu-cur" else "c2plu"], n=n, m=m,
        rank=rank, stop_tol=float(stop_tol), P=P, Q=Q, h=h, A=Ad, lda=lda,
        uniforms=uni.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if uni is not None else None,
        n_uniforms=uni.size if uni is not None else 0,
        stream=torch.cuda.current_stream(dev).cuda_stream,
        flags=_ffi.FLAG_TIME_KERNELS if time_gemv else 0)
    out = _ffi.MfOut(rows=rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                     cols=cols.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                     total_sq_norms=totals.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     clamped=clamped.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                     core=core.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     row_norms_dev=nrow.data_ptr())
    c = _device.ctx(dev)
    try:
        status = c._lib.rplu_mf_run(c.handle, ctypes.byref(args), ctypes.byref(out))
        stream.used = int(out.uniforms_consumed)
    finally:
        stream.commit()
    del keep
    _ffi.check(status)
    k = int(out.steps_done)
    W = torch.from_numpy(core[:k * k].reshape(k, k).copy()).to(dev)
    if core_mode == "inverse" and out.core_fell_back:
        warnings.warn("degenerate pivot complement in block-inverse update; core fell back to QR",
                      stacklevel=3)
    fact = CurFactorization.from_core(rows[:k], cols[:k], W, mode=core_mode,
                                      fell_back=core_mode == "inverse" and bool(out.core_fell_back))
    info.total_sq_norms = [float(x) for x in totals[:k + 1]]
    info.clamped = [int(x) for x in clamped[:k]]
    info.rebuilds = int(out.rebuilds)
    info.degenerate_stop = bool(out.degenerate_stop)
    info.tol_stop = bool(out.tol_stop)
    info.row_norms = nrow.cpu().numpy()
    info.near_boundary_draws = int(out.near_boundary_draws)
    info.uniforms_consumed = int(out.uniforms_consumed)
    info.kernel_launches = int(out.kernel_launches)
    if time_gemv and k:
        # K7 time of the run (the initial row-norm pass and the k g = A l
        # passes), spread evenly over the steps
        info.gemv_ms = [float(out.gemv_ms) / k] * k
    return fact, info


def _cur_build_torch(op, rule, rank, stop_tol, rng, core_mode, time_gemv):
    """Complex operators (a complex DenseMatrix): the same loop driven from
    Python over torch / cuBLAS device ops and the K2 draw kernel."""
    n, m = op.shape
    dev = op.device
    info = CurBuildInfo()
    fact = CurFactorization(mode=core_mode, device=dev, dtype=op.dtype)

    nrow = op.row_norms_dev().to(torch.float64).clone()
    total0 = float(nrow.sum())
    info.total_sq_norms.append(total0)
    if total0 == 0.0:
        info.degenerate_stop = True
        info.row_norms = nrow.cpu().numpy()
        return fact, info
    eps = np.finfo(float).eps
    stream = _Stream(rng if rule == "rplu-cur" else None, 3 * max(rank, 1))
    real = not torch.is_complex(torch.empty(0, dtype=op.dtype))
    from . import _device, _ffi
    import ctypes
    c_ctx = _device.ctx(dev)
    cur_total = total0

    def draw_row():
        if rule == "rplu-cur":
            i = sample_index(nrow, stream.next())
        else:
            i = int(torch.argmax(nrow))
        rhat, r = _residual_row_dev(op, fact, i)
        return i, rhat, r

    try:
        for _ in range(rank):
            if cur_total <= 0.0:
                info.degenerate_stop = True
                break
            i, rhat, r = draw_row()
            w = rhat.abs() ** 2
            energy = float(w.sum())
            if energy <= eps ** 2 * total0:
                i, rhat, r = draw_row()
                w = rhat.abs() ** 2
                energy = float(w.sum())
                if energy <= eps ** 2 * total0:
                    info.degenerate_stop = True
                    break
            if rule == "rplu-cur":
                j = sample_index(w, stream.next())
            else:
                j = int(torch.argmax(rhat.abs()))
            a = rhat[j].item()
            chat, c = _residual_col_dev(op, fact, j)
            if real:   # numpy complex division by a real value is x * (1/a)
                l = rhat * (1.0 / a)
            else:
                l = torch.conj(rhat) / np.conj(a)
            g = op.apply_dev(l, timed=time_gemv)
            if time_gemv:
                info.gemv_ms.append(op.last_kernel_ms)
            I = _sel(fact.row_indices, dev)
            yv = fact.core_solve(g[I]) if fact.rank else torch.zeros(0, dtype=g.dtype, device=dev)
            v = op.restricted_dev(1, _sel(fact.col_indices, dev), yv)
            prev = info.total_sq_norms[-1]
            l2 = float((l.abs() ** 2).sum())
            floor = eps * prev / n
            if real:
                cl = ctypes.c_int64(0)
                tot = ctypes.c_double(0.0)
                _ffi.check(c_ctx._lib.rplu_cur_downdate(
                    c_ctx.handle, n, nrow.data_ptr(), g.contiguous().data_ptr(),
                    v.contiguous().data_ptr(), chat.contiguous().data_ptr(), l2, floor,
                    ctypes.byref(cl), ctypes.byref(tot), _device.stream_handle(dev)))
                clamped, cur_total = int(cl.value), float(tot.value)
            else:
                nrow -= 2.0 * torch.real((g - v) * torch.conj(chat))
                nrow += l2 * chat.abs() ** 2
                clamped = int((nrow < -floor).sum())
                nrow.clamp_(min=0.0)
                cur_total = float(nrow.sum())
            info.clamped.append(clamped)
            fact = fact.extended(i, j, c[I] if fact.rank else None,
                                 r[_sel(fact.col_indices, dev)] if fact.rank else None,
                                 r[j].item())
            if clamped > CLAMP_REBUILD_FRACTION * n:
                _rebuild_row_norms(op, fact, nrow)
                info.rebuilds += 1
                cur_total = float(nrow.sum())
            info.total_sq_norms.append(cur_total)
            if stop_tol > 0 and cur_total <= stop_tol ** 2 * total0:
                info.tol_stop = True
                break
    finally:
        stream.commit()
    info.row_norms = nrow.cpu().numpy()
    info.uniforms_consumed = stream.used
    return fact, info
