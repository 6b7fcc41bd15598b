"""Cauchy-like matrices and structured RPLU on the B200 — drop-in for
``rplu.cauchy`` (pkg/src/rplu/cauchy.py).

``CauchyLikeMatrix`` keeps its O((n+m)p) generators in HBM: x[n], y[m]
(complex128), G (n x p, row-major as the reference's C-order G) and B stored
as Bt (m x p, i.e. the reference's F-order B, column j contiguous).
``structured_eliminate`` with ``plan=None`` runs the exact-norm Alg 3 loop
entirely on the device (K5 generated-entry row masses, K2 selects, K6 row /
column generation and generator update) through ``rplu_cauchy_run``; with a
plan (certified tree bounds + rejection sampling) it raises
CapabilityError instead of silently switching to exact norms, because the
plan path consumes a different uniform stream.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _ffi
from .accessors import CapabilityError, MatrixAccessor
from .rng import UniformBlock

__all__ = ["CauchyLikeMatrix", "StructuredPivotTrace", "generator_schur_update",
           "exact_row_norms", "structured_eliminate", "MAX_DISPLACEMENT_RANK",
           "PIVOT_REL_TOL"]

MAX_DISPLACEMENT_RANK = 8    # cauchy.py:30
PIVOT_REL_TOL = 1e-14        # cauchy.py:33
REJECTION_CAP_FACTOR = 64    # cauchy.py:36


def _c128(a, dev):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128))).to(dev)


class CauchyLikeMatrix(MatrixAccessor):
    """Points x, y and generators G (n x p), B (p x m) in device memory
    (cauchy.py:39-116).  Entries (G_i . B_:,j) / (x_i - y_j)."""

    has_apply = True
    has_adjoint_apply = True
    has_entry = True
    has_row = True
    has_column = True
    has_row_norms = True
    on_device = True

    def __init__(self, x, y, G, B, check_points=True, device=None, _bt=None):
        dev = _device.require_cuda(device)
        self.x = _c128(x, dev).reshape(-1)
        self.y = _c128(y, dev).reshape(-1)
        Gt = _c128(G, dev)
        if _bt is not None:
            Bt = _bt
        else:
            Bd = _c128(B, dev)
            if Gt.dim() != 2 or Bd.dim() != 2:
                raise ValueError("generators must be 2-D")
            Bt = Bd.T.contiguous()
        if Gt.dim() != 2:
            raise ValueError("generators must be 2-D")
        n, p = Gt.shape
        m, p2 = Bt.shape
        if p != p2 or n != self.x.numel() or m != self.y.numel():
            raise ValueError("generator shapes do not match the point sets")
        if p > MAX_DISPLACEMENT_RANK:
            raise ValueError(f"displacement rank {p} exceeds {MAX_DISPLACEMENT_RANK}")
        for t in (self.x, self.y, Gt, Bt):
            if not bool(torch.isfinite(torch.view_as_real(t)).all()):
                raise ValueError("points and generators must be finite")
        self.G = Gt
        self.Bt = Bt
        self.shape = (n, m)
        if check_points and _min_cross_distance(self.x, self.y) == 0.0:
            raise ValueError("x and y share a point; entries are undefined")

    @property
    def B(self):
        return self.Bt.T

    @property
    def displacement_rank(self):
        return self.G.shape[1]

    @property
    def device(self):
        return self.G.device

    def entry(self, i, j):
        v = (self.G[i] @ self.Bt[j]) / (self.x[i] - self.y[j])
        return complex(v.item())

    def row(self, i):
        return ((self.Bt @ self.G[i]) / (self.x[i] - self.y)).cpu().numpy()

    def column(self, j):
        return ((self.G @ self.Bt[j]) / (self.x - self.y[j])).cpu().numpy()

    def _blocks(self, rows=None):
        n, m = self.shape
        rows = rows or max(1, (1 << 24) // max(m, 1))
        for lo in range(0, n, rows):
            hi = min(lo + rows, n)
            K = (self.G[lo:hi] @ self.Bt.T) / (self.x[lo:hi, None] - self.y[None, :])
            yield lo, hi, K

    def apply(self, v):
        vt = _c128(v, self.device)
        out = torch.empty(self.shape[0], dtype=torch.complex128, device=self.device)
        for lo, hi, K in self._blocks():
            out[lo:hi] = K @ vt
        return out.cpu().numpy()

    def adjoint_apply(self, v):
        vt = _c128(v, self.device)
        out = torch.zeros(self.shape[1], dtype=torch.complex128, device=self.device)
        for lo, hi, K in self._blocks():
            out += K.conj().T @ vt[lo:hi]
        return out.cpu().numpy()

    def row_norms(self):
        return exact_row_norms(self)

    def materialize(self):
        out = torch.empty(self.shape, dtype=torch.complex128, device=self.device)
        for lo, hi, K in self._blocks():
            out[lo:hi] = K
        return out.cpu().numpy()

    def displacement_residual(self):
        A = torch.from_numpy(self.materialize()).to(self.device)
        R = self.x[:, None] * A - A * self.y[None, :] - self.G @ self.Bt.T
        return float(R.abs().max())

    def copy(self):
        return CauchyLikeMatrix(self.x, self.y, self.G.clone(), None, check_points=False,
                                _bt=self.Bt.clone())


def _min_cross_distance(x, y):
    best = float("inf")
    rows = max(1, (1 << 24) // max(y.numel(), 1))
    for lo in range(0, x.numel(), rows):
        d = (x[lo:lo + rows, None] - y[None, :]).abs().min()
        best = min(best, float(d))
        if best == 0.0:
            break
    return best


def exact_row_norms(M):
    """Squared residual row norms by direct O(nmp) evaluation on the device
    (cauchy.py:129-137; K5 generated-entry kernel).  Returns numpy."""
    return exact_row_norms_device(M).cpu().numpy()


def exact_row_norms_device(M):
    n, m = M.shape
    out = torch.empty(n, dtype=torch.float64, device=M.device)
    c = _device.ctx(M.device)
    _ffi.check(c._lib.rplu_cauchy_row_norms(
        c.handle, M.displacement_rank, n, m, M.x.data_ptr(), M.y.data_ptr(), M.G.data_ptr(),
        M.Bt.data_ptr(), out.data_ptr(), _device.stream_handle(M.device)))
    return out


def generator_schur_update(M, pivot):
    """Eliminate one pivot by updating the generators (cauchy.py:140-154).

    O((n+m)p) device work; returns a new CauchyLikeMatrix over the same points.
    """
    i, j = pivot
    r = (M.Bt @ M.G[i]) / (M.x[i] - M.y)
    a = r[j]
    if float(a.abs()) <= PIVOT_REL_TOL * float(r.abs().max()):
        raise ZeroDivisionError(f"pivot ({i}, {j}) is numerically zero")
    c = (M.G @ M.Bt[j]) / (M.x - M.y[j])
    G1 = M.G - torch.outer(c / a, M.G[i])
    Bt1 = M.Bt - torch.outer(r / a, M.Bt[j])
    return CauchyLikeMatrix(M.x, M.y, G1, None, check_points=False, _bt=Bt1.contiguous())


@dataclass
class StructuredPivotTrace:
    """Selected index sets plus sampling statistics (cauchy.py:157-174).

    ``steps`` holds (column, row, pivot) triples when keep_steps=True
    (numpy for host use; ``steps_device`` keeps the (C, R, a) device tensors).
    ``residual`` is the CauchyLikeMatrix of the final generators.
    """

    row_indices: list = field(default_factory=list)
    col_indices: list = field(default_factory=list)
    steps: list = field(default_factory=list)
    proposals: int = 0
    acceptances: int = 0
    exact_fallbacks: int = 0
    bound_sums: list = field(default_factory=list)
    bound_maxes: list = field(default_factory=list)
    tol_stop: bool = False
    degenerate_stop: bool = False
    near_boundary_draws: int = 0
    uniforms_consumed: int = 0
    steps_device: tuple = None
    residual: object = None
    kernel_stats: dict = None

    @property
    def rank(self):
        return len(self.row_indices)

    def factors(self):
        """(L, U) with L[:, t] = c_t / a_t and U[t] = r_t (keep_steps=True)."""
        if self.steps_device is None:
            raise ValueError("factors need keep_steps=True")
        C, R, a = self.steps_device
        k = self.rank
        return (C[:k] / a[:k, None]).T, R[:k]


def structured_eliminate(M, rule, rank, stop_tol=0.0, nu=5.0, plan=None, rng=None,
                         keep_steps=False, *, host_steps=True, time_kernels=False):
    """Pivoted elimination of a Cauchy-like matrix via generator updates
    (cauchy.py:177-256), exact-row-norm (plan=None) path on the device.

    Consumes the caller's RngState exactly as the reference: one uniform for
    the row draw, one for the column draw, one more per column resample.
    """
    if rule not in ("rplu", "c2plu"):
        raise ValueError(f"unknown structured rule {rule!r}")
    if rule == "rplu" and rng is None:
        raise ValueError("structured rplu needs an RngState")
    n, m = M.shape
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    if plan is not None:
        raise CapabilityError(
            "certified-bound rejection sampling (plan) is not on the B200 path yet "
            "(SURVEY §8(f1)); pass plan=None for exact row norms")
    if not isinstance(M, CauchyLikeMatrix):
        raise CapabilityError("structured_eliminate needs a CauchyLikeMatrix")
    cur = M.copy()
    dev = cur.device
    p = cur.displacement_rank
    C = R = A = None
    if keep_steps and rank > 0:
        C = torch.empty((rank, n), dtype=torch.complex128, device=dev)
        R = torch.empty((rank, m), dtype=torch.complex128, device=dev)
        A = torch.empty(rank, dtype=torch.complex128, device=dev)
    block = UniformBlock(rng, 3 * rank) if (rule == "rplu" and rank > 0) else None
    rows = np.zeros(max(rank, 1), dtype=np.int64)
    cols = np.zeros(max(rank, 1), dtype=np.int64)
    bmax = np.zeros(max(rank, 1))
    bsum = np.zeros(max(rank, 1))
    args = _ffi.CauchyArgs(
        rule=_ffi.RULE_IDS[rule], p=p, n=n, m=m, rank=rank, stop_tol=float(stop_tol),
        x=cur.x.data_ptr(), y=cur.y.data_ptr(), G=cur.G.data_ptr(), Bt=cur.Bt.data_ptr(),
        C=C.data_ptr() if C is not None else None, Rrow=R.data_ptr() if R is not None else None,
        a=A.data_ptr() if A is not None else None,
        uniforms=block.pointer() if block else None,
        n_uniforms=block.values.size if block else 0,
        stream=torch.cuda.current_stream(dev).cuda_stream,
        flags=_ffi.FLAG_TIME_KERNELS if time_kernels else 0)
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)
    out = _ffi.CauchyOut(rows=rows.ctypes.data_as(i64p), cols=cols.ctypes.data_as(i64p),
                         bound_maxes=bmax.ctypes.data_as(f64p),
                         bound_sums=bsum.ctypes.data_as(f64p))
    c = _device.ctx(dev)
    status = c._lib.rplu_cauchy_run(c.handle, ctypes.byref(args), ctypes.byref(out))
    if block is not None:
        block.commit(out.uniforms_consumed)
    _ffi.check(status)
    k = int(out.steps_done)
    nb = int(out.bounds_recorded)
    tr = StructuredPivotTrace(
        row_indices=[int(v) for v in rows[:k]], col_indices=[int(v) for v in cols[:k]],
        bound_sums=[float(v) for v in bsum[:nb]], bound_maxes=[float(v) for v in bmax[:nb]],
        tol_stop=bool(out.tol_stop), degenerate_stop=bool(out.degenerate_stop),
        near_boundary_draws=int(out.near_boundary_draws),
        uniforms_consumed=int(out.uniforms_consumed), residual=cur,
        kernel_stats={"masses_ms": out.masses_ms, "masses_launches": int(out.masses_launches),
                      "kernel_launches": int(out.kernel_launches)})
    if C is not None:
        tr.steps_device = (C, R, A)
        if host_steps and k:
            Ch, Rh, Ah = C[:k].cpu().numpy(), R[:k].cpu().numpy(), A[:k].cpu().numpy()
            tr.steps = [(Ch[t], Rh[t], complex(Ah[t])) for t in range(k)]
    return tr
