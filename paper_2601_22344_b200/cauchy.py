"""Cauchy-like matrices and structured RPLU on the B200 — drop-in for
``rplu.cauchy`` (pkg/src/rplu/cauchy.py).

``CauchyLikeMatrix`` keeps its O((n+m)p) generators in HBM: x[n], y[m]
(complex128), G (n x p, row-major as the reference's C-order G) and B stored
as Bt (m x p, i.e. the reference's F-order B, column j contiguous).
``structured_eliminate`` with ``plan=None`` runs the exact-norm Alg 3 loop
entirely on the device (K5 generated-entry row masses, K2 selects, K6 row /
column generation and generator update) through ``rplu_cauchy_run``; with a
plan (certified tree bounds + rejection sampling) it runs the
reference's proposal / acceptance loop and uniform stream (cauchy.py:259-277)
over device bound kernels (``csrc/tree.cu``) and the same K6 row / update
kernels.  ``generator_schur_update`` is the single-step K6 update.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _ffi
from .accessors import CapabilityError, MatrixAccessor
from .rng import UniformBlock

__all__ = ["CauchyLikeMatrix", "StructuredPivotTrace", "generator_schur_update",
           "exact_row_norms", "structured_eliminate", "loewner_build",
           "MAX_DISPLACEMENT_RANK", "PIVOT_REL_TOL"]

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


def tree_bounds_device(plan, M):
    """Certified upper bounds of M's squared row norms from a plan (Alg C.2),
    as a float64 CUDA tensor (``rplu_tree_bounds``)."""
    from .treebounds import device_plan
    dp = device_plan(plan, M.device)
    n, m = M.shape
    out = torch.empty(n, dtype=torch.float64, device=M.device)
    s = _ffi.TreePlan(
        n=n, m=m, p=M.displacement_rank, n_tleaves=dp.n_tleaves,
        tperm=dp.tperm.data_ptr(), tstart=dp.tstart.data_ptr(),
        agg_start=dp.agg_start.data_ptr(), agg_node=dp.agg_node.data_ptr(),
        agg_alpha=dp.agg_alpha.data_ptr(), ex_start=dp.ex_start.data_ptr(),
        ex_leaf=dp.ex_leaf.data_ptr(), n_snodes=dp.n_snodes, n_sleaves=dp.n_sleaves,
        spts=dp.spts.data_ptr(), sstart=dp.sstart.data_ptr(), cstart=dp.cstart.data_ptr(),
        cidx=dp.cidx.data_ptr(), leaf_node=dp.leaf_node.data_ptr(),
        lvl_nodes=dp.lvl_nodes.data_ptr(), lvl_start=dp.lvl_start.ctypes.data,
        n_levels=dp.n_levels)
    c = _device.ctx(M.device)
    _ffi.check(c._lib.rplu_tree_bounds(c.handle, ctypes.byref(s), M.x.data_ptr(), M.y.data_ptr(),
                                       M.G.data_ptr(), M.Bt.data_ptr(), out.data_ptr(),
                                       _device.stream_handle(M.device)))
    return out


def generator_schur_update(M, pivot):
    """Eliminate one pivot by updating the generators (cauchy.py:140-154).

    O((n+m)p) device work in the K6 kernels the plan path uses
    (``rplu_cauchy_plan_row`` then ``rplu_cauchy_plan_update``: numpy-exact
    complex products and Smith division): r = row i, the relative zero-pivot
    guard |r_j| <= 1e-14 max|r| (ZeroDivisionError), then
    G1 = G - (c / a) G_i and B1 = B - B_:,j (r / a) with c = column j.
    Returns a new CauchyLikeMatrix over the same points (the input's
    generators are not modified, as the reference allocates new ones).
    """
    i, j = int(pivot[0]), int(pivot[1])
    n, m = M.shape
    if not (0 <= i < n and 0 <= j < m):
        raise IndexError(f"pivot ({i}, {j}) out of range for shape {(n, m)}")
    dev = M.device
    c = _device.ctx(dev)
    stream_h = _device.stream_handle(dev)
    G1 = M.G.clone()
    Bt1 = M.Bt.clone()
    rbuf = torch.empty(m, dtype=torch.complex128, device=dev)
    wbuf = torch.empty(m, dtype=torch.float64, device=dev)
    out3 = np.zeros(3)
    p = M.displacement_rank
    _ffi.check(c._lib.rplu_cauchy_plan_row(
        c.handle, p, n, m, M.x.data_ptr(), M.y.data_ptr(), G1.data_ptr(), Bt1.data_ptr(), i,
        rbuf.data_ptr(), wbuf.data_ptr(), None, out3.ctypes.data, stream_h))
    a = complex(rbuf[j].item())
    if abs(a) <= PIVOT_REL_TOL * float(out3[1]):
        raise ZeroDivisionError(f"pivot ({i}, {j}) is numerically zero")
    _ffi.check(c._lib.rplu_cauchy_plan_update(
        c.handle, p, n, m, M.x.data_ptr(), M.y.data_ptr(), G1.data_ptr(), Bt1.data_ptr(), i, j,
        rbuf.data_ptr(), None, None, stream_h))
    return CauchyLikeMatrix(M.x, M.y, G1, None, check_points=False, _bt=Bt1)


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
    #: plan path: proposals whose norm / bound test rho >= u_i was decided
    #: within 1e-12 relative (exact-interaction leaves make u_i == rho in
    #: exact arithmetic, so whether an acceptance uniform is drawn is a
    #: rounding-level tie, like a draw on a CDF boundary)
    near_tie_acceptances: int = 0
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


class _UniformCursor:
    """Uniforms from a pre-drawn block, committed exactly at the end."""

    def __init__(self, rng, cap):
        self.block = UniformBlock(rng, cap) if rng is not None else None
        self.used = 0

    def next(self):
        if self.used >= self.block.values.size:     # extend (rare): keep exactness
            extra = self.block._gen.random(self.block.values.size)
            self.block.values = np.concatenate([self.block.values, extra])
        u = float(self.block.values[self.used])
        self.used += 1
        return u

    def commit(self):
        if self.block is not None:
            self.block.commit(self.used)


def _row_dev(cur, i):
    return (cur.Bt @ cur.G[i]) / (cur.x[i] - cur.y)


def _column_dev(cur, j):
    return (cur.G @ cur.Bt[j]) / (cur.x - cur.y[j])


def _structured_eliminate_plan(M, rule, rank, stop_tol, nu, plan, rng, keep_steps, host_steps):
    """Alg 3 with certified tree bounds and rejection sampling
    (cauchy.py:177-277, plan branch).

    Per step: device bounds u (``rplu_tree_bounds``), max/sum, stop rules;
    rplu: propose i ~ u (one uniform), accept when rho = ||r_i||^2 >= u_i or
    with probability rho/u_i (one more uniform); after 64*nu proposals fall
    back to exact norms (K5) with a warning; column j ~ |r|^2; relative
    zero-pivot guard with one column resample; generator update on the
    device.  The proposal/acceptance counters match the reference's trace.
    """
    import warnings

    from .rng import sample_index as _si
    tgt, src = plan.target_tree, plan.source_tree
    if tgt.points.size != M.shape[0] or src.points.size != M.shape[1]:
        raise ValueError("generator dimensions do not match the plan's points")
    cur = M.copy()
    n, m = M.shape
    cap = int(REJECTION_CAP_FACTOR * max(nu, 1.0))
    stream = _UniformCursor(rng if rule == "rplu" else None, max(8, (2 * cap + 3) * rank))
    tr = StructuredPivotTrace(residual=cur)

    def sample_index(w, u):
        i, near = _si(w, u, return_near=True)
        tr.near_boundary_draws += int(near)
        return i
    u0_max = None
    p = cur.displacement_rank
    dev = cur.device
    c = _device.ctx(dev)
    stream_h = _device.stream_handle(dev)
    rbuf = torch.empty(m, dtype=torch.complex128, device=dev)
    wbuf = torch.empty(m, dtype=torch.float64, device=dev)
    C = torch.empty((rank, n), dtype=torch.complex128, device=dev) if keep_steps else None
    R = torch.empty((rank, m), dtype=torch.complex128, device=dev) if keep_steps else None
    A_steps = []
    out3 = np.zeros(3)
    last_rmax = [0.0]

    def row(i, u):
        """pivot row i into rbuf / wbuf; returns (||r||^2, max|r|, u_i)"""
        _ffi.check(c._lib.rplu_cauchy_plan_row(
            c.handle, p, n, m, cur.x.data_ptr(), cur.y.data_ptr(), cur.G.data_ptr(),
            cur.Bt.data_ptr(), int(i), rbuf.data_ptr(), wbuf.data_ptr(),
            u.data_ptr() if u is not None else None, out3.ctypes.data, stream_h))
        last_rmax[0] = float(out3[1])
        return float(out3[0]), float(out3[1]), float(out3[2])

    out5 = np.zeros(5)

    def propose(u, uniform):
        """i ~ u and its pivot row in one host synchronisation; returns
        (i, ||r||^2, u_i)"""
        _ffi.check(c._lib.rplu_cauchy_plan_propose(
            c.handle, p, n, m, cur.x.data_ptr(), cur.y.data_ptr(), cur.G.data_ptr(),
            cur.Bt.data_ptr(), u.data_ptr(), float(uniform), rbuf.data_ptr(), wbuf.data_ptr(),
            out5.ctypes.data, stream_h))
        tr.near_boundary_draws += int(out5[1])
        last_rmax[0] = float(out5[3])
        return int(out5[0]), float(out5[2]), float(out5[4])

    val2 = np.zeros(2)

    def draw_column(uniform):
        """j ~ |r|^2 and the pivot value r_j in one host synchronisation"""
        j64, near = ctypes.c_int64(-1), ctypes.c_int32(0)
        _ffi.check(c._lib.rplu_sample_index_gather(
            c.handle, ctypes.c_void_p(wbuf.data_ptr()), m, float(uniform),
            ctypes.c_void_p(rbuf.data_ptr()), ctypes.byref(j64), ctypes.byref(near),
            val2.ctypes.data, stream_h))
        tr.near_boundary_draws += int(near.value)
        return int(j64.value), complex(val2[0], val2[1])
    try:
        for _ in range(rank):
            u = tree_bounds_device(plan, cur)
            umax, usum = torch.stack([u.max(), u.sum()]).tolist()   # one host sync
            tr.bound_maxes.append(umax)
            tr.bound_sums.append(usum)
            u0_max = umax if u0_max is None else u0_max
            if umax <= 0.0:
                tr.degenerate_stop = True
                break
            if stop_tol > 0 and umax <= (stop_tol ** 2) * u0_max:
                tr.tol_stop = True
                break
            if rule == "c2plu":
                i = int(torch.argmax(u))
                row(i, None)
            else:
                i = None
                for _p in range(cap):
                    ii, rho, ui = propose(u, stream.next())
                    tr.proposals += 1
                    if abs(rho - ui) <= 1e-12 * ui:
                        tr.near_tie_acceptances += 1
                    if rho >= ui or stream.next() <= rho / ui:
                        tr.acceptances += 1
                        i = ii
                        break
                if i is None:
                    tr.exact_fallbacks += 1
                    warnings.warn("rejection sampling exceeded its proposal budget; this step "
                                  "used exact row norms (possible bound violation)",
                                  stacklevel=3)
                    i = sample_index(exact_row_norms_device(cur), stream.next())
                    row(i, None)
            rmax = last_rmax[0]
            if rule == "c2plu":
                j = int(torch.argmax(wbuf))
                a = complex(rbuf[j].item())
            else:
                j, a = draw_column(stream.next())
            thr = PIVOT_REL_TOL * rmax
            if abs(a) <= thr:
                if rule == "c2plu":
                    raise ZeroDivisionError(f"pivot ({i}, {j}) is numerically zero")
                j, a = draw_column(stream.next())
                if abs(a) <= thr:
                    raise ZeroDivisionError(
                        f"pivot ({i}, {j}) is numerically zero after resampling")
            t = len(tr.row_indices)
            cbuf = C[t] if keep_steps else None
            rout = R[t] if keep_steps else None
            _ffi.check(c._lib.rplu_cauchy_plan_update(
                c.handle, p, n, m, cur.x.data_ptr(), cur.y.data_ptr(), cur.G.data_ptr(),
                cur.Bt.data_ptr(), int(i), int(j), rbuf.data_ptr(),
                cbuf.data_ptr() if cbuf is not None else None,
                rout.data_ptr() if rout is not None else None, stream_h))
            tr.row_indices.append(int(i))
            tr.col_indices.append(int(j))
            if keep_steps:
                A_steps.append(a)
    finally:
        stream.commit()
    tr.uniforms_consumed = stream.used
    k = len(tr.row_indices)
    if keep_steps and k:
        A = torch.tensor(A_steps, dtype=torch.complex128, device=dev)
        tr.steps_device = (C[:k], R[:k], A)
        if host_steps:
            Ch, Rh = _device.to_numpy(C[:k]), _device.to_numpy(R[:k])
            tr.steps = [(Ch[t], Rh[t], A_steps[t]) for t in range(k)]
    return tr


def structured_eliminate(M, rule, rank, stop_tol=0.0, nu=5.0, plan=None, rng=None,
                         keep_steps=False, *, host_steps=True, time_kernels=False,
                         persistent=True):
    """Pivoted elimination of a Cauchy-like matrix via generator updates
    (cauchy.py:177-256), exact-row-norm (plan=None) path on the device.

    Consumes the caller's RngState exactly as the reference: one uniform for
    the row draw, one for the column draw, one more per column resample.
    Small problems (the generators fit in shared memory, displacement rank
    <= 2) run the whole loop as one resident cooperative launch;
    ``persistent=False`` keeps the per-step kernels (K5 / select / update).
    """
    if rule not in ("rplu", "c2plu"):
        raise ValueError(f"unknown structured rule {rule!r}")
    if rule == "rplu" and rng is None:
        raise ValueError("structured rplu needs an RngState")
    n, m = M.shape
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    if not isinstance(M, CauchyLikeMatrix):
        raise CapabilityError("structured_eliminate needs a CauchyLikeMatrix")
    if plan is not None:
        from .treebounds import InteractionPlan
        if not isinstance(plan, InteractionPlan):
            raise ValueError("plan must be an InteractionPlan (treebounds.build_plan)")
        return _structured_eliminate_plan(M, rule, rank, stop_tol, nu, plan, rng, keep_steps,
                                          host_steps)
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
        flags=(_ffi.FLAG_TIME_KERNELS if time_kernels else 0)
        | (0 if persistent else _ffi.FLAG_STEPWISE))
    i64p = ctypes.POINTER(ctypes.c_int64)
    f64p = ctypes.POINTER(ctypes.c_double)
    out = _ffi.CauchyOut(rows=rows.ctypes.data_as(i64p), cols=cols.ctypes.data_as(i64p),
                         bound_maxes=bmax.ctypes.data_as(f64p),
                         bound_sums=bsum.ctypes.data_as(f64p))
    c = _device.ctx(dev)
    pre = None
    if C is not None and host_steps and rank * (n + m) * 16 >= (1 << 20):
        # pin the host copies of the kept steps while the loop runs
        pre = _device.PinnedPrefetch([((rank, n), torch.complex128),
                                      ((rank, m), torch.complex128)])
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
            Ch = _device.copy_to_host(C[:k], pre.get(0) if pre else None)
            Rh = _device.copy_to_host(R[:k], pre.get(1) if pre else None)
            Ah = A[:k].cpu().numpy()
            tr.steps = [(Ch[t], Rh[t], complex(Ah[t])) for t in range(k)]
    return tr


def _host_c128(a):
    if isinstance(a, torch.Tensor):
        return a.detach().to("cpu", torch.complex128).reshape(-1).numpy()
    return np.asarray(a, dtype=np.complex128).ravel()


def loewner_build(x, f_x, y, f_y, device=None):
    """Divided-difference matrix (f_x[i] - f_y[j]) / (x[i] - y[j]) as a
    displacement-rank-2 CauchyLikeMatrix (cauchy.py:280-306).

    Generators G = [f_x/alpha, alpha], B = [alpha; -f_y/alpha] with the
    balanced scale alpha = sqrt(max |f|) (alpha = 1 with a warning when every
    sample is zero).  The O(n + m) scale search runs on the samples as given
    (host arrays, as SampleSet holds them); the generators are formed on the
    device, dividing by alpha as numpy does for a real-valued complex divisor
    (times 1/alpha, bit for bit).
    """
    import warnings
    x, y, fx, fy = (_host_c128(a) for a in (x, y, f_x, f_y))
    if x.size != fx.size or y.size != fy.size:
        raise ValueError("points and values must have matching lengths")
    for arr in (fx, fy):
        if not np.all(np.isfinite(arr.real)) or not np.all(np.isfinite(arr.imag)):
            raise ValueError("sample values must be finite")
    fmax = max(float(np.max(np.abs(fx), initial=0.0)), float(np.max(np.abs(fy), initial=0.0)))
    if fmax == 0.0:
        warnings.warn("all sample values are zero; scaling factor set to 1", stacklevel=2)
        alpha = 1.0
    else:
        alpha = float(np.sqrt(fmax))
    dev = _device.require_cuda(device)
    inv = 1.0 / alpha
    fxd = _c128(fx, dev)
    fyd = _c128(fy, dev)
    G = torch.stack([fxd * inv, torch.full_like(fxd, alpha)], dim=1).contiguous()
    Bt = torch.stack([torch.full_like(fyd, alpha), -(fyd * inv)], dim=1).contiguous()
    return CauchyLikeMatrix(x, y, G, None, device=dev, _bt=Bt)
