"""Barycentric rational approximation on the B200 — drop-in for
``rplu.rational`` (pkg/src/rplu/rational.py), SURVEY §8(f4).

``cur_aaa`` picks its support points with one structured pivoted
elimination of the split Loewner matrix (``loewner_build`` ->
``build_plan`` -> ``structured_eliminate(plan=...)``, all on the device),
then solves for the weights once per candidate support set.  ``aaa`` is the
classical greedy loop.  The arithmetic runs in ``librplu_b200.so``:

* ``rplu_loewner_fill`` — the divided-difference matrix of a weight solve
  (rational.py:124-127), numpy-exact elementwise arithmetic;
* ``rplu_bary_eval`` — r(z) with the Cauchy entries 1/(z - t_j) generated in
  registers (rational.py:63-80, the AAA refit :165-169), no nz x k matrix;
* the smallest right singular vector of the Loewner matrix comes from the
  device SVD (cuSOLVER through torch.linalg — a library factorisation, like
  the reference's LAPACK call).

Parity (tests/test_rational_gpu.py): support indices identical to the
reference's, the fitted rational agreeing on the samples to 1e-9 relative
of max|f|.  Weights are compared up to the unit-modulus phase that a
singular vector is only defined up to (the rational is invariant to it).
"""

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _ffi
from .cauchy import loewner_build, structured_eliminate
from .rng import RngState
from .treebounds import build_plan

__all__ = ["BarycentricRational", "SampleSet", "bary_eval", "aaa", "cur_aaa"]

SUPPORT_HIT_TOL = 1e-14        # rational.py:22
_TINY = float(np.finfo(float).tiny)


def _dev_c128(a, dev):
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.complex128).reshape(-1).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.complex128).ravel())).to(dev)


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _bary_kernel(z, t, f, w, hit_tol, mode):
    """rplu_bary_eval on device tensors; returns (values, near_pole or None)."""
    dev = z.device
    out = torch.empty_like(z)
    flags = torch.zeros(z.numel(), dtype=torch.int32, device=dev) if mode == 0 else None
    if z.numel():
        c = _device.ctx(dev)
        _ffi.check(c._lib.rplu_bary_eval(c.handle, z.data_ptr(), z.numel(), t.data_ptr(),
                                         f.data_ptr(), w.data_ptr(), t.numel(), float(hit_tol),
                                         int(mode), out.data_ptr(),
                                         flags.data_ptr() if flags is not None else None,
                                         _stream(dev)))
    return out, flags


def _svd_sv(M):
    """Singular values and right vectors (cuSOLVER; Jacobi first, the
    QR-iteration driver if Jacobi does not converge)."""
    try:
        _, s, Vh = torch.linalg.svd(M, full_matrices=False)
    except RuntimeError:
        _, s, Vh = torch.linalg.svd(M, full_matrices=False, driver="gesvd")
    return s, Vh


def _loewner_weights(support_pts, support_vals, other_pts, other_vals):
    """Weights as the smallest right singular vector of the Loewner matrix
    (rational.py:124-131); device tensors in, (w, L, smin) out."""
    dev = support_pts.device
    k, no = support_pts.numel(), other_pts.numel()
    L = torch.empty((no, k), dtype=torch.complex128, device=dev)
    if no * k:
        c = _device.ctx(dev)
        _ffi.check(c._lib.rplu_loewner_fill(c.handle, other_pts.data_ptr(), other_vals.data_ptr(),
                                            no, support_pts.data_ptr(), support_vals.data_ptr(),
                                            k, L.data_ptr(), _stream(dev)))
    if no >= k:
        # tall: Householder QR, then the SVD of the k x k triangle (same right
        # singular vectors, a fraction of the work on the tall matrix)
        Rm = torch.linalg.qr(L, mode="r")[1] if no > 2 * k else L
        s, Vh = _svd_sv(Rm)
        smin = float(s[-1]) if s.numel() else 0.0
    else:   # fewer equations than unknowns: Vh[-1] spans part of the null space
        _, s, Vh = torch.linalg.svd(L, full_matrices=True)
        smin = 0.0
    w = Vh[-1, :].conj().contiguous()
    return w, L, smin


class BarycentricRational:
    """r(z) = sum_j w_j f_j/(z - t_j) / sum_j w_j/(z - t_j)  (rational.py:25-60).

    Support, values and weights live on the device; the ``support``,
    ``values`` and ``weights`` attributes return host copies as the
    reference's numpy arrays.  Weights are normalised to unit 2-norm.
    """

    def __init__(self, support, values, weights, device=None):
        dev = (support.device if isinstance(support, torch.Tensor) and support.is_cuda
               else _device.require_cuda(device))
        t, f, w = (_dev_c128(a, dev) for a in (support, values, weights))
        if not (t.numel() == f.numel() == w.numel()) or t.numel() == 0:
            raise ValueError("support, values, and weights must match and be nonempty")
        if t.numel() > 1:
            d = (t[:, None] - t[None, :]).abs()
            d.fill_diagonal_(float("inf"))
            if float(d.min()) == 0.0:
                raise ValueError("support points must be pairwise distinct")
        nw = float(torch.linalg.vector_norm(w))
        if nw == 0.0:
            raise ValueError("weights must not all be zero")
        self._t, self._f, self._w = t, f, w / nw
        self._host = None

    def _h(self):
        if self._host is None:
            self._host = tuple(a.cpu().numpy() for a in (self._t, self._f, self._w))
        return self._host

    @property
    def support(self):
        return self._h()[0]

    @property
    def values(self):
        return self._h()[1]

    @property
    def weights(self):
        return self._h()[2]

    @property
    def device(self):
        return self._t.device

    @property
    def degree(self):
        return self._t.numel()

    def __call__(self, z):
        return bary_eval(self, z)

    def eval_flagged(self, z):
        """Evaluate and also report where the denominator underflowed."""
        return _bary_eval_impl(self, z)

    def eval_dev(self, z):
        """Device evaluation: (values, near_pole) tensors for a device z."""
        zv = _dev_c128(z, self.device)
        scale = max(float(self._t.abs().max()), 1.0)
        out, flags = _bary_kernel(zv, self._t, self._f, self._w, SUPPORT_HIT_TOL * scale, 0)
        return out, flags.bool()


def _bary_eval_impl(r, z):
    scalar = np.isscalar(z) or (not isinstance(z, torch.Tensor) and np.asarray(z).ndim == 0) or \
        (isinstance(z, torch.Tensor) and z.dim() == 0)
    out, near = r.eval_dev(z)
    if scalar:
        return complex(out[0].item()), bool(near[0].item())
    if isinstance(z, torch.Tensor):
        return out, near
    return out.cpu().numpy(), near.cpu().numpy()


def bary_eval(r, z):
    """Evaluate a barycentric rational at scalar or array arguments
    (rational.py:83-93); warns when a point lands numerically on a pole."""
    out, near_pole = _bary_eval_impl(r, z)
    if bool(np.any(near_pole.cpu().numpy() if isinstance(near_pole, torch.Tensor) else near_pole)):
        warnings.warn("evaluation point is numerically on a pole", stacklevel=2)
    return out


@dataclass
class SampleSet:
    """Distinct sample points with finite values (rational.py:96-116)."""

    points: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.points = np.asarray(self.points, dtype=np.complex128).ravel()
        self.values = np.asarray(self.values, dtype=np.complex128).ravel()
        if self.points.size != self.values.size:
            raise ValueError("points and values must have equal length")
        if not np.all(np.isfinite(self.values.real)) or not np.all(np.isfinite(self.values.imag)):
            raise ValueError("sample values must be finite")
        if self.points.size != np.unique(self.points).size:
            raise ValueError("sample points must be pairwise distinct")

    @property
    def size(self):
        return self.points.size


def aaa(samples, tol=1e-13, max_degree=100, device=None):
    """Greedy barycentric rational fit (rational.py:134-175).

    Each round moves the worst sample (first index of the maximum of
    |f - r|, as np.argmax) into the support, refits the weights on the
    device and re-evaluates r on the remaining samples with the generated-
    entry kernel.  Returns (rational, error history).
    """
    if samples.size < 2:
        raise ValueError("need at least two samples")
    if tol <= 0:
        raise ValueError("tol must be positive")
    dev = _device.require_cuda(device)
    Z = _dev_c128(samples.points, dev)
    F = _dev_c128(samples.values, dev)
    N = Z.numel()
    fscale = float(F.abs().max())
    remaining = torch.ones(N, dtype=torch.bool, device=dev)
    sup = []
    errors = []
    R = torch.full_like(F, complex(np.mean(samples.values)))
    w = torch.ones(1, dtype=torch.complex128, device=dev)
    for _ in range(min(max_degree, N - 1)):
        rel = torch.where(remaining, (F - R).abs(), torch.full((N,), -1.0, dtype=torch.float64,
                                                                device=dev))
        pick = int(torch.argmax(rel))
        sup.append(pick)
        remaining[pick] = False
        idx = torch.nonzero(remaining).reshape(-1)
        S = torch.tensor(sup, dtype=torch.int64, device=dev)
        w, _, _ = _loewner_weights(Z[S], F[S], Z[idx], F[idx])
        vals, _ = _bary_kernel(Z[idx].contiguous(), Z[S].contiguous(), F[S].contiguous(), w,
                               0.0, 1)
        R = F.clone()
        R[idx] = vals
        err = float((F - R).abs().max())
        errors.append(err)
        if err <= tol * max(fscale, _TINY):
            break
    S = torch.tensor(sup, dtype=torch.int64, device=dev)
    return BarycentricRational(Z[S], F[S], w), np.array(errors)


def cur_aaa(samples, tol=1e-11, rule="rplu", nu=5.0, rng=None, leaf_size=None,
            max_degree=None, device=None):
    """Barycentric fit with support points chosen by structured pivoting
    (rational.py:178-238).

    The random half split consumes ``rng`` exactly as the reference
    (one permutation); the elimination runs on its own stream seeded
    ``rng.seed ^ 0x517CC1B727220A95``.  Returns (rational, side) with side
    "rows", "cols" or "fallback".
    """
    if rng is None:
        raise ValueError("cur_aaa needs an RngState")
    if samples.size < 4:
        raise ValueError("need at least four samples")
    if tol <= 0:
        raise ValueError("tol must be positive")
    dev = _device.require_cuda(device)
    Z, F = samples.points, samples.values
    m = Z.size
    perm = rng.permutation(m)
    half = (m + 1) // 2
    xi, yi = perm[:half], perm[half:]
    L = loewner_build(Z[xi], F[xi], Z[yi], F[yi], device=dev)

    cap = min(L.shape) - 1 if max_degree is None else min(max_degree, min(L.shape) - 1)
    if float(np.max(np.abs(F - F[0]))) == 0.0:
        trace = None   # constant samples: the divided differences all vanish
    else:
        kwargs = {} if leaf_size is None else {"leaf_size": leaf_size}
        plan = build_plan(Z[xi], Z[yi], nu=nu, **kwargs)
        elim_seed = rng.seed ^ 0x517CC1B727220A95
        trace = structured_eliminate(L, rule, cap, stop_tol=tol, nu=nu, plan=plan,
                                     rng=RngState(elim_seed), host_steps=False)
    if trace is None or trace.rank == 0:
        warnings.warn("structured elimination stopped before any pivot; "
                      "falling back to the greedy fit", stacklevel=2)
        return aaa(samples, tol=tol, device=dev)[0], "fallback"

    Zd, Fd = _dev_c128(Z, dev), _dev_c128(F, dev)
    fscale = max(float(np.max(np.abs(F))), _TINY)
    best_err, best_r, best_side = np.inf, None, "rows"
    # An exactly low-rank Loewner matrix stops one pivot short of the support
    # the barycentric form needs: retry one pivot deeper (rational.py:218-237).
    for _attempt in range(4):
        for side, pick in (("rows", xi[trace.row_indices]), ("cols", yi[trace.col_indices])):
            mask = np.ones(m, dtype=bool)
            mask[pick] = False
            P = torch.from_numpy(np.asarray(pick, dtype=np.int64)).to(dev)
            O = torch.from_numpy(np.nonzero(mask)[0]).to(dev)
            w, _, _ = _loewner_weights(Zd[P], Fd[P], Zd[O], Fd[O])
            r = BarycentricRational(Zd[P], Fd[P], w)
            vals, near = r.eval_dev(Zd)
            if bool(near.any()):
                warnings.warn("evaluation point is numerically on a pole", stacklevel=2)
            err = float((vals - Fd).abs().max())
            if err < best_err:
                best_err, best_r, best_side = err, r, side
        if best_err <= 10.0 * tol * fscale or trace.rank >= cap:
            break
        deeper = structured_eliminate(L, rule, min(trace.rank + 1, cap), stop_tol=0.0, nu=nu,
                                      plan=plan, rng=RngState(elim_seed), host_steps=False)
        if deeper.rank <= trace.rank:
            break
        trace = deeper
    return best_r, best_side
