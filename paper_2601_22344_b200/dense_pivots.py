"""Dense pivoted elimination (Alg 1) on the B200 — drop-in for
``rplu.dense_pivots.eliminate`` (pkg/src/rplu/dense_pivots.py:129-209).

Same signature, validation order, exception classes, uniform consumption
(row draw then column draw, 2 per step, a resampled pair on a zero pivot,
dense_pivots.py:116-117, :178-184) and trace fields.  The residual lives in
HBM and the whole step loop runs in ``librplu_b200.so``:

* K1 row masses (step 0), K2 single-CTA two-stage inverse-CDF select,
  K3 fused rank-1 Schur update + next-step masses (one HBM pass per step).

Rules: ``rplu`` (the north-star path), and the greedy siblings ``c2plu``
and ``cplu`` on the same kernels.  The PSD rules
(rpcholesky / greedy-cholesky / srplu) are outside the hot-path scope and
raise CapabilityError rather than falling back to the CPU.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _ffi
from .accessors import CapabilityError, DenseMatrix
from .rng import RngState, UniformBlock

__all__ = ["PivotRule", "EliminationTrace", "eliminate", "RULES"]

RULES = ("rplu", "cplu", "c2plu", "rpcholesky", "greedy-cholesky", "srplu")
_RANDOM_RULES = ("rplu", "rpcholesky", "srplu")
_DEVICE_RULES = ("rplu", "cplu", "c2plu")


@dataclass
class PivotRule:
    """A pivot selection rule; random rules carry their own RngState
    (dense_pivots.py:48-59)."""

    tag: str
    rng: RngState = None

    def __post_init__(self):
        if self.tag not in RULES:
            raise ValueError(f"unknown pivot rule {self.tag!r}")
        if self.tag in _RANDOM_RULES and self.rng is None:
            raise ValueError(f"rule {self.tag!r} needs an RngState")


class EliminationTrace:
    """Pivot sequence plus factor blocks and residual norm history
    (dense_pivots.py:62-83).

    ``L`` / ``U`` / ``residual`` are numpy arrays for host inputs and CUDA
    tensors for device inputs.  ``residual`` is materialized on first access
    (it is the full n x m matrix).  Extra diagnostics: ``near_boundary_draws``
    (draws within 1e-12 relative of a CDF boundary) and ``uniforms_consumed``.
    """

    def __init__(self, pivots, L, U, resid_fro, residual, steps, resid_trace=None,
                 clean_early_stop=False, tol_stop=False, near_boundary_draws=0,
                 uniforms_consumed=0, host=True):
        self.pivots = pivots
        self.L = L
        self.U = U
        self.resid_fro = resid_fro
        self._residual = residual
        self.steps = steps
        self.resid_trace = resid_trace
        self.clean_early_stop = clean_early_stop
        self.tol_stop = tol_stop
        self.near_boundary_draws = near_boundary_draws
        self.uniforms_consumed = uniforms_consumed
        self._host = host

    @property
    def residual(self):
        r = self._residual
        if self._host and isinstance(r, torch.Tensor):
            r = self._residual = _device.to_numpy(r)
        return r

    @property
    def residual_device(self):
        return self._residual

    def approximation(self):
        return self.L @ self.U

    def __repr__(self):
        return (f"EliminationTrace(steps={self.steps}, pivots={self.pivots[:4]}..., "
                f"clean_early_stop={self.clean_early_stop}, tol_stop={self.tol_stop})")


def _input_tensor(A, compute_dtype):
    """(device matrix, host-results?) -- accessor inputs (this package's
    DenseMatrix, or the reference's own rplu.DenseMatrix) return numpy
    results as the reference does; only CUDA tensors keep them on device."""
    if isinstance(A, DenseMatrix):
        t = A.tensor
        if compute_dtype is not None:
            t = t.to(_device._resolve_dtype(t.is_complex(), compute_dtype))
        return t, True, t is not A.tensor
    if isinstance(A, torch.Tensor) and A.is_cuda:
        t = _device.as_device_matrix(A, dtype=compute_dtype, copy=False)
        return t, False, t is not A
    # host arrays (and the reference's DenseMatrix): the upload is private
    return _device.as_device_matrix(A, dtype=compute_dtype, copy=False), True, True


def eliminate(A, rule, steps, stop_tol=0.0, *, compute_dtype=None, overwrite_a=False,
              return_device=None, time_kernels=False, update="auto", persistent=True,
              fused_updates=False, gram_masses=True):
    """Run pivoted elimination for up to ``steps`` pivots (dense_pivots.py:129).

    Stops early, with a flag, when the residual Frobenius norm falls to
    ``stop_tol`` times the input norm, or cleanly when the residual is
    exactly drained first.  Zero pivots are resampled once, then
    ZeroDivisionError.

    Keyword-only B200 extensions: ``compute_dtype`` (None = reference
    promotion; torch.float32 for the fp32 residual), ``overwrite_a`` (reuse a
    CUDA input tensor as the residual buffer instead of copying it), and
    ``return_device`` (keep L/U/residual as CUDA tensors; default: True iff
    the input was a CUDA tensor -- numpy arrays and DenseMatrix accessors,
    ours or the reference's, get numpy results), ``time_kernels`` (bracket the K2/K3 launches
    with CUDA events; results in ``trace.kernel_stats``), ``update``
    ("auto" | "eager" | "lazy": update the residual every step, or apply the
    pending rank-1 terms on the fly and write R every few steps — about half
    the HBM traffic; "auto" = lazy when R does not fit in L2),
    ``persistent`` (False: per-step K2/K3 launches even where an L2-resident
    residual would run the whole loop as one persistent cooperative launch),
    ``fused_updates`` (delayed-update loop: apply each pending term with one
    FMA instead of the reference's multiply-then-subtract; L/U then agree
    with the reference to rounding (the north star's 1e-10) instead of bit
    for bit; measured no faster at C3 -- the pass is shared-memory / power
    bound -- so off by default).  The eager and the resident loops always
    use the reference's rounding.  ``gram_masses`` (fp64 delayed-update
    loop, default True): the per-step sampling masses come from the Gram
    form |r0 - sum_s L_s U_s|^2 (one dot product per element instead of
    applying the pending terms, flush every 16 steps); L, U and the residual
    are unchanged (bit-identical to the eager loop), the masses agree to
    rounding.
    """
    if update not in ("auto", "eager", "lazy"):
        raise ValueError(f"unknown update mode {update!r}")
    if isinstance(rule, str):
        rule = PivotRule(rule)
    if rule.tag not in _DEVICE_RULES:
        raise CapabilityError(
            f"rule {rule.tag!r} is not on the B200 RPLU path (supported: {_DEVICE_RULES})")
    src, host_in, private = _input_tensor(A, compute_dtype)
    n, m = src.shape
    if not 0 <= steps <= min(n, m):
        raise ValueError(f"steps {steps} out of range [0, {min(n, m)}]")
    if stop_tol < 0:
        raise ValueError("stop_tol must be nonnegative")
    if return_device is None:
        return_device = not host_in

    dev = src.device
    vec = _device.vec_of(src.dtype)
    if (overwrite_a or private) and src.is_contiguous() and m % vec == 0:
        buf, R = src, src    # the conversion already made a private copy
    else:
        buf, R = _device.padded_residual(src)
    ld = buf.stride(0)
    ldu = ((m + vec - 1) // vec) * vec
    Lt = torch.empty((max(steps, 1), n), dtype=src.dtype, device=dev)
    U = torch.empty((max(steps, 1), ldu), dtype=src.dtype, device=dev)

    block = None
    if rule.tag == "rplu" and steps > 0:
        block = UniformBlock(rule.rng, 4 * steps)

    pivots = np.zeros(2 * max(steps, 1), dtype=np.int64)
    resid = np.zeros(steps + 1, dtype=np.float64)
    args = _ffi.DenseArgs(
        dtype=_device.DTYPE_IDS[src.dtype], rule=_ffi.RULE_IDS[rule.tag],
        n=n, m=m, ld=ld, steps=steps, stop_tol=float(stop_tol),
        R=buf.data_ptr(), Lt=Lt.data_ptr(), U=U.data_ptr(), ldu=ldu,
        uniforms=block.pointer() if block else None,
        n_uniforms=block.values.size if block else 0,
        stream=torch.cuda.current_stream(dev).cuda_stream,
        flags=((_ffi.FLAG_TIME_KERNELS if time_kernels else 0)
               | {"auto": 0, "eager": _ffi.FLAG_EAGER, "lazy": _ffi.FLAG_LAZY}[update]
               | (0 if persistent else _ffi.FLAG_STEPWISE)
               | (0 if fused_updates else _ffi.FLAG_EXACT)
               | (0 if gram_masses else _ffi.FLAG_NO_GRAM)))
    out = _ffi.DenseOut(pivots=pivots.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        resid_fro=resid.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    c = _device.ctx(dev)
    # host results: pin their buffers while the loop runs
    pre = None
    if not return_device and steps * (n + m) * src.element_size() >= (1 << 20):
        pre = _device.PinnedPrefetch([((steps, n), src.dtype), ((steps, m), src.dtype)])
    status = c._lib.rplu_dense_run(c.handle, ctypes.byref(args), ctypes.byref(out))
    if block is not None:
        # the reference consumed exactly these draws, even when it raised
        block.commit(out.uniforms_consumed)
    _ffi.check(status)

    k = int(out.steps_done)
    piv = [(int(pivots[2 * t]), int(pivots[2 * t + 1])) for t in range(k)]
    Ld = Lt[:k].T
    Ud = U[:k, :m]
    if return_device:
        L_out, U_out = Ld, Ud
    else:
        L_out = _device.copy_to_host(Lt[:k], pre.get(0) if pre else None).T
        U_out = _device.copy_to_host(Ud, pre.get(1) if pre else None)
    trace = EliminationTrace(
        pivots=piv, L=L_out, U=U_out, resid_fro=resid[:k + 1].copy(), residual=R, steps=k,
        resid_trace=None, clean_early_stop=bool(out.clean_early_stop),
        tol_stop=bool(out.tol_stop), near_boundary_draws=int(out.near_boundary_draws),
        uniforms_consumed=int(out.uniforms_consumed), host=not return_device)
    trace.kernel_stats = {"sweep_ms": out.sweep_ms, "select_ms": out.select_ms,
                          "sweep_bytes": out.sweep_bytes, "lazy_block": int(out.lazy_block),
                          "sweep_launches": int(out.sweep_launches),
                          "kernel_launches": int(out.kernel_launches)}
    return trace
