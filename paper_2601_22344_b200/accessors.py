"""Matrix accessor contract, device-resident.

Mirrors ``rplu.accessors`` (pkg/src/rplu/accessors.py:36-90 contract,
:93-131 DenseMatrix, :180-214 CallableOperator): capability flags,
``require`` raising :class:`CapabilityError`, and the conventions
``apply(v) = A @ v``, ``adjoint_apply(v) = A^H @ v``,
``row_norms() = squared row 2-norms``.

B200 difference: a :class:`DenseMatrix` keeps its array in HBM (a torch CUDA
tensor used purely as a buffer) so the pivot loops read it without a host
copy; ``row_norms`` runs the K1 mass kernel.  Host-callable operators
(:class:`CallableOperator`) keep the reference behaviour for callers that use
them directly, but the GPU pivot loops only accept device operators and say
so with a CapabilityError instead of falling back to the CPU.
"""

import numpy as np

__all__ = [
    "CapabilityError",
    "MatrixAccessor",
    "DenseMatrix",
    "CallableOperator",
    "materialize",
    "foreign_dense_array",
    "is_host_accessor",
]

CAPABILITIES = ("apply", "adjoint_apply", "entry", "row", "column", "row_norms")


class CapabilityError(ValueError):
    """An algorithm asked an accessor for an operation it does not support."""


class MatrixAccessor:
    """Base contract (accessors.py:36-90); backends override what they can do."""

    has_apply = False
    has_adjoint_apply = False
    has_entry = False
    has_row = False
    has_column = False
    has_row_norms = False
    #: True when the operator lives in device memory and the B200 kernels can
    #: evaluate it directly.
    on_device = False

    shape = (0, 0)

    def require(self, *names):
        for name in names:
            if not getattr(self, "has_" + name):
                raise CapabilityError(
                    f"{type(self).__name__} does not support '{name.replace('_', '-')}'")

    def apply(self, v):
        raise CapabilityError(f"{type(self).__name__} does not support 'apply'")

    def adjoint_apply(self, v):
        raise CapabilityError(f"{type(self).__name__} does not support 'adjoint-apply'")

    def entry(self, i, j):
        raise CapabilityError(f"{type(self).__name__} does not support 'entry'")

    def row(self, i):
        raise CapabilityError(f"{type(self).__name__} does not support 'row'")

    def column(self, j):
        raise CapabilityError(f"{type(self).__name__} does not support 'column'")

    def row_norms(self):
        raise CapabilityError(f"{type(self).__name__} does not support 'row-norms'")

    @property
    def capabilities(self):
        return frozenset(c for c in CAPABILITIES if getattr(self, "has_" + c))


class DenseMatrix(MatrixAccessor):
    """Dense matrix held in HBM; every capability, exact.

    ``dtype=None`` follows the reference's promotion for numerics parity:
    complex input stays complex128 and real input is computed in float64
    (the reference embeds reals into complex128 with a zero imaginary part,
    which is arithmetically identical).  ``dtype=torch.float32``
    selects the fp32 residual (BASELINE config C3-fp32).
    """

    has_apply = True
    has_adjoint_apply = True
    has_entry = True
    has_row = True
    has_column = True
    has_row_norms = True
    on_device = True

    def __init__(self, array, dtype=None, device=None):
        from . import _device
        t = _device.as_device_matrix(array, dtype=dtype, device=device, copy=True)
        if not bool(_device.torch.isfinite(t).all()):
            raise ValueError("matrix entries must be finite")
        self.tensor = t
        self.shape = tuple(t.shape)

    @property
    def array(self):
        """Host copy (numpy), as the reference's ``DenseMatrix.array``."""
        return self.tensor.cpu().numpy()

    def apply(self, v):
        from . import _device
        return _device.matvec(self.tensor, v, adjoint=False)

    def adjoint_apply(self, v):
        from . import _device
        return _device.matvec(self.tensor, v, adjoint=True)

    def entry(self, i, j):
        return complex(self.tensor[i, j].item())

    def row(self, i):
        return self.tensor[i, :].cpu().numpy().copy()

    def column(self, j):
        return self.tensor[:, j].cpu().numpy().copy()

    def row_norms(self):
        from . import _device
        return _device.row_masses(self.tensor).cpu().numpy()

    def col_norms(self):
        t = self.tensor
        return (t.real ** 2 + (t.imag ** 2 if t.is_complex() else 0)).sum(0).cpu().numpy()


class CallableOperator(MatrixAccessor):
    """Implicit operator defined by host matvec callables (accessors.py:180-214).

    Only the capabilities whose callables are supplied are advertised.  Host
    callables cannot be evaluated by the B200 kernels, so the GPU pivot loops
    reject this type with a CapabilityError (there is no CPU fallback).
    """

    def __init__(self, shape, apply_fn, adjoint_fn=None, row_norms_fn=None, col_norms_fn=None):
        self.shape = tuple(shape)
        self._apply = apply_fn
        self._adjoint = adjoint_fn
        self._row_norms = row_norms_fn
        self._col_norms = col_norms_fn
        self.has_apply = apply_fn is not None
        self.has_adjoint_apply = adjoint_fn is not None
        self.has_row_norms = row_norms_fn is not None

    def apply(self, v):
        return self._apply(v)

    def adjoint_apply(self, v):
        if self._adjoint is None:
            return super().adjoint_apply(v)
        return self._adjoint(v)

    def row_norms(self):
        if self._row_norms is None:
            return super().row_norms()
        return np.asarray(self._row_norms(), dtype=float)


def foreign_dense_array(A):
    """The host array of a dense accessor that is not this package's
    :class:`DenseMatrix` -- e.g. the reference's ``rplu.DenseMatrix``
    (accessors.py:93-131 keeps it in ``.array``) -- else None.  Lets the
    reference's own objects cross the boundary (cli.py:150 passes one to
    eliminate)."""
    if isinstance(A, DenseMatrix) or isinstance(A, np.ndarray):
        return None
    arr = getattr(A, "array", None)
    if isinstance(arr, np.ndarray) and arr.ndim == 2:
        return arr
    return None


def is_host_accessor(A):
    """Duck-typed accessor with host callables (the reference's
    MatrixAccessor family: ``shape`` plus ``apply``)."""
    if isinstance(A, MatrixAccessor):
        return not getattr(A, "on_device", False)
    return hasattr(A, "shape") and callable(getattr(A, "apply", None)) and \
        not isinstance(A, np.ndarray)


def materialize(acc):
    """Dense host array of an accessor (desk-scale helper)."""
    if isinstance(acc, DenseMatrix):
        return acc.array
    if hasattr(acc, "materialize"):
        return acc.materialize()
    n, m = acc.shape
    acc.require("apply")
    cols = []
    for j in range(m):
        e = np.zeros(m, dtype=np.complex128)
        e[j] = 1.0
        cols.append(np.asarray(acc.apply(e)))
    return np.column_stack(cols)
