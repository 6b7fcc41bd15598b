"""Device-resident operators for the matrix-free CUR path.

``GaussianKernelOperator`` is BASELINE configs[4]'s nonsymmetric Gaussian
kernel A_ij = exp(-|p_i - q_j|^2 / (2 h^2)) on points p_i in [0,1]^3 and
q_j from a mixture: only the 3-D points live in HBM (48 MB at n = 2e6) and
every apply regenerates the entries (K7/K8 kernels in ``librplu_b200.so``).
It implements the reference accessor contract (accessors.py:36-90):
apply, adjoint_apply, row_norms, entry/row/column.

``DeviceOperator`` is the internal protocol ``cur_build`` drives (device
tensors in and out); ``as_device_operator`` adapts a DenseMatrix (cuBLAS
GEMV) or a GaussianKernelOperator (hand-written kernels).
"""

import ctypes

import numpy as np
import torch

from . import _device, _ffi
from .accessors import CapabilityError, DenseMatrix, MatrixAccessor, foreign_dense_array

__all__ = ["GaussianKernelOperator", "as_device_operator"]


class _GaussOpStruct(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("P", ctypes.c_void_p),
                ("Q", ctypes.c_void_p), ("h", ctypes.c_double)]


class GaussianKernelOperator(MatrixAccessor):
    """A_ij = exp(-|p_i - q_j|^2 / (2 h^2)) with P (n x 3), Q (m x 3) on the device."""

    has_apply = True
    has_adjoint_apply = True
    has_entry = True
    has_row = True
    has_column = True
    has_row_norms = True
    on_device = True

    def __init__(self, P, Q, h=0.1, device=None):
        dev = _device.require_cuda(device)
        self.P = torch.as_tensor(np.asarray(P, dtype=np.float64) if not isinstance(P, torch.Tensor)
                                 else P, dtype=torch.float64).to(dev).contiguous()
        self.Q = torch.as_tensor(np.asarray(Q, dtype=np.float64) if not isinstance(Q, torch.Tensor)
                                 else Q, dtype=torch.float64).to(dev).contiguous()
        if self.P.dim() != 2 or self.P.shape[1] != 3 or self.Q.dim() != 2 or self.Q.shape[1] != 3:
            raise ValueError("points must be (n, 3) and (m, 3) arrays")
        if not h > 0:
            raise ValueError("bandwidth h must be positive")
        self.h = float(h)
        self.shape = (self.P.shape[0], self.Q.shape[0])
        self._s = _GaussOpStruct(self.shape[0], self.shape[1], self.P.data_ptr(),
                                 self.Q.data_ptr(), self.h)
        self.last_kernel_ms = 0.0

    @property
    def device(self):
        return self.P.device

    # -- device primitives (torch in / torch out) -------------------------
    def _ctx(self):
        return _device.ctx(self.device)

    def _stream(self):
        return _device.stream_handle(self.device)

    def apply_dev(self, v, adjoint=False, timed=False):
        c = self._ctx()
        v = v.to(device=self.device, dtype=torch.float64).contiguous()
        out = torch.empty(self.shape[1] if adjoint else self.shape[0], dtype=torch.float64,
                          device=self.device)
        ms = ctypes.c_double(0.0)
        _ffi.check(c._lib.rplu_gauss_apply(c.handle, ctypes.byref(self._s), int(adjoint),
                                           v.data_ptr(), out.data_ptr(),
                                           ctypes.byref(ms) if timed else None, self._stream()))
        self.last_kernel_ms = ms.value
        return out

    def row_norms_dev(self):
        c = self._ctx()
        out = torch.empty(self.shape[0], dtype=torch.float64, device=self.device)
        _ffi.check(c._lib.rplu_gauss_row_norms(c.handle, ctypes.byref(self._s), out.data_ptr(),
                                               self._stream()))
        return out

    def line_dev(self, axis, index):
        c = self._ctx()
        out = torch.empty(self.shape[1] if axis == 0 else self.shape[0], dtype=torch.float64,
                          device=self.device)
        _ffi.check(c._lib.rplu_gauss_line(c.handle, ctypes.byref(self._s), int(axis),
                                          int(index), out.data_ptr(), self._stream()))
        return out

    def restricted_dev(self, axis, sel, w):
        c = self._ctx()
        out = torch.empty(self.shape[1] if axis == 0 else self.shape[0], dtype=torch.float64,
                          device=self.device)
        k = int(sel.numel())
        w = w.to(device=self.device, dtype=torch.float64).contiguous()
        _ffi.check(c._lib.rplu_gauss_restricted(c.handle, ctypes.byref(self._s), int(axis),
                                                sel.data_ptr() if k else None,
                                                w.data_ptr() if k else None, k,
                                                out.data_ptr(), self._stream()))
        return out

    def block_cols_dev(self, j0, j1):
        """Dense block A[:, j0:j1] (rebuild path only)."""
        d2 = ((self.P[:, None, :] - self.Q[None, j0:j1, :]) ** 2).sum(-1)
        return torch.exp(-d2 / (2.0 * self.h * self.h))

    # -- reference accessor contract (numpy in / numpy out) ----------------
    def apply(self, v):
        v = np.asarray(v)
        if np.iscomplexobj(v):
            re = self.apply_dev(torch.from_numpy(np.ascontiguousarray(v.real)))
            im = self.apply_dev(torch.from_numpy(np.ascontiguousarray(v.imag)))
            return (re.cpu().numpy() + 1j * im.cpu().numpy())
        return self.apply_dev(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))).cpu().numpy()

    def adjoint_apply(self, v):
        v = np.asarray(v)
        if np.iscomplexobj(v):
            re = self.apply_dev(torch.from_numpy(np.ascontiguousarray(v.real)), adjoint=True)
            im = self.apply_dev(torch.from_numpy(np.ascontiguousarray(v.imag)), adjoint=True)
            return (re.cpu().numpy() + 1j * im.cpu().numpy())
        return self.apply_dev(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)),
                              adjoint=True).cpu().numpy()

    def row_norms(self):
        return self.row_norms_dev().cpu().numpy()

    def entry(self, i, j):
        return float(self.line_dev(0, i)[j])

    def row(self, i):
        return self.line_dev(0, i).cpu().numpy()

    def column(self, j):
        return self.line_dev(1, j).cpu().numpy()

    def materialize(self):
        return self.block_cols_dev(0, self.shape[1]).cpu().numpy()


class _DenseDeviceOp:
    """cur_build protocol over a dense device matrix (cuBLAS GEMV/GEMM)."""

    def __init__(self, t):
        self.t = t
        self.shape = tuple(t.shape)
        self.device = t.device
        self.dtype = t.dtype
        self.last_kernel_ms = 0.0

    def apply_dev(self, v, adjoint=False, timed=False):
        v = v.to(device=self.device, dtype=self.dtype)
        return (self.t.conj().T @ v) if adjoint else (self.t @ v)

    def row_norms_dev(self):
        return _device.row_masses(self.t)

    def line_dev(self, axis, index):
        return (self.t[index, :] if axis == 0 else self.t[:, index]).clone()

    def restricted_dev(self, axis, sel, w):
        w = w.to(device=self.device, dtype=self.dtype)
        if sel.numel() == 0:
            return torch.zeros(self.shape[1] if axis == 0 else self.shape[0], dtype=self.dtype,
                               device=self.device)
        if axis == 0:
            return self.t[sel, :].T @ w
        return self.t[:, sel] @ w

    def block_cols_dev(self, j0, j1):
        return self.t[:, j0:j1]


class _GaussDeviceOp:
    def __init__(self, g):
        self.g = g
        self.shape = g.shape
        self.device = g.device
        self.dtype = torch.float64

    @property
    def last_kernel_ms(self):
        return self.g.last_kernel_ms

    def apply_dev(self, v, adjoint=False, timed=False):
        return self.g.apply_dev(v, adjoint, timed)

    def row_norms_dev(self):
        return self.g.row_norms_dev()

    def line_dev(self, axis, index):
        return self.g.line_dev(axis, index)

    def restricted_dev(self, axis, sel, w):
        return self.g.restricted_dev(axis, sel, w)

    def block_cols_dev(self, j0, j1):
        return self.g.block_cols_dev(j0, j1)


def as_device_operator(A):
    """Adapt an accessor to the device protocol, or raise CapabilityError
    (host-callable operators cannot run on the B200 path)."""
    if isinstance(A, GaussianKernelOperator):
        return _GaussDeviceOp(A)
    if isinstance(A, DenseMatrix):
        return _DenseDeviceOp(A.tensor)
    if isinstance(A, torch.Tensor) and A.is_cuda:
        return _DenseDeviceOp(A)
    arr = foreign_dense_array(A)
    if arr is not None:     # the reference's rplu.DenseMatrix: upload its array
        from . import _device
        return _DenseDeviceOp(_device.as_device_matrix(A))
    raise CapabilityError(
        f"{type(A).__name__} is not a device operator: the B200 cur_build needs a "
        "DenseMatrix or GaussianKernelOperator (host callables have no device path)")
