"""Device buffers and streams (PyTorch as plumbing only).

Torch is used for HBM allocation, host<->device copies and the current CUDA
stream; all pivot-loop arithmetic runs in ``librplu_b200.so``.
"""

import ctypes

import numpy as np
import torch

from . import _ffi

DTYPE_IDS = {torch.float32: _ffi.RPLU_F32, torch.float64: _ffi.RPLU_F64,
             torch.complex128: _ffi.RPLU_C128}


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 RPLU path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device() if device is None else
                        torch.device(device).index or 0)


def stream_handle(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ctx(device):
    return _ffi.context(device.index if device.index is not None else 0)


def _resolve_dtype(src_dtype_is_complex, dtype):
    if dtype is not None:
        if isinstance(dtype, str):
            dtype = {"f32": torch.float32, "float32": torch.float32, "f64": torch.float64,
                     "float64": torch.float64, "c128": torch.complex128,
                     "complex128": torch.complex128}[dtype]
        if dtype not in DTYPE_IDS:
            raise ValueError(f"unsupported compute dtype {dtype}")
        return dtype
    return torch.complex128 if src_dtype_is_complex else torch.float64


def vec_of(dtype):
    """Elements per 16-byte vector for the row-stride padding."""
    return {torch.float32: 4, torch.float64: 2, torch.complex128: 1}[dtype]


def as_device_matrix(A, dtype=None, device=None, copy=True):
    """Return a contiguous (n, m) CUDA tensor holding A in the compute dtype.

    numpy input follows the reference promotion (real -> float64, complex ->
    complex128) unless ``dtype`` is given; torch input keeps its dtype when it
    is one of fp32 / fp64 / complex128.
    """
    dev = require_cuda(device)
    if hasattr(A, "tensor") and isinstance(getattr(A, "tensor"), torch.Tensor):
        A = A.tensor
    else:
        from .accessors import foreign_dense_array
        arr = foreign_dense_array(A)
        if arr is not None:
            # the reference's DenseMatrix stores complex128 always
            # (accessors.py:100); a real-valued one computes in float64,
            # arithmetically identical
            A = real_if_zero_imag(arr) if dtype is None else arr
    if isinstance(A, torch.Tensor):
        if A.dim() != 2:
            raise ValueError("expected a 2-D array")
        want = dtype if dtype is not None else (A.dtype if A.dtype in DTYPE_IDS else None)
        want = _resolve_dtype(A.is_complex(), want)
        t = A.to(device=dev, dtype=want, non_blocking=A.is_pinned())
        if copy and t.data_ptr() == A.data_ptr():
            t = t.clone()
        return t.contiguous()
    a = np.asarray(A)
    if a.ndim != 2:
        raise ValueError("expected a 2-D array")
    want = _resolve_dtype(np.iscomplexobj(a), dtype)
    np_want = {torch.float32: np.float32, torch.float64: np.float64,
               torch.complex128: np.complex128}[want]
    a = np.ascontiguousarray(a, dtype=np_want)
    return upload(a, dev)


_UPLOAD_MIN_BYTES = 16 << 20


def upload(a, dev):
    """Contiguous numpy array -> new CUDA tensor.  Large pageable arrays go
    through the library's pinned staging ring (rplu_upload: multi-threaded
    host copies overlapped with the DMA); a torch pinned tensor's numpy
    view and small arrays use a plain copy."""
    t = torch.from_numpy(a)
    if a.nbytes < _UPLOAD_MIN_BYTES or t.is_pinned():
        return t.to(dev, non_blocking=t.is_pinned())
    out = torch.empty(a.shape, dtype=t.dtype, device=dev)
    c = ctx(dev)
    import os
    # 8 staging threads measured best on the 16-vCPU B200 hosts (52 GB/s against
    # 54 GB/s for a pinned source; 4: 36, 12: 48, 16: 46 -- scripts/time_upload.py)
    threads = max(1, min(int(os.environ.get("RPLU_UPLOAD_THREADS", "8")),
                         len(os.sched_getaffinity(0))))
    _ffi.check(c._lib.rplu_upload(c.handle, ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(a.ctypes.data), a.nbytes, threads,
                                  stream_handle(dev)))
    return out


def real_if_zero_imag(a):
    """float64 view of a complex array whose imaginary parts are all zero."""
    if np.iscomplexobj(a) and not np.any(a.imag):
        return np.ascontiguousarray(a.real)
    return a


def padded_residual(t):
    """Copy a (n, m) device matrix into an (n, ld) buffer with 16-byte rows.

    Returns (buffer, view) where view = buffer[:, :m] is the residual.
    """
    n, m = t.shape
    v = vec_of(t.dtype)
    ld = ((m + v - 1) // v) * v
    if ld == m:
        buf = t.clone() if t.is_contiguous() else t.contiguous().clone()
        return buf, buf
    buf = torch.empty((n, ld), dtype=t.dtype, device=t.device)
    buf[:, :m].copy_(t)
    buf[:, m:].zero_()
    return buf, buf[:, :m]


def row_masses(t):
    """K1 on a device matrix: squared row norms as a float64 CUDA tensor."""
    n, m = t.shape
    if t.dtype not in DTYPE_IDS:
        t = t.to(torch.complex128 if t.is_complex() else torch.float64)
    if t.stride(1) != 1:
        t = t.contiguous()
    out = torch.empty(n, dtype=torch.float64, device=t.device)
    c = ctx(t.device)
    _ffi.check(c._lib.rplu_row_masses(c.handle, DTYPE_IDS[t.dtype], ctypes.c_void_p(t.data_ptr()),
                                      n, m, t.stride(0), ctypes.c_void_p(out.data_ptr()),
                                      stream_handle(t.device)))
    return out


def matvec(t, v, adjoint=False):
    """A @ v or A^H @ v on the device (cuBLAS GEMV); returns numpy."""
    vt = torch.as_tensor(np.asarray(v), device=t.device)
    if t.is_complex() or vt.is_complex():
        tt = t.to(torch.complex128)
        vt = vt.to(torch.complex128)
    else:
        tt = t.to(torch.float64)
        vt = vt.to(torch.float64)
    r = (tt.conj().T @ vt) if adjoint else (tt @ vt)
    return r.cpu().numpy()


_PINNED_MIN_BYTES = 1 << 20


def to_numpy(t):
    """Device tensor -> numpy through page-locked host memory.

    A device->pageable copy into freshly allocated numpy memory runs at
    ~2 GB/s on the B200 boxes (measured: 121 ms for L and U at C3); a copy
    into a block of torch's caching pinned-host allocator runs at PCIe speed
    and the numpy result is a view of that block (kept alive by the array).
    """
    if not t.is_cuda or t.numel() * t.element_size() < _PINNED_MIN_BYTES:
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


class PinnedPrefetch:
    """Page-locked host buffers allocated on a helper thread while the device
    loop runs (the ctypes call releases the GIL), so the results' copy-back
    does not pay cudaHostAlloc on the critical path (268 MB of L and U at
    C3 cost ~40-80 ms to pin).  ``get(i)`` joins and returns buffer i, or
    None if the allocation failed (the caller then copies the usual way)."""

    def __init__(self, specs):
        import threading
        self._bufs = [None] * len(specs)

        def work():
            for i, (shape, dtype) in enumerate(specs):
                try:
                    self._bufs[i] = torch.empty(shape, dtype=dtype, pin_memory=True)
                except Exception:  # pinned memory exhausted: plain copy-back
                    self._bufs[i] = None
        self._thread = threading.Thread(target=work, daemon=True)
        self._thread.start()

    def get(self, i):
        self._thread.join()
        return self._bufs[i]


def copy_to_host(t, buf):
    """numpy copy of device tensor t, into the pinned buffer's leading slice
    when one is given (else through to_numpy)."""
    if buf is None:
        return to_numpy(t)
    h = buf.view(-1)[:t.numel()].view(t.shape)
    h.copy_(t)
    return h.numpy()

