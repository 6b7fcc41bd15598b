"""Seeded uniform stream and inverse-CDF sampling (mirror of ``rplu.rng``).

``RngState`` keeps the reference's stream exactly (pkg/src/rplu/rng.py:16-47):
numpy ``Philox(key=seed)`` — Random123 philox4x64-10 — and ``uniform()`` =
(raw64 >> 11) * 2**-53.  The stream is host plumbing: the pivot loops pre-draw
a bounded block of uniforms, run on the device, then rewind the generator and
re-draw exactly the number the device consumed (``consume_block`` /
``commit``), so the caller's state ends where the reference would leave it.
A reference ``rplu.rng.RngState`` is accepted interchangeably.

``sample_index`` runs the device K2 CDF kernel (rng.py:50-74 semantics).
"""

import ctypes

import numpy as np

__all__ = ["RngState", "sample_index", "UniformBlock"]


class RngState:
    """A stream of uniforms owned by a single algorithm run (rng.py:16-47)."""

    algorithm = "philox4x64"

    def __init__(self, seed):
        self.seed = int(seed)
        self._gen = np.random.Generator(np.random.Philox(key=self.seed))

    def uniform(self):
        return float(self._gen.random())

    def uniforms(self, k):
        return self._gen.random(k)

    def standard_normal(self, shape):
        return self._gen.standard_normal(shape)

    def complex_normal(self, shape):
        re = self._gen.standard_normal(shape)
        im = self._gen.standard_normal(shape)
        return (re + 1j * im) / np.sqrt(2.0)

    def permutation(self, n):
        return self._gen.permutation(n)

    def __repr__(self):
        return f"RngState(seed={self.seed}, algorithm={self.algorithm!r})"


class UniformBlock:
    """Pre-draw ``k`` uniforms from an RngState and later commit only the used ones.

    Works with this package's RngState and with the reference's (both expose
    a numpy ``Generator`` as ``_gen``).
    """

    def __init__(self, rng, k):
        gen = getattr(rng, "_gen", None)
        if gen is None or not hasattr(gen, "bit_generator"):
            raise TypeError("rng must be an RngState (numpy Generator-backed)")
        self._gen = gen
        self._saved = gen.bit_generator.state
        self.values = np.ascontiguousarray(gen.random(int(k)), dtype=np.float64)

    def pointer(self):
        return self.values.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

    def commit(self, consumed):
        """Rewind and advance the caller's generator by exactly ``consumed`` draws."""
        self._gen.bit_generator.state = self._saved
        if consumed:
            self._gen.random(int(consumed))


def sample_index(weights, u, *, return_near=False):
    """Index with probability proportional to nonnegative weights (rng.py:50-74).

    Runs the same device CDF code the pivot loops use.  Raises ValueError on
    empty, negative or all-zero weights, as the reference does.  With
    ``return_near`` also reports whether the draw fell within 1e-12 relative
    of a CDF boundary.
    """
    import torch

    from . import _device, _ffi
    w = weights
    if isinstance(w, torch.Tensor):
        if w.dim() != 1 or w.numel() == 0:
            raise ValueError("weights must be a nonempty 1-D array")
        dev = w.device if w.is_cuda else _device.require_cuda()
        w = w.to(device=dev, dtype=torch.float64).contiguous()
    else:
        a = np.asarray(weights, dtype=float)
        if a.ndim != 1 or a.size == 0:
            raise ValueError("weights must be a nonempty 1-D array")
        dev = _device.require_cuda()
        w = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    c = _device.ctx(w.device)
    idx = ctypes.c_int64(-1)
    near = ctypes.c_int32(0)
    _ffi.check(c._lib.rplu_sample_index(c.handle, ctypes.c_void_p(w.data_ptr()), w.numel(),
                                        float(u), ctypes.byref(idx), ctypes.byref(near),
                                        _device.stream_handle(w.device)))
    if return_near:
        return int(idx.value), bool(near.value)
    return int(idx.value)
