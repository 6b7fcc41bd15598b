"""ctypes binding of ``librplu_b200.so`` (the C ABI in ``include/rplu_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing or a CUDA device is not
present, the public entry points raise instead of computing on the CPU.

Status codes map onto the reference's exception classes
(SURVEY §8(b)): ARG -> ValueError, ZERO_PIVOT -> ZeroDivisionError,
CAPABILITY -> CapabilityError, CUDA -> RuntimeError.
"""

import ctypes
import os
import threading

from .accessors import CapabilityError

LIB_NAME = "librplu_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

RPLU_OK = 0
RPLU_ERR_ARG = -1
RPLU_ERR_ZERO_PIVOT = -2
RPLU_ERR_CAPABILITY = -3
RPLU_ERR_CUDA = -4

RPLU_F32 = 1
RPLU_F64 = 2
RPLU_C128 = 3

RULE_IDS = {"rplu": 0, "c2plu": 1, "cplu": 2}

FLAG_TIME_KERNELS = 1
FLAG_NO_GRAPH = 2
FLAG_LAZY = 4
FLAG_EAGER = 8
FLAG_STEPWISE = 16
FLAG_EXACT = 32
FLAG_NO_GRAM = 64

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class DenseArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", c_i32), ("rule", c_i32),
        ("n", c_i64), ("m", c_i64), ("ld", c_i64), ("steps", c_i64),
        ("stop_tol", c_dbl),
        ("R", c_vp), ("Lt", c_vp), ("U", c_vp), ("ldu", c_i64),
        ("uniforms", ctypes.POINTER(c_dbl)), ("n_uniforms", c_i64),
        ("stream", c_vp), ("flags", c_i32), ("reserved", c_i32),
    ]


class DenseOut(ctypes.Structure):
    _fields_ = [
        ("pivots", ctypes.POINTER(c_i64)), ("resid_fro", ctypes.POINTER(c_dbl)),
        ("steps_done", c_i64), ("uniforms_consumed", c_i64),
        ("near_boundary_draws", c_i64),
        ("clean_early_stop", c_i32), ("tol_stop", c_i32),
        ("zero_pivot_i", c_i64), ("zero_pivot_j", c_i64),
        ("sweep_ms", c_dbl), ("select_ms", c_dbl), ("sweep_launches", c_i64),
        ("kernel_launches", c_i64), ("sweep_bytes", c_dbl), ("lazy_block", c_i64),
    ]


MF_GAUSS3D = 1
MF_DENSE = 2


class MfArgs(ctypes.Structure):
    _fields_ = [
        ("op_kind", c_i32), ("rule", c_i32), ("n", c_i64), ("m", c_i64), ("rank", c_i64),
        ("stop_tol", c_dbl), ("P", c_vp), ("Q", c_vp), ("h", c_dbl), ("A", c_vp),
        ("lda", c_i64), ("uniforms", ctypes.POINTER(c_dbl)), ("n_uniforms", c_i64),
        ("stream", c_vp), ("flags", c_i32), ("reserved", c_i32),
    ]


class MfOut(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.POINTER(c_i64)), ("cols", ctypes.POINTER(c_i64)),
        ("total_sq_norms", ctypes.POINTER(c_dbl)), ("clamped", ctypes.POINTER(c_i64)),
        ("core", ctypes.POINTER(c_dbl)), ("row_norms", ctypes.POINTER(c_dbl)),
        ("row_norms_dev", c_vp),
        ("steps_done", c_i64), ("uniforms_consumed", c_i64), ("near_boundary_draws", c_i64),
        ("rebuilds", c_i64), ("degenerate_stop", c_i32), ("tol_stop", c_i32),
        ("core_fell_back", c_i32), ("reserved", c_i32), ("gemv_ms", c_dbl),
        ("kernel_launches", c_i64),
    ]


class GroupShard(ctypes.Structure):
    _fields_ = [("R", c_vp), ("Lt", c_vp), ("U", c_vp), ("n_local", c_i64), ("ld", c_i64),
                ("row_offset", c_i64)]


class GroupDenseArgs(ctypes.Structure):
    _fields_ = [("dtype", c_i32), ("lazy_block", c_i32), ("m", c_i64), ("steps", c_i64),
                ("ldu", c_i64), ("stop_tol", c_dbl), ("uniforms", ctypes.POINTER(c_dbl)),
                ("n_uniforms", c_i64), ("shards", ctypes.POINTER(GroupShard))]


class CauchyArgs(ctypes.Structure):
    _fields_ = [
        ("rule", c_i32), ("p", c_i32), ("n", c_i64), ("m", c_i64), ("rank", c_i64),
        ("stop_tol", c_dbl),
        ("x", c_vp), ("y", c_vp), ("G", c_vp), ("Bt", c_vp),
        ("C", c_vp), ("Rrow", c_vp), ("a", c_vp),
        ("uniforms", ctypes.POINTER(c_dbl)), ("n_uniforms", c_i64),
        ("stream", c_vp), ("flags", c_i32), ("reserved", c_i32),
    ]


class CauchyOut(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.POINTER(c_i64)), ("cols", ctypes.POINTER(c_i64)),
        ("bound_maxes", ctypes.POINTER(c_dbl)), ("bound_sums", ctypes.POINTER(c_dbl)),
        ("steps_done", c_i64), ("bounds_recorded", c_i64), ("uniforms_consumed", c_i64),
        ("near_boundary_draws", c_i64), ("tol_stop", c_i32), ("degenerate_stop", c_i32),
        ("zero_pivot_i", c_i64), ("zero_pivot_j", c_i64),
        ("masses_ms", c_dbl), ("masses_launches", c_i64), ("kernel_launches", c_i64),
    ]


class ShardArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", c_i32), ("world", c_i32), ("rank", c_i32), ("lazy_block", c_i32),
        ("n_local", c_i64), ("m", c_i64), ("ld", c_i64), ("row_offset", c_i64),
        ("steps", c_i64), ("stop_tol", c_dbl),
        ("R", c_vp), ("Lt", c_vp), ("U", c_vp), ("ldu", c_i64),
        ("uniforms", ctypes.POINTER(c_dbl)), ("n_uniforms", c_i64),
        ("stream", c_vp),
    ]


class CauchyShardArgs(ctypes.Structure):
    _fields_ = [
        ("rule", c_i32), ("p", c_i32), ("world", c_i32), ("rank", c_i32),
        ("n_local", c_i64), ("m", c_i64), ("row_offset", c_i64), ("steps", c_i64),
        ("stop_tol", c_dbl),
        ("x", c_vp), ("y", c_vp), ("G", c_vp), ("Bt", c_vp),
        ("C", c_vp), ("Rrow", c_vp), ("a", c_vp),
        ("uniforms", ctypes.POINTER(c_dbl)), ("n_uniforms", c_i64),
        ("stream", c_vp),
    ]


CAUCHY_MSG_DOUBLES = 20   # RPLU_CAUCHY_MSG_DOUBLES


class TreePlan(ctypes.Structure):
    _fields_ = [
        ("n", c_i64), ("m", c_i64), ("p", c_i32), ("n_levels", c_i32), ("n_tleaves", c_i64),
        ("tperm", c_vp), ("tstart", c_vp), ("agg_start", c_vp), ("agg_node", c_vp),
        ("agg_alpha", c_vp), ("ex_start", c_vp), ("ex_leaf", c_vp),
        ("n_snodes", c_i64), ("n_sleaves", c_i64), ("spts", c_vp), ("sstart", c_vp),
        ("cstart", c_vp), ("cidx", c_vp), ("leaf_node", c_vp), ("lvl_nodes", c_vp),
        ("lvl_start", c_vp),
    ]


# name -> (restype, argtypes); every symbol declared in include/rplu_b200.h
SIGNATURES = {
    "rplu_abi_version": (ctypes.c_int, []),
    "rplu_last_error": (ctypes.c_char_p, []),
    "rplu_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    "rplu_ctx_destroy": (ctypes.c_int, [c_vp]),
    "rplu_dense_run": (ctypes.c_int, [c_vp, ctypes.POINTER(DenseArgs), ctypes.POINTER(DenseOut)]),
    "rplu_row_masses": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "rplu_sample_index": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, ctypes.POINTER(c_i64),
                                         ctypes.POINTER(c_i32), c_vp]),
    "rplu_sample_target": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, ctypes.POINTER(c_i64),
                                          ctypes.POINTER(c_i32), c_vp]),
    "rplu_cdf_total": (ctypes.c_int, [c_vp, c_vp, c_i64, ctypes.POINTER(c_dbl), c_vp]),
    "rplu_cauchy_run": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyArgs),
                                       ctypes.POINTER(CauchyOut)]),
    "rplu_cauchy_row_norms": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                             c_vp, c_vp]),
    "rplu_diag_fp64_peak": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl)]),
    "rplu_diag_dmma_peak": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl)]),
    "rplu_tree_bounds": (ctypes.c_int, [c_vp, ctypes.POINTER(TreePlan), c_vp, c_vp, c_vp, c_vp,
                                        c_vp, c_vp]),
    # Gaussian-kernel operator struct is passed by pointer (operators._GaussOpStruct)
    "rplu_gauss_apply": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(c_dbl),
                                        c_vp]),
    "rplu_gauss_row_norms": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "rplu_gauss_line": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "rplu_gauss_restricted": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "rplu_cur_downdate": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_dbl, c_dbl,
                                         ctypes.POINTER(c_i64), ctypes.POINTER(c_dbl), c_vp]),
    "rplu_kernel_launch_count": (c_i64, []),
    "rplu_mf_run": (ctypes.c_int, [c_vp, ctypes.POINTER(MfArgs), ctypes.POINTER(MfOut)]),
    "rplu_upload": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp]),
    "rplu_group_create": (ctypes.c_int, [c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_vp)]),
    "rplu_group_destroy": (ctypes.c_int, [c_vp]),
    "rplu_group_dense_run": (ctypes.c_int, [c_vp, ctypes.POINTER(GroupDenseArgs),
                                            ctypes.POINTER(DenseOut)]),
    "rplu_lu_error": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp,
                                     c_i64, c_i64, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl),
                                     c_vp]),
    "rplu_cauchy_plan_row": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64,
                                            c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rplu_cauchy_plan_update": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                               c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "rplu_cauchy_plan_propose": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                                c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp]),
    "rplu_sample_index_gather": (ctypes.c_int, [c_vp, c_vp, c_i64, c_dbl, c_vp,
                                                ctypes.POINTER(c_i64), ctypes.POINTER(c_i32),
                                                c_vp, c_vp]),
    "rplu_plan_build": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_dbl, c_i64, c_vp,
                                       ctypes.POINTER(c_vp)]),
    "rplu_plan_counts": (ctypes.c_int, [c_vp, c_vp]),
    "rplu_plan_tree": (ctypes.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp]),
    "rplu_plan_lists": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rplu_plan_free": (ctypes.c_int, [c_vp]),
    "rplu_loewner_fill": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "rplu_bary_eval": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_dbl, c_i32,
                                      c_vp, c_vp, c_vp]),
    "rplu_mgs_arnoldi": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "rplu_shard_begin": (ctypes.c_int, [c_vp, ctypes.POINTER(ShardArgs), c_vp]),
    "rplu_shard_select": (ctypes.c_int, [c_vp, ctypes.POINTER(ShardArgs), c_i64, c_vp, c_vp]),
    "rplu_shard_update": (ctypes.c_int, [c_vp, ctypes.POINTER(ShardArgs), c_i64, c_vp, c_vp]),
    "rplu_shard_active": (ctypes.c_int, [c_vp, ctypes.POINTER(ShardArgs), ctypes.POINTER(c_i32)]),
    "rplu_shard_lazy_block": (ctypes.c_int, [ctypes.POINTER(ShardArgs)]),
    "rplu_shard_finish": (ctypes.c_int, [c_vp, ctypes.POINTER(ShardArgs),
                                         ctypes.POINTER(DenseOut)]),
    "rplu_cauchy_shard_begin": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyShardArgs), c_vp]),
    "rplu_cauchy_shard_select": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyShardArgs), c_i64,
                                                c_vp, c_vp]),
    "rplu_cauchy_shard_update": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyShardArgs), c_i64,
                                                c_vp, c_vp]),
    "rplu_cauchy_shard_active": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyShardArgs),
                                                ctypes.POINTER(c_i32)]),
    "rplu_cauchy_shard_finish": (ctypes.c_int, [c_vp, ctypes.POINTER(CauchyShardArgs),
                                                ctypes.POINTER(CauchyOut)]),
}


def kernel_launch_count():
    """Process-wide count of kernels launched by the standalone primitives."""
    return int(load_library().rplu_kernel_launch_count())


def fp64_peak_tflops(device=0):
    """Measured FP64 FMA throughput of `device` (TFLOP/s) via the library probe."""
    c = context(device)
    tf, ms = c_dbl(0.0), c_dbl(0.0)
    check(c._lib.rplu_diag_fp64_peak(c.handle, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value


def dmma_peak_tflops(device=0):
    """Measured FP64 tensor-core (DMMA) throughput of `device` (TFLOP/s)."""
    c = context(device)
    tf, ms = c_dbl(0.0), c_dbl(0.0)
    check(c._lib.rplu_diag_dmma_peak(c.handle, ctypes.byref(tf), ctypes.byref(ms)))
    return tf.value


_lib = None
_lib_lock = threading.Lock()


class ExtensionMissingError(RuntimeError):
    """The CUDA extension has not been built (there is no CPU fallback)."""


def load_library(path=LIB_PATH):
    """Load and type the shared library (no GPU needed to load it)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ExtensionMissingError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). The B200 path has no CPU fallback.")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(status):
    """Raise the reference's exception class for a non-zero status."""
    if status == RPLU_OK:
        return
    msg = load_library().rplu_last_error().decode(errors="replace")
    if status == RPLU_ERR_ARG:
        raise ValueError(msg)
    if status == RPLU_ERR_ZERO_PIVOT:
        raise ZeroDivisionError(msg)
    if status == RPLU_ERR_CAPABILITY:
        raise CapabilityError(msg)
    raise RuntimeError(msg)


class Context:
    """One ``rplu_ctx`` (workspace + device binding) per (thread, device)."""

    def __init__(self, device):
        lib = load_library()
        h = c_vp()
        check(lib.rplu_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self._lib = lib

    def __del__(self):
        try:
            if self.handle:
                self._lib.rplu_ctx_destroy(self.handle)
        except Exception:
            pass


_tls = threading.local()


def context(device):
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(int(device))
    if c is None:
        c = ctxs[int(device)] = Context(device)
    return c
