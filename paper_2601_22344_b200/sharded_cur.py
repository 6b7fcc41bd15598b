"""Row-sharded matrix-free CUR-form RPLU (Alg 2) across GPUs — SURVEY §8(e), C5.

The operator's points (or the dense matrix) are replicated; rank s owns the
rows [lo_s, hi_s) of the maintained row norms and of every length-n vector
(c, ĉ, g, v).  Per step, mirroring ``cur_build`` (lowmem_cur.py:212-300):

  row draw     shard CDF over the allgathered per-shard totals picks the owner
               with u1; the owner draws its local row against the absolute
               target (``rplu_sample_target``); the global index travels by a
               sum-allreduce of one fp64 (-0.0 from the other ranks).  c2plu:
               the first shard holding the global maximum.
  r, r̂         recomputed on every rank from the replicated operator (same
               kernels, same inputs -> identical bits), so the column draw
               with u2 and the degenerate checks agree everywhere
  c, ĉ         local rows only (c[I] from the replicated column)
  g = A l      the dominant O(n m) generated GEMV, local rows only
  g[I]         one sum-allreduce of k values (owners write theirs, -0.0
               elsewhere) for v = A[:, J] W^{-1} g[I]
  downdate     local rows; per-shard [total, CDF total, max, argmax, clamps]
               allgathered for the stop rules, the rebuild rule and the next
               draw
  core         extended identically on every rank (replicated k x k)

Collectives per step: two allgathers of 5 fp64, one allreduce of 1 fp64 and
one of k fp64 — O(G + k) bytes against O(n m / G) FP64 work.

``comm`` is any object with ``world``, ``rank``, ``allgather(x)`` (1-D,
rank-ordered concatenation) and ``allreduce_sum(x)`` (in place):
``TorchComm`` runs over torch.distributed (NCCL on GPUs, gloo on CPU); the
tests also drive it with a threaded single-GPU emulation.  ``ops`` holds the
draw / downdate primitives (``CudaCurOps``: the library's kernels).
"""

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _ffi
from .lowmem_cur import (CLAMP_REBUILD_FRACTION, CUR_RULES, CurBuildInfo, CurFactorization,
                         _residual_row_dev, _sel, _Stream)
from .operators import (GaussianKernelOperator, _DenseDeviceOp, _GaussDeviceOp,
                        as_device_operator)

__all__ = ["TorchComm", "CudaCurOps", "sharded_cur_build"]


class TorchComm:
    """The sharded drivers' collectives over torch.distributed."""

    def __init__(self, group=None):
        self.group = group
        on = dist.is_initialized()
        self.world = dist.get_world_size(group) if on else 1
        self.rank = dist.get_rank(group) if on else 0

    def allgather(self, x):
        x = x.reshape(-1).contiguous()
        if not dist.is_initialized():
            return x.clone()
        out = torch.empty(self.world * x.numel(), dtype=x.dtype, device=x.device)
        dist.all_gather_into_tensor(out, x, group=self.group)
        return out

    def allreduce_sum(self, x):
        if dist.is_initialized():
            dist.all_reduce(x, op=dist.ReduceOp.SUM, group=self.group)
        return x


class CudaCurOps:
    """Draw and downdate primitives on the device (the library's kernels)."""

    def __init__(self, device):
        self.dev = device
        self.c = _device.ctx(device)

    def _stream(self):
        return _device.stream_handle(self.dev)

    def cdf_total(self, w):
        tot = ctypes.c_double(0.0)
        w = w.contiguous()
        _ffi.check(self.c._lib.rplu_cdf_total(self.c.handle, w.data_ptr() if w.numel() else None,
                                              w.numel(), ctypes.byref(tot), self._stream()))
        return tot.value

    def sample_target(self, w, target):
        idx = ctypes.c_int64(-1)
        w = w.contiguous()
        _ffi.check(self.c._lib.rplu_sample_target(self.c.handle, w.data_ptr(), w.numel(),
                                                  float(target), ctypes.byref(idx), None,
                                                  self._stream()))
        return int(idx.value)

    def sample(self, w, u):
        from .rng import sample_index
        return sample_index(w, u)

    def downdate(self, nrow, g, v, chat, l2, floor, real):
        if real:
            cl, tot = ctypes.c_int64(0), ctypes.c_double(0.0)
            _ffi.check(self.c._lib.rplu_cur_downdate(
                self.c.handle, nrow.numel(), nrow.data_ptr(), g.contiguous().data_ptr(),
                v.contiguous().data_ptr(), chat.contiguous().data_ptr(), l2, floor,
                ctypes.byref(cl), ctypes.byref(tot), self._stream()))
            return int(cl.value), float(tot.value)
        nrow -= 2.0 * torch.real((g - v) * torch.conj(chat))
        nrow += l2 * chat.abs() ** 2
        clamped = int((nrow < -floor).sum())
        nrow.clamp_(min=0.0)
        return clamped, float(nrow.sum())


def _row_block_op(op, rows):
    """The operator restricted to the rows ``rows`` (slice or index tensor)."""
    if isinstance(op, _GaussDeviceOp):
        g = op.g
        return _GaussDeviceOp(GaussianKernelOperator(g.P[rows].contiguous(), g.Q, g.h,
                                                     device=g.device))
    if isinstance(op, _DenseDeviceOp):
        return type(op)(op.t[rows].contiguous())
    raise TypeError(f"cannot shard operator {type(op).__name__}")


def _local_rebuild(op_loc, op, fact, nrow, chunk=256):
    """Row norms of the local rows from m residual columns
    (lowmem_cur.py:204-209); the core solves use the replicated rows I."""
    n_loc, m = op_loc.shape
    nrow.zero_()
    op_I = _row_block_op(op, _sel(fact.row_indices, op.device))
    CJ = torch.stack([op_loc.line_dev(1, j) for j in fact.col_indices], dim=1)
    for j0 in range(0, m, chunk):
        j1 = min(j0 + chunk, m)
        blk = op_loc.block_cols_dev(j0, j1)
        blk_I = op_I.block_cols_dev(j0, j1)
        X = torch.stack([fact.core_solve(blk_I[:, c]) for c in range(j1 - j0)], dim=1)
        res = blk - CJ @ X
        nrow += (res.real ** 2 + (res.imag ** 2 if torch.is_complex(res) else 0)).sum(1)


def sharded_cur_build(A, rows, rule, rank, stop_tol=0.0, rng=None, core_mode="qr", *,
                      comm=None, ops=None):
    """CUR-form RPLU on a row shard (lowmem_cur.py:212-300): call on every rank
    with the full (replicated) operator ``A``, this rank's row range
    ``rows = (lo, hi)`` and an RngState with the same seed.

    Returns ``(CurFactorization, CurBuildInfo)`` — the index sets and the core
    are global and identical on every rank; ``info.row_norms`` holds the
    local rows' maintained norms.
    """
    if rule not in CUR_RULES:
        raise ValueError(f"unknown CUR rule {rule!r}")
    if rule == "rplu-cur" and rng is None:
        raise ValueError("rplu-cur needs an RngState")
    comm = comm if comm is not None else TorchComm()
    op = A if isinstance(A, (_DenseDeviceOp, _GaussDeviceOp)) else as_device_operator(A)
    n, m = op.shape
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    lo, hi = int(rows[0]), int(rows[1])
    if not 0 <= lo <= hi <= n:
        raise ValueError(f"row range {rows} outside [0, {n}]")
    dev = op.device
    ops = ops if ops is not None else CudaCurOps(dev)
    op_loc = _row_block_op(op, slice(lo, hi))
    real = not torch.is_complex(torch.empty(0, dtype=op.dtype))
    info = CurBuildInfo()
    fact = CurFactorization(mode=core_mode, device=dev, dtype=op.dtype)
    eps = np.finfo(float).eps
    world = comm.world

    nrow = (op_loc.row_norms_dev().to(torch.float64).clone() if hi > lo
            else torch.zeros(0, dtype=torch.float64, device=dev))

    def gather_stats(total_loc, clamped_loc=0):
        mx, am = 0.0, -1.0
        if nrow.numel():
            k = int(torch.argmax(nrow))
            mx, am = float(nrow[k]), float(lo + k)
        x = torch.tensor([total_loc, ops.cdf_total(nrow), mx, am, float(clamped_loc)],
                         dtype=torch.float64, device=dev)
        return comm.allgather(x).reshape(world, 5).cpu().numpy()

    st = gather_stats(float(nrow.sum()))
    total0 = 0.0
    for s in range(world):
        total0 += st[s, 0]
    info.total_sq_norms.append(total0)
    if total0 == 0.0:
        info.degenerate_stop = True
        info.row_norms = nrow.cpu().numpy()
        return fact, info
    stream = _Stream(rng if rule == "rplu-cur" else None, 3 * max(rank, 1))
    cur_total = total0

    def draw_row():
        if rule == "rplu-cur":
            u = stream.next()
            T = 0.0
            for s in range(world):
                T += st[s, 1]
            tg = u * T
            c, owner, target, last_pos = 0.0, -1, 0.0, -1
            for s in range(world):
                if st[s, 1] > 0.0:
                    last_pos = s
                if owner < 0 and c + st[s, 1] > tg and st[s, 1] > 0.0:
                    owner, target = s, tg - c
                c += st[s, 1]
            if owner < 0:
                owner, target = last_pos, st[last_pos, 1]
            msg = torch.full((1,), -0.0, dtype=torch.float64, device=dev)
            if owner == comm.rank:
                msg[0] = float(lo + ops.sample_target(nrow, target))
            i = int(comm.allreduce_sum(msg)[0])
        else:
            gmax = float(st[:, 2].max())
            owner = int(np.flatnonzero(st[:, 2] == gmax)[0])
            i = int(st[owner, 3])
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
                j = ops.sample(w, stream.next())
            else:
                j = int(torch.argmax(rhat.abs()))
            a = rhat[j].item()
            I = _sel(fact.row_indices, dev)
            J = _sel(fact.col_indices, dev)
            c_I = op.line_dev(1, j)[I] if fact.rank else None
            if hi > lo:
                c_loc = op_loc.line_dev(1, j)
                yc = fact.core_solve(c_I) if fact.rank else torch.zeros(0, dtype=op.dtype,
                                                                        device=dev)
                chat = c_loc - op_loc.restricted_dev(1, J, yc)
            if real:   # numpy complex division by a real value is x * (1/a)
                l = rhat * (1.0 / a)
            else:
                l = torch.conj(rhat) / np.conj(a)
            g = op_loc.apply_dev(l) if hi > lo else None
            k = fact.rank
            # g[I]: owners contribute their rows, everyone else -0.0 (x + -0 == x)
            gI = torch.full((k,), -0.0, dtype=torch.float64, device=dev)
            if not real:
                gI = torch.complex(gI, gI.clone())
            if k and hi > lo:
                own = (I >= lo) & (I < hi)
                if bool(own.any()):
                    gI[own] = g[I[own] - lo].to(gI.dtype)
            if k:
                comm.allreduce_sum(gI)
            prev = info.total_sq_norms[-1]
            l2 = float((l.abs() ** 2).sum())
            floor = eps * prev / n
            clamped_loc, total_loc = 0, 0.0
            if hi > lo:
                yv = fact.core_solve(gI) if k else torch.zeros(0, dtype=op.dtype, device=dev)
                v = op_loc.restricted_dev(1, J, yv)
                clamped_loc, total_loc = ops.downdate(nrow, g, v, chat, l2, floor, real)
            fact = fact.extended(i, j, c_I, r[J] if k else None, r[j].item())
            st = gather_stats(total_loc, clamped_loc)
            clamped = int(st[:, 4].sum())
            info.clamped.append(clamped)
            if clamped > CLAMP_REBUILD_FRACTION * n:
                if hi > lo:
                    _local_rebuild(op_loc, op, fact, nrow)
                info.rebuilds += 1
                st = gather_stats(float(nrow.sum()))
            cur_total = 0.0
            for s in range(world):
                cur_total += st[s, 0]
            info.total_sq_norms.append(cur_total)
            if stop_tol > 0 and cur_total <= stop_tol ** 2 * total0:
                info.tol_stop = True
                break
    finally:
        stream.commit()
    info.row_norms = nrow.cpu().numpy()
    info.uniforms_consumed = stream.used
    return fact, info
