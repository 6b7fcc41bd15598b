"""Row-block sharded dense RPLU across GPUs (one process per GPU, NCCL).

SURVEY §8(e): rank s owns the contiguous rows [s*n/G, (s+1)*n/G) of the
residual (cyclic sharding would break the CDF order).  Per pivot step:

  select   every rank sums the allgathered shard totals in rank order, picks
           the owning shard with u1 and (owner only) draws the local row and
           the column; the owner writes the pivot header [i, j, a] and the
           pivot row into U[t,:], every other rank writes -0.0
  allreduce(sum) of the header (4 fp64) and U[t,:] (m elements): x + (-0) == x
           bit for bit, so the sum IS a broadcast from the owner without a
           host round trip to learn who the owner is
  update   post the pivot, fused Schur update + masses of the local rows (the
           single-GPU K3 kernel), local total
  allgather of the local totals (one fp64 per rank) for the next step

Work per rank per step is n*m/G*2*s bytes of HBM traffic against two small
collectives, so the path scales with G until the per-step collective latency
(~tens of microseconds) dominates.  L stays row-sharded; U and the pivots are
replicated on every rank.

``run_sharded`` is the collective choreography; it drives any backend with
``begin / select / update / active / finish`` (the CUDA backend here; the
CPU tests drive it with a numpy backend over gloo).
"""

import ctypes
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _ffi
from .accessors import CapabilityError
from .dense_pivots import EliminationTrace, PivotRule
from .rng import UniformBlock

__all__ = ["shard_rows", "run_sharded", "run_sharded_graph", "sharded_eliminate", "group_eliminate",
           "CudaShardBackend", "run_sharded_cauchy", "CudaCauchyShardBackend",
           "sharded_structured_eliminate"]


def shard_rows(n, world, rank):
    """Contiguous row block [lo, hi) of shard `rank` (balanced, in rank order)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _all_gather_scalar(x, group, world, out=None):
    if not dist.is_initialized():
        if out is not None:      # static buffer (graph replay)
            out.copy_(x.reshape(1))
            return out
        return x.reshape(1)
    out = torch.empty(world, dtype=x.dtype, device=x.device) if out is None else out
    dist.all_gather_into_tensor(out, x.reshape(1), group=group)
    return out


def run_sharded(backend, steps, group=None, poll_every=32, step_hook=None):
    """Collective choreography of one sharded elimination (see module doc):
    per step one sum-allreduce of the pivot message and one allgather of the
    shard totals."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    local_total = backend.begin()
    totals = _all_gather_scalar(local_total, group, world)
    for t in range(steps + 1):
        msg = backend.select(t, totals)
        if t == steps:
            break
        if dist.is_initialized():   # (also at world 1: exercises the NCCL path)
            dist.all_reduce(msg, op=dist.ReduceOp.SUM, group=group)
        if step_hook is not None:
            step_hook("pre_update", t)
        local_total = backend.update(t, msg)
        if step_hook is not None:
            step_hook("post_update", t)
        totals = _all_gather_scalar(local_total, group, world)
        # the stop decision is global (same totals on every rank), so every
        # rank breaks at the same step
        if poll_every and (t + 1) % poll_every == 0 and not backend.active():
            break
    return backend.finish()


class _capture:
    """CUDA-graph capture of the enclosed launches on a side stream.

    torch.cuda.graph() would do: it also runs gc.collect() and
    torch.cuda.empty_cache() on entry, which hands every cached block back to
    the driver -- at C3 size the next call then pays a fresh 8.6 GB cudaMalloc
    for its residual copy (0.1-0.3 s, more than a tenth of the run).  The
    shard kernels launch on torch's current stream, which this switches."""

    def __init__(self, graph, dev):
        self.graph, self.dev = graph, dev
        self.stream = torch.cuda.Stream(dev)

    def __enter__(self):
        torch.cuda.synchronize(self.dev)
        self.stream.wait_stream(torch.cuda.current_stream(self.dev))
        self._ctx = torch.cuda.stream(self.stream)
        self._ctx.__enter__()
        self.graph.capture_begin()
        return self

    def __exit__(self, et, ev, tb):
        try:
            if et is None:
                self.graph.capture_end()
            else:       # leave capture mode without keeping the graph
                try:
                    self.graph.capture_end()
                except RuntimeError:
                    pass
        finally:
            self._ctx.__exit__(et, ev, tb)
        torch.cuda.current_stream(self.dev).wait_stream(self.stream)
        return False


def _run_sharded_block_graph(backend, steps, group, block):
    """Delayed-update shards: one whole block of `block` steps (per step the
    select kernels, the allreduce, post + pivot column + read pass -- the
    flush at the block's last position -- and the allgather) is captured once
    and replayed.  Inside a block the number of pending terms of each step is
    fixed at capture; the absolute step comes from the device counter.  The
    first block runs uncaptured (it also warms every kernel variant), a
    trailing partial block runs with explicit steps."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    local_total = backend.begin()
    totals = torch.empty(world, dtype=torch.float64, device=backend.dev)
    totals.copy_(_all_gather_scalar(local_total, group, world))

    def step(t):
        msg = backend.select(t, totals)
        if dist.is_initialized():
            dist.all_reduce(msg, op=dist.ReduceOp.SUM, group=group)
        lt = backend.update(t, msg)
        _all_gather_scalar(lt, group, world, out=totals)

    nblocks = steps // block
    t = 0
    if nblocks >= 1:
        for _ in range(block):
            step(t)
            t += 1
    if nblocks >= 2 and backend.active():
        torch.cuda.synchronize(backend.dev)
        g = torch.cuda.CUDAGraph()
        try:
            with _capture(g, backend.dev):
                for pos in range(block):
                    step(-1 - pos)
        except RuntimeError:
            # capture refused (e.g. a collective backend that cannot be
            # captured): nothing of the block has run, the device step
            # counter is untouched -- carry on with explicit steps
            g = None
            torch.cuda.synchronize(backend.dev)
        for k in range(1, nblocks if g is not None else 0):
            g.replay()
            t += block
            if k % 2 == 0 and k + 1 < nblocks and not backend.active():
                break
    if t < steps and backend.active():
        for tt in range(t, steps):      # trailing partial block (or a one-block run)
            step(tt)
    backend.select(-1, totals)          # final residual norm / stop flags
    return backend.finish()


def run_sharded_graph(backend, steps, group=None, chunk=32):
    """The same choreography with one step (select, allreduce, update,
    allgather) captured once in a CUDA graph and replayed: the kernels read
    the step index from the device counter, the collectives run on static
    buffers.  Replays go in chunks of `chunk` steps with a stop poll between
    chunks.  Delayed-update backends capture one flush block instead
    (`_run_sharded_block_graph`)."""
    block = getattr(backend, "block_len", 0)
    if block > 0:
        return _run_sharded_block_graph(backend, steps, group, block)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    local_total = backend.begin()
    totals = torch.empty(world, dtype=torch.float64, device=backend.dev)
    totals.copy_(_all_gather_scalar(local_total, group, world))
    if steps == 0:
        backend.select(-1, totals)
        return backend.finish()
    # capture on a side stream (torch.cuda.graph); the backend launches on
    # the current stream, which the capture context switches for us
    torch.cuda.synchronize(backend.dev)
    g = torch.cuda.CUDAGraph()
    with _capture(g, backend.dev):
        msg = backend.select(-1, totals)
        if dist.is_initialized():
            dist.all_reduce(msg, op=dist.ReduceOp.SUM, group=group)
        lt = backend.update(-1, msg)
        _all_gather_scalar(lt, group, world, out=totals)
    done = 0
    while done < steps:
        n = min(chunk, steps - done)
        for _ in range(n):
            g.replay()
        done += n
        if done < steps and not backend.active():
            break
    backend.select(-1, totals)          # final residual norm / stop flags
    return backend.finish()


class CudaShardBackend:
    """Product backend: the rplu_shard_* C ABI on this rank's GPU."""

    def __init__(self, R, row_offset, world, rank, rule, steps, stop_tol=0.0, ctx=None,
                 lazy_block=0):
        if rule.tag != "rplu":
            raise CapabilityError("the sharded path implements rule 'rplu'")
        self.dev = R.device
        self.R = R
        n_local, m = R.shape
        vec = _device.vec_of(R.dtype)
        self.ldu = ((m + vec - 1) // vec) * vec
        self.Lt = torch.empty((max(steps, 1), max(n_local, 1)), dtype=R.dtype, device=self.dev)
        self.U = torch.empty((max(steps, 1) + 1, self.ldu), dtype=R.dtype, device=self.dev)
        # pivot message: 4 fp64 header + the pivot row, reduced as one buffer
        # (fp64 view for fp64/complex128 rows, fp32 view for fp32 rows)
        esz = R.element_size()
        nbytes = 32 + m * esz
        red = torch.float32 if R.dtype == torch.float32 else torch.float64
        self.msg = torch.empty(nbytes // torch.empty(0, dtype=red).element_size(), dtype=red,
                               device=self.dev)
        self.total = torch.empty(1, dtype=torch.float64, device=self.dev)
        self.block = UniformBlock(rule.rng, 2 * steps + 2)
        self.steps = steps
        self.m = m
        self.n_local = n_local
        self.args = _ffi.ShardArgs(
            dtype=_device.DTYPE_IDS[R.dtype], world=world, rank=rank, n_local=n_local, m=m,
            ld=R.stride(0), row_offset=row_offset, steps=steps, stop_tol=float(stop_tol),
            R=R.data_ptr() if n_local else None, Lt=self.Lt.data_ptr(), U=self.U.data_ptr(),
            ldu=self.ldu, uniforms=self.block.pointer(), n_uniforms=self.block.values.size,
            stream=None, lazy_block=int(lazy_block))
        c = ctx if ctx is not None else _device.ctx(self.dev)
        self._ctx = c
        self._lib, self._h = c._lib, c.handle
        # resolved flush interval (0: eager updates)
        self.block_len = int(self._lib.rplu_shard_lazy_block(ctypes.byref(self.args)))
        self.pivots = np.zeros(2 * max(steps, 1), dtype=np.int64)
        self.resid = np.zeros(steps + 1)

    def _args(self):
        # launch on whatever stream is current (a graph capture switches it)
        self.args.stream = torch.cuda.current_stream(self.dev).cuda_stream
        return ctypes.byref(self.args)

    def begin(self):
        _ffi.check(self._lib.rplu_shard_begin(self._h, self._args(), self.total.data_ptr()))
        return self.total

    def select(self, t, totals):
        totals = totals.contiguous()
        self._totals = totals   # keep alive until the kernel ran
        _ffi.check(self._lib.rplu_shard_select(self._h, self._args(), t, totals.data_ptr(),
                                               self.msg.data_ptr()))
        return self.msg

    def update(self, t, msg):
        _ffi.check(self._lib.rplu_shard_update(self._h, self._args(), t, msg.data_ptr(),
                                               self.total.data_ptr()))
        return self.total

    def active(self):
        a = ctypes.c_int32(0)
        _ffi.check(self._lib.rplu_shard_active(self._h, self._args(), ctypes.byref(a)))
        return bool(a.value)

    def finish(self):
        out = _ffi.DenseOut(
            pivots=self.pivots.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            resid_fro=self.resid.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        status = self._lib.rplu_shard_finish(self._h, self._args(), ctypes.byref(out))
        self.block.commit(out.uniforms_consumed)
        _ffi.check(status)
        k = int(out.steps_done)
        self.lazy_block_used = int(out.lazy_block)
        return dict(pivots=[(int(self.pivots[2 * t]), int(self.pivots[2 * t + 1]))
                            for t in range(k)],
                    resid_fro=self.resid[:k + 1].copy(), steps=k,
                    clean_early_stop=bool(out.clean_early_stop), tol_stop=bool(out.tol_stop),
                    near_boundary_draws=int(out.near_boundary_draws),
                    uniforms_consumed=int(out.uniforms_consumed),
                    L_local=self.Lt[:k, :self.n_local].T, U=self.U[:k, :self.m])


def sharded_eliminate(A_local, row_offset, rule, steps, stop_tol=0.0, group=None,
                      compute_dtype=None, overwrite_a=False, step_hook=None, graph=False,
                      update="auto", lazy_block=None):
    """RPLU on a row-block shard (call on every rank with the same rule seed).

    ``A_local`` is this rank's contiguous row block (global rows
    [row_offset, row_offset + n_local)); every rank must pass the same
    ``steps``/``stop_tol`` and an RngState with the same seed.  Returns an
    EliminationTrace whose L holds this rank's rows of L (device tensor) and
    whose U / pivots / resid_fro are the global (replicated) values.

    ``update``: "eager" (fused K3 update every step), "lazy" (delayed
    updates: one read of the row block per step, a write every ``lazy_block``
    steps), or "auto" (lazy when the local block exceeds 256 MB, as on one
    GPU).  ``graph=True`` captures one step (eager) or one whole flush block
    (lazy) with its collectives in a CUDA graph and replays it.  Results are
    bit-identical across modes.
    """
    if update not in ("auto", "eager", "lazy"):
        raise ValueError(f"update must be 'auto', 'eager' or 'lazy', not {update!r}")
    if isinstance(rule, str):
        rule = PivotRule(rule)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    src = _device.as_device_matrix(A_local, dtype=compute_dtype, copy=False)
    vec = _device.vec_of(src.dtype)
    if (overwrite_a or src is not A_local) and src.is_contiguous() and src.shape[1] % vec == 0:
        R = src
    else:
        R = _device.padded_residual(src)[1]   # (n_local, m) view, 16-byte rows
    n_local, m = src.shape
    if update == "auto":
        big = n_local * m * R.element_size() > 256e6
        update = "lazy" if big and steps >= 2 else "eager"
    lb = 0 if update == "eager" else (-1 if lazy_block is None else int(lazy_block))
    backend = CudaShardBackend(R, row_offset, world, rank, rule, steps, stop_tol, lazy_block=lb)
    if graph and step_hook is None:
        res = run_sharded_graph(backend, steps, group=group)
    else:
        res = run_sharded(backend, steps, group=group, step_hook=step_hook)
    tr = EliminationTrace(
        pivots=res["pivots"], L=res["L_local"], U=res["U"], resid_fro=res["resid_fro"],
        residual=R[:, :m], steps=res["steps"], clean_early_stop=res["clean_early_stop"],
        tol_stop=res["tol_stop"], near_boundary_draws=res["near_boundary_draws"],
        uniforms_consumed=res["uniforms_consumed"], host=False)
    tr.lazy_block = backend.lazy_block_used   # 0: eager updates
    return tr


def group_eliminate(A, rule, steps, devices=(0,), stop_tol=0.0, compute_dtype=None,
                    update="eager"):
    """Row-block sharded RPLU across ``devices`` from ONE process, driven by
    the library's C loop (``rplu_group_dense_run``: NCCL communicators from
    ncclCommInitAll, grouped allreduce / allgather per step -- no
    torch.distributed, no Python per step).  ``A`` (host or device) is split
    into contiguous row blocks in device order.  Returns an EliminationTrace
    with L gathered on devices[0] and U / pivots / resid_fro replicated.
    ``update``: "eager" (fused update every step) or "lazy" (delayed updates,
    fp64 with Gram-form masses)."""
    if update not in ("eager", "lazy"):
        raise ValueError(f"update must be 'eager' or 'lazy', not {update!r}")
    if isinstance(rule, str):
        rule = PivotRule(rule)
    if rule.tag != "rplu":
        raise CapabilityError("the sharded path implements rule 'rplu'")
    devices = [int(d) for d in devices]
    G = len(devices)
    host = _device.as_device_matrix(A, dtype=compute_dtype, device=devices[0])
    n, m = host.shape
    if not 0 <= steps <= min(n, m):
        raise ValueError(f"steps {steps} out of range [0, {min(n, m)}]")
    vec = _device.vec_of(host.dtype)
    ldu = ((m + vec - 1) // vec) * vec
    lib = _ffi.load_library()
    bufs, shards = [], (_ffi.GroupShard * G)()
    for d, dev in enumerate(devices):
        lo, hi = shard_rows(n, G, d)
        R = torch.zeros((hi - lo, ldu), dtype=host.dtype, device=f"cuda:{dev}")
        R[:, :m].copy_(host[lo:hi])
        Lt = torch.empty((max(steps, 1), max(hi - lo, 1)), dtype=host.dtype, device=R.device)
        U = torch.empty((max(steps, 1) + 1, ldu), dtype=host.dtype, device=R.device)
        bufs.append((R, Lt, U, lo, hi))
        shards[d] = _ffi.GroupShard(R=R.data_ptr(), Lt=Lt.data_ptr(), U=U.data_ptr(),
                                    n_local=hi - lo, ld=ldu, row_offset=lo)
    for dev in devices:
        torch.cuda.synchronize(dev)
    block = UniformBlock(rule.rng, 2 * steps + 2)
    args = _ffi.GroupDenseArgs(dtype=_device.DTYPE_IDS[host.dtype],
                               lazy_block=0 if update == "eager" else -1, m=m, steps=steps,
                               ldu=ldu, stop_tol=float(stop_tol), uniforms=block.pointer(),
                               n_uniforms=block.values.size, shards=shards)
    pivots = np.zeros(2 * max(steps, 1), dtype=np.int64)
    resid = np.zeros(steps + 1)
    out = _ffi.DenseOut(pivots=pivots.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        resid_fro=resid.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    grp = ctypes.c_void_p()
    _ffi.check(lib.rplu_group_create(G, (ctypes.c_int32 * G)(*devices), ctypes.byref(grp)))
    try:
        status = lib.rplu_group_dense_run(grp, ctypes.byref(args), ctypes.byref(out))
        block.commit(out.uniforms_consumed)
        _ffi.check(status)
    finally:
        lib.rplu_group_destroy(grp)
    k = int(out.steps_done)
    L = torch.cat([Lt[:k, :hi - lo].T.to(f"cuda:{devices[0]}") for (_, Lt, _, lo, hi) in bufs],
                  dim=0)
    Rfull = torch.cat([R[:, :m].to(f"cuda:{devices[0]}") for (R, _, _, _, _) in bufs], dim=0)
    tr = EliminationTrace(
        pivots=[(int(pivots[2 * t]), int(pivots[2 * t + 1])) for t in range(k)], L=L,
        U=bufs[0][2][:k, :m], resid_fro=resid[:k + 1].copy(), residual=Rfull, steps=k,
        clean_early_stop=bool(out.clean_early_stop), tol_stop=bool(out.tol_stop),
        near_boundary_draws=int(out.near_boundary_draws),
        uniforms_consumed=int(out.uniforms_consumed), host=False)
    tr.lazy_block = int(out.lazy_block)
    return tr


# ---------------------------------------------------------------------------
# Cauchy-like (C4): x / G row blocks, y / B replicated.

def _all_gather_vec(x, group, world):
    if not dist.is_initialized():
        return x.reshape(-1)
    out = torch.empty(world * x.numel(), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, x.reshape(-1), group=group)
    return out


def run_sharded_cauchy(backend, steps, group=None, poll_every=16):
    """Per step: select (global stats, owner, pivot message), one
    sum-allreduce of the 20-double message (i, x_i, G_i; -0.0 from
    non-owners), update (pivot row regenerated on every rank, same column
    draw, local G rows + replicated B, local K5 masses), allgather of the
    [sum, max] row-mass stats."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    stats = backend.begin()
    totals = _all_gather_vec(stats, group, world)
    for t in range(steps):
        msg = backend.select(t, totals)
        if dist.is_initialized():
            dist.all_reduce(msg, op=dist.ReduceOp.SUM, group=group)
        stats = backend.update(t, msg)
        if t + 1 < steps:
            totals = _all_gather_vec(stats, group, world)
        if poll_every and (t + 1) % poll_every == 0 and not backend.active():
            break
    return backend.finish()


class CudaCauchyShardBackend:
    """Product backend: the rplu_cauchy_shard_* C ABI on this rank's GPU.
    M_local is a CauchyLikeMatrix holding this rank's rows of x / G and the
    full y / B (updated in place)."""

    def __init__(self, M_local, row_offset, world, rank, rule, rng, steps, stop_tol=0.0,
                 keep_steps=False, ctx=None):
        from .cauchy import CauchyLikeMatrix  # noqa: F401  (type of M_local)
        self.M = M_local
        self.dev = M_local.device
        n_local, m = M_local.shape
        self.steps = steps
        self.C = self.R = self.A = None
        if keep_steps and steps > 0:
            self.C = torch.empty((steps, max(n_local, 1)), dtype=torch.complex128, device=self.dev)
            self.R = torch.empty((steps, m), dtype=torch.complex128, device=self.dev)
            self.A = torch.empty(steps, dtype=torch.complex128, device=self.dev)
        self.block = UniformBlock(rng, 3 * steps + 2) if rule == "rplu" else None
        self.msg = torch.empty(_ffi.CAUCHY_MSG_DOUBLES, dtype=torch.float64, device=self.dev)
        self.stats = torch.empty(2, dtype=torch.float64, device=self.dev)
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        self.args = _ffi.CauchyShardArgs(
            rule=_ffi.RULE_IDS[rule], p=M_local.displacement_rank, world=world, rank=rank,
            n_local=n_local, m=m, row_offset=row_offset, steps=steps, stop_tol=float(stop_tol),
            x=M_local.x.data_ptr() if n_local else None, y=M_local.y.data_ptr(),
            G=M_local.G.data_ptr() if n_local else None, Bt=M_local.Bt.data_ptr(),
            C=ptr(self.C), Rrow=ptr(self.R), a=ptr(self.A),
            uniforms=self.block.pointer() if self.block else None,
            n_uniforms=self.block.values.size if self.block else 0, stream=None)
        c = ctx if ctx is not None else _device.ctx(self.dev)
        self._ctx = c
        self._lib, self._h = c._lib, c.handle
        k = max(steps, 1)
        self.rows = np.zeros(k, dtype=np.int64)
        self.cols = np.zeros(k, dtype=np.int64)
        self.bmax = np.zeros(k)
        self.bsum = np.zeros(k)

    def _args(self):
        self.args.stream = torch.cuda.current_stream(self.dev).cuda_stream
        return ctypes.byref(self.args)

    def begin(self):
        _ffi.check(self._lib.rplu_cauchy_shard_begin(self._h, self._args(),
                                                     self.stats.data_ptr()))
        return self.stats

    def select(self, t, totals):
        totals = totals.contiguous()
        self._totals = totals
        _ffi.check(self._lib.rplu_cauchy_shard_select(self._h, self._args(), t,
                                                      totals.data_ptr(), self.msg.data_ptr()))
        return self.msg

    def update(self, t, msg):
        _ffi.check(self._lib.rplu_cauchy_shard_update(self._h, self._args(), t, msg.data_ptr(),
                                                      self.stats.data_ptr()))
        return self.stats

    def active(self):
        a = ctypes.c_int32(0)
        _ffi.check(self._lib.rplu_cauchy_shard_active(self._h, self._args(), ctypes.byref(a)))
        return bool(a.value)

    def finish(self):
        i64p = ctypes.POINTER(ctypes.c_int64)
        f64p = ctypes.POINTER(ctypes.c_double)
        out = _ffi.CauchyOut(rows=self.rows.ctypes.data_as(i64p),
                             cols=self.cols.ctypes.data_as(i64p),
                             bound_maxes=self.bmax.ctypes.data_as(f64p),
                             bound_sums=self.bsum.ctypes.data_as(f64p))
        status = self._lib.rplu_cauchy_shard_finish(self._h, self._args(), ctypes.byref(out))
        if self.block is not None:
            self.block.commit(out.uniforms_consumed)
        _ffi.check(status)
        return out


def sharded_structured_eliminate(M_local, row_offset, rule, rank, stop_tol=0.0, rng=None,
                                 keep_steps=False, group=None):
    """Exact-norm structured RPLU (cauchy.py:177-256, plan=None) on a row
    shard: call on every rank with this rank's rows of x / G (M_local, a
    CauchyLikeMatrix whose y / B are the full, replicated generators) and an
    RngState with the same seed.  Returns a StructuredPivotTrace with GLOBAL
    row indices, the global bound statistics, ``residual`` = M_local after
    the updates (local G rows, replicated B), and with keep_steps the LOCAL
    rows of each column c (``steps_device`` = (C_local, R, a)).
    """
    from .cauchy import CauchyLikeMatrix, StructuredPivotTrace
    if rule not in ("rplu", "c2plu"):
        raise ValueError(f"unknown structured rule {rule!r}")
    if rule == "rplu" and rng is None:
        raise ValueError("structured rplu needs an RngState")
    if not isinstance(M_local, CauchyLikeMatrix):
        raise CapabilityError("sharded_structured_eliminate needs a CauchyLikeMatrix")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank_id = dist.get_rank(group) if dist.is_initialized() else 0
    n_local, m = M_local.shape
    n_global = n_local
    if dist.is_initialized():
        nt = torch.tensor([n_local], dtype=torch.int64,
                          device=M_local.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(nt, group=group)
        n_global = int(nt.item())
    if not 0 <= rank <= min(n_global, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n_global, m)}]")
    if rank == 0:
        return StructuredPivotTrace(residual=M_local)
    be = CudaCauchyShardBackend(M_local, row_offset, world, rank_id, rule, rng, rank,
                                stop_tol=stop_tol, keep_steps=keep_steps)
    out = run_sharded_cauchy(be, rank, group=group)
    k, nb = int(out.steps_done), int(out.bounds_recorded)
    tr = StructuredPivotTrace(
        row_indices=[int(v) for v in be.rows[:k]], col_indices=[int(v) for v in be.cols[:k]],
        bound_sums=[float(v) for v in be.bsum[:nb]], bound_maxes=[float(v) for v in be.bmax[:nb]],
        tol_stop=bool(out.tol_stop), degenerate_stop=bool(out.degenerate_stop),
        near_boundary_draws=int(out.near_boundary_draws),
        uniforms_consumed=int(out.uniforms_consumed), residual=M_local)
    if be.C is not None:
        tr.steps_device = (be.C[:, :n_local], be.R, be.A)
    return tr


def bench_sharded(args, cfg, dist_mod, rank, world, dev, metric, unit, sampler_cls=None):
    """bench.py --gpus N leg: C3 row-block sharded over N ranks (strong scaling).

    Every rank builds the full seeded C3 input on its GPU (input construction,
    untimed) and keeps its row block.  K timed eliminations of `rank` pivots,
    CUDA events per rank, max over ranks.
    """
    import json
    import os

    from . import gen

    n, k, seed = cfg["n"], cfg["rank"], cfg["seed"]
    tdtype = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    esize = 4 if cfg["dtype"] == "f32" else 8
    lo, hi = shard_rows(n, world, rank)
    A = gen.c3_dense_device(seed, n=n, dtype=tdtype, device=dev)
    A_loc = A[lo:hi].clone()
    del A
    torch.cuda.empty_cache()

    sweep_ev = []

    def hook(kind, t):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        sweep_ev.append(e)

    # RPLU_SHARD_UPDATE=lazy (default: delayed updates, one flush block with
    # its collectives captured in a CUDA graph and replayed) or eager (fused
    # K3 update; one step captured and replayed); RPLU_SHARD_GRAPH=0: host
    # step loop
    mode = os.environ.get("RPLU_SHARD_UPDATE", "lazy")
    use_graph = os.environ.get("RPLU_SHARD_GRAPH", "1") == "1"
    lazy_used = [0]

    def one(timed=False):
        tr = sharded_eliminate(A_loc, lo, PivotRule("rplu", _rng(seed)), k,
                               compute_dtype=tdtype, step_hook=hook if timed else None,
                               graph=use_graph and not timed, update=mode)
        lazy_used[0] = tr.lazy_block
        return tr

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    sampler = sampler_cls(torch.cuda.current_device()) if sampler_cls is not None else None
    if sampler is not None:
        sampler.start()
        time.sleep(0.3)
    dist_mod.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tr = one()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    clk = sampler.stop() if sampler is not None else None
    # per-update durations from a second pass of the same runs with CUDA
    # events around every update (plain launches, no graph)
    dist_mod.barrier()
    for _ in range(args.steps):
        one(timed=True)
    torch.cuda.synchronize()
    upd = sum(sweep_ev[2 * q].elapsed_time(sweep_ev[2 * q + 1])
              for q in range(len(sweep_ev) // 2))
    nupd = len(sweep_ev) // 2
    upd_t = torch.tensor([upd / max(nupd, 1)], dtype=torch.float64, device=dev)
    dist_mod.all_reduce(ms, op=dist_mod.ReduceOp.MAX)
    dist_mod.all_reduce(upd_t, op=dist_mod.ReduceOp.MAX)
    total_ms = float(ms)
    value = args.steps * tr.steps / (total_ms / 1e3)
    # e2e: host row block in (pinned), L rows / U / pivots out, per rank
    host = torch.empty(A_loc.shape, dtype=tdtype, pin_memory=True)
    host.copy_(A_loc)
    dist_mod.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    trh = sharded_eliminate(host.numpy(), lo, PivotRule("rplu", _rng(seed)), k,
                            compute_dtype=tdtype)
    Lh = torch.as_tensor(_device.to_numpy(trh.L.contiguous()) if torch.is_tensor(trh.L) else trh.L)
    Uh = torch.as_tensor(_device.to_numpy(trh.U.contiguous()) if torch.is_tensor(trh.U) else trh.U)
    f1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    dist_mod.all_reduce(ems, op=dist_mod.ReduceOp.MAX)
    # algorithmic bytes per update: read + write of the row block (eager, or
    # a lazy flush), a read (lazy pass); averaged over the k steps
    b = lazy_used[0]
    blk = (hi - lo) * n * esize
    if b > 0:
        nflush = sum(1 for t in range(k) if (t + 1) % b == 0 or t == k - 1)
        bytes_launch = blk * (k + nflush) / k
    else:
        bytes_launch = 2.0 * blk
    achieved = bytes_launch / (float(upd_t) / 1e3) / 1e9
    peak = 6553.6
    try:
        import os
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    except Exception:
        pass
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic (seeded BASELINE construction)",
            "config": {"workload": cfg["desc"], "n": n, "m": n, "rank": k, "seed": seed,
                       "parallelism": f"row-block shards x{world} (NCCL allgather + allreduce)",
                       "step_loop": (("CUDA graph of one flush block replayed" if b else
                                      "CUDA graph of one step replayed") if use_graph else "host loop"),
                       "update": f"delayed (flush every {b} steps)" if b else "eager (K3)",
                       "step": f"one full elimination of {k} pivot steps",
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)",
                         "launch_timing": "CUDA events around every update, second pass of the "
                                          "same runs, max over ranks",
                         "kernel": ("shard update (post + pivot column + delayed-update pass + local total)"
                                    if b else "shard update (post + K3 sweep + local total)")
                                   + ", per rank, max over ranks",
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "avg_launch_ms": float(upd_t)},
            "e2e": {"value": trh.steps / (float(ems) / 1e3), "unit": unit,
                    "h2d_bytes_per_step": (hi - lo) * n * esize * world,
                    "d2h_bytes_per_step": (Lh.numel() + Uh.numel()) * esize},
            "gpu_launches": args.steps * (((6 if b else 3) * k) + 3),
            "near_boundary_draws": tr.near_boundary_draws,
            "clocks": clk if clk is not None else {"sm_mhz": None, "reasons": ["not sampled"]},
        }
        print(json.dumps(line), flush=True)


def _rng(seed):
    from .rng import RngState
    return RngState(seed)
