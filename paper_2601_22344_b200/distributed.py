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

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _ffi
from .accessors import CapabilityError
from .dense_pivots import EliminationTrace, PivotRule
from .rng import UniformBlock

__all__ = ["shard_rows", "run_sharded", "run_sharded_graph", "sharded_eliminate",
           "CudaShardBackend"]


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


def run_sharded_graph(backend, steps, group=None, chunk=32):
    """The same choreography with one step (select, allreduce, update,
    allgather) captured once in a CUDA graph and replayed: the kernels read
    the step index from the device counter, the collectives run on static
    buffers.  Replays go in chunks of `chunk` steps with a stop poll between
    chunks."""
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
    with torch.cuda.graph(g):
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

    def __init__(self, R, row_offset, world, rank, rule, steps, stop_tol=0.0, ctx=None):
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
            stream=None)
        c = ctx if ctx is not None else _device.ctx(self.dev)
        self._ctx = c
        self._lib, self._h = c._lib, c.handle
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
        return dict(pivots=[(int(self.pivots[2 * t]), int(self.pivots[2 * t + 1]))
                            for t in range(k)],
                    resid_fro=self.resid[:k + 1].copy(), steps=k,
                    clean_early_stop=bool(out.clean_early_stop), tol_stop=bool(out.tol_stop),
                    near_boundary_draws=int(out.near_boundary_draws),
                    uniforms_consumed=int(out.uniforms_consumed),
                    L_local=self.Lt[:k, :self.n_local].T, U=self.U[:k, :self.m])


def sharded_eliminate(A_local, row_offset, rule, steps, stop_tol=0.0, group=None,
                      compute_dtype=None, overwrite_a=False, step_hook=None, graph=False):
    """RPLU on a row-block shard (call on every rank with the same rule seed).

    ``A_local`` is this rank's contiguous row block (global rows
    [row_offset, row_offset + n_local)); every rank must pass the same
    ``steps``/``stop_tol`` and an RngState with the same seed.  Returns an
    EliminationTrace whose L holds this rank's rows of L (device tensor) and
    whose U / pivots / resid_fro are the global (replicated) values.
    """
    if isinstance(rule, str):
        rule = PivotRule(rule)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    src = _device.as_device_matrix(A_local, dtype=compute_dtype, copy=False)
    vec = _device.vec_of(src.dtype)
    if (overwrite_a or src is not A_local) and src.is_contiguous() and src.shape[1] % vec == 0:
        R = src
    else:
        R = _device.padded_residual(src)[0]
    n_local, m = src.shape
    backend = CudaShardBackend(R, row_offset, world, rank, rule, steps, stop_tol)
    if graph and step_hook is None:
        res = run_sharded_graph(backend, steps, group=group)
    else:
        res = run_sharded(backend, steps, group=group, step_hook=step_hook)
    tr = EliminationTrace(
        pivots=res["pivots"], L=res["L_local"], U=res["U"], resid_fro=res["resid_fro"],
        residual=R[:, :m], steps=res["steps"], clean_early_stop=res["clean_early_stop"],
        tol_stop=res["tol_stop"], near_boundary_draws=res["near_boundary_draws"],
        uniforms_consumed=res["uniforms_consumed"], host=False)
    return tr


def bench_sharded(args, cfg, dist_mod, rank, world, dev, metric, unit):
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

    use_graph = os.environ.get("RPLU_SHARD_GRAPH", "1") == "1"

    def one(timed=False):
        return sharded_eliminate(A_loc, lo, PivotRule("rplu", _rng(seed)), k,
                                 compute_dtype=tdtype, step_hook=hook if timed else None,
                                 graph=use_graph and not timed)

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    dist_mod.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tr = one(timed=not use_graph)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if use_graph:
        # per-update durations from a second, hook-timed (non-graph) pass
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
    Lh, Uh = trh.L.cpu(), trh.U.cpu()
    f1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    dist_mod.all_reduce(ems, op=dist_mod.ReduceOp.MAX)
    bytes_launch = 2.0 * (hi - lo) * n * esize
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
                       "step_loop": "CUDA graph of one step replayed" if use_graph else "host loop",
                       "step": f"one full elimination of {k} pivot steps",
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "shard update (post + K3 sweep + local total), per rank, max over ranks",
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "avg_launch_ms": float(upd_t)},
            "e2e": {"value": trh.steps / (float(ems) / 1e3), "unit": unit,
                    "h2d_bytes_per_step": (hi - lo) * n * esize * world,
                    "d2h_bytes_per_step": (Lh.numel() + Uh.numel()) * esize},
            "gpu_launches": args.steps * (3 * k + 3) * 1,
            "near_boundary_draws": tr.near_boundary_draws,
        }
        print(json.dumps(line), flush=True)


def _rng(seed):
    from .rng import RngState
    return RngState(seed)
