"""World-size-2 gloo tests of the sharded driver on CPU.

The choreography (allgather of shard totals, root-free allreduce of the pivot
header and row with -0.0 contributions, global stop decisions) is the code
the GPU ranks run (paper_2601_22344_b200.distributed.run_sharded); here it
drives a numpy backend.  The sharded run must reproduce the single-process
oracle's pivots and factors.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _collect(q, procs, world, key, timeout=180):
    """Results of all workers; fails as soon as one exits non-zero."""
    import queue
    import time
    outs, t0 = [], time.time()
    while len(outs) < world:
        try:
            outs.append(q.get(timeout=1.0))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.time() - t0 > timeout:
                for p in procs:
                    p.kill()
                pytest.fail(f"shard worker failed (exit codes {dead})")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(outs, key=key)


def _worker(rank, world, port, A, seed, steps, stop_tol, lazy_block, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import NumpyShardBackend

        from paper_2601_22344_b200.distributed import run_sharded, shard_rows
        lo, hi = shard_rows(A.shape[0], world, rank)
        be = NumpyShardBackend(A[lo:hi], lo, world, rank, seed, steps, stop_tol,
                               lazy_block=lazy_block)
        res = run_sharded(be, steps, poll_every=4)
        out_q.put((rank, lo, hi, res["pivots"], res["resid_fro"], res["L_local"], res["U"],
                   res["status"], res["residual"]))
    finally:
        dist.destroy_process_group()


def _run(A, seed, steps, world=2, stop_tol=0.0, lazy_block=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, A, seed, steps, stop_tol,
                                                   lazy_block, q))
             for r in range(world)]
    for p in procs:
        p.start()
    return _collect(q, procs, world, key=lambda o: o[:3])


def test_shard_rows_partition():
    from paper_2601_22344_b200.distributed import shard_rows
    for n in (1, 7, 32768, 1000003):
        for w in (1, 2, 3, 8):
            blocks = [shard_rows(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[r][1] == blocks[r + 1][0] for r in range(w - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world,lazy_block", [(2, 0), (3, 0), (2, 3), (3, 5), (8, 0), (8, 4)])
def test_sharded_matches_single_process(world, lazy_block):
    import oracle
    from paper_2601_22344_b200 import gen
    A = gen.c1_dense(4, n=90, m=70)
    steps = 40
    outs = _run(A, seed=4, steps=steps, world=world, lazy_block=lazy_block)
    ref = oracle.eliminate_real(A, "rplu", steps, seed=4, margins=True)
    pivots = outs[0][3]
    for o in outs:
        assert o[3] == pivots, "ranks disagree on the pivot sequence"
    mism = [t for t, (a, b) in enumerate(zip(pivots, ref["pivots"])) if a != b]
    if mism:
        assert ref["margins"][mism[0]] <= oracle.NEAR_REL
        return
    assert pivots == ref["pivots"]
    L = np.concatenate([o[5] for o in outs], axis=0)
    np.testing.assert_array_equal(L, ref["L"])
    for o in outs:
        np.testing.assert_array_equal(o[6], ref["U"])
    np.testing.assert_allclose(outs[0][4], ref["resid_fro"], rtol=1e-12)
    np.testing.assert_array_equal(np.concatenate([o[8] for o in outs], axis=0), ref["residual"])


@pytest.mark.parametrize("lazy_block", [0, 5])
def test_sharded_tol_stop_is_global(lazy_block):
    """Every rank stops at the same step; with delayed updates finish applies
    the pending steps, so the residual equals the eager one."""
    import oracle
    from paper_2601_22344_b200 import gen
    A = gen.c1_dense(3, n=64)
    outs = _run(A, seed=3, steps=60, stop_tol=0.3, lazy_block=lazy_block)
    ref = oracle.eliminate_real(A, "rplu", 60, seed=3, stop_tol=0.3)
    assert ref["tol_stop"]
    assert ref["steps"] % 5 != 0   # the stop leaves pending steps
    for o in outs:
        assert o[7] == "tol"
        assert len(o[3]) == ref["steps"]
    if outs[0][3] == ref["pivots"]:
        np.testing.assert_array_equal(np.concatenate([o[8] for o in outs], axis=0), ref["residual"])


def test_negative_zero_allreduce_is_exact():
    """x + (-0.0) == x bit for bit, including x = -0.0 and tiny subnormals."""
    x = np.array([-0.0, 0.0, 5e-324, -5e-324, 1.0, -3.5, np.finfo(float).max])
    y = x + (-0.0)
    assert np.array_equal(x.view(np.int64), y.view(np.int64))


def _cauchy_worker(rank, world, port, x, y, G, B, rule, seed, steps, stop_tol, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import NumpyCauchyShardBackend

        from paper_2601_22344_b200.distributed import run_sharded_cauchy, shard_rows
        lo, hi = shard_rows(x.size, world, rank)
        be = NumpyCauchyShardBackend(x[lo:hi], y, G[lo:hi], B, lo, world, rank, rule, seed,
                                     steps, stop_tol)
        res = run_sharded_cauchy(be, steps, poll_every=4)
        out_q.put((rank, res["rows"], res["cols"], res["bound_maxes"], res["bound_sums"],
                   res["status"], res["G"], res["B"]))
    finally:
        dist.destroy_process_group()


def _run_cauchy(x, y, G, B, rule, seed, steps, world=2, stop_tol=0.0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cauchy_worker,
                         args=(r, world, port, x, y, G, B, rule, seed, steps, stop_tol, q))
             for r in range(world)]
    for p in procs:
        p.start()
    return _collect(q, procs, world, key=lambda o: o[0])


@pytest.mark.parametrize("world,rule,stop_tol", [(2, "rplu", 0.0), (3, "rplu", 1e-3),
                                                 (2, "c2plu", 0.0), (8, "rplu", 0.0)])
def test_sharded_cauchy_matches_single_process(world, rule, stop_tol):
    """Row-sharded Cauchy-like elimination (x / G sharded, y / B replicated)
    reproduces the single-process oracle: pivots, bound statistics, and the
    generators after the updates."""
    import oracle
    from paper_2601_22344_b200 import gen
    x, y, G, B = gen.c4_cauchy_like(5, n=150, m=130, p=3)
    steps = 80 if stop_tol else 40     # the tol case stops at step 70
    outs = _run_cauchy(x, y, G, B, rule, 5, steps, world=world, stop_tol=stop_tol)
    ref = oracle.structured_eliminate(x, y, G, B, rule, steps, seed=5, stop_tol=stop_tol)
    for o in outs:
        assert o[1] == outs[0][1] and o[2] == outs[0][2], "ranks disagree on the pivots"
    assert outs[0][1] == ref["row_indices"]
    assert outs[0][2] == ref["col_indices"]
    np.testing.assert_allclose(outs[0][3], ref["bound_maxes"], rtol=1e-12)
    np.testing.assert_allclose(outs[0][4], ref["bound_sums"], rtol=1e-12)
    if stop_tol:
        assert outs[0][5] == "tol" and ref["tol_stop"]
    # (BLAS blocks a row-block matvec differently from the full one: the
    # generators agree to rounding, the pivots and bounds exactly / 1e-12)
    Gs = np.concatenate([o[6] for o in outs], axis=0)
    np.testing.assert_allclose(Gs, ref["G"], rtol=1e-10, atol=1e-13 * np.abs(ref["G"]).max())
    for o in outs:
        np.testing.assert_allclose(o[7], ref["B"], rtol=1e-10,
                                   atol=1e-13 * np.abs(ref["B"]).max())


def _cur_worker(rank, world, port, A, seed, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu_backend import CpuDenseOp, NumpyCurOps

        import paper_2601_22344_b200 as rp
        from paper_2601_22344_b200.distributed import shard_rows
        from paper_2601_22344_b200.sharded_cur import TorchComm, sharded_cur_build
        lo, hi = shard_rows(A.shape[0], world, rank)
        op = CpuDenseOp(torch.from_numpy(A))
        fact, info = sharded_cur_build(op, (lo, hi), "rplu-cur", k, rng=rp.RngState(seed),
                                       comm=TorchComm(), ops=NumpyCurOps())
        out_q.put((rank, fact.row_indices, fact.col_indices, fact.core_matrix(),
                   info.row_norms, info.total_sq_norms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_cur_matches_oracle(world):
    """Row-sharded cur_build (replicated operator, local row norms / g / c
    rows, g[I] by a -0.0 allreduce) picks the oracle's skeleton."""
    import oracle
    rs = np.random.default_rng(11)
    n, m, k = 130, 110, 25
    U, _ = np.linalg.qr(rs.standard_normal((n, n)))
    V, _ = np.linalg.qr(rs.standard_normal((m, m)))
    A = (U[:, :m] * 0.8 ** np.arange(m)) @ V.T
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cur_worker, args=(r, world, port, A, 11, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = _collect(q, procs, world, key=lambda o: o[0])
    core, info = oracle.cur_build(oracle.DenseHost(A), "rplu-cur", k, seed=11)
    for o in outs:
        assert o[1] == core.I and o[2] == core.J
    np.testing.assert_allclose(outs[0][3], core.W, rtol=1e-12, atol=1e-14)
    rn = np.concatenate([o[4] for o in outs])
    # eliminated rows sit at the downdate's rounding floor (eps * total0)
    np.testing.assert_allclose(rn, info["row_norms"], rtol=1e-8,
                               atol=1e-14 * info["total_sq_norms"][0])
    np.testing.assert_allclose(outs[0][5], info["total_sq_norms"], rtol=1e-10)
