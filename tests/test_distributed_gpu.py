"""The sharded kernels on one GPU.

* world = 1: sharded_eliminate (no process group) == eliminate.
* 2 and 3 shards emulated in ONE process on one GPU: each shard has its own
  context; the collectives are replaced by device-side sums of the shards'
  buffers, issued sequentially (no kernel waits on another), so the real
  select / update kernels run with the multi-shard owner logic.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import _ffi, gen
from paper_2601_22344_b200.distributed import CudaShardBackend, shard_rows, sharded_eliminate

pytestmark = pytest.mark.gpu


def test_world1_equals_eliminate(cuda_device):
    A = torch.from_numpy(gen.c1_dense(2, n=400, m=300)).cuda()
    tr = sharded_eliminate(A, 0, rp.PivotRule("rplu", rp.RngState(2)), 100)
    ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(2)), 100)
    assert tr.pivots == ref.pivots
    assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
    np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-12)


def test_world1_graph_replay_equals_eliminate(cuda_device):
    """One step captured in a CUDA graph and replayed (device step counter)."""
    A = torch.from_numpy(gen.c1_dense(5, n=300, m=260)).cuda()
    tr = sharded_eliminate(A, 0, rp.PivotRule("rplu", rp.RngState(5)), 90, graph=True)
    ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(5)), 90)
    assert tr.pivots == ref.pivots
    assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
    np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-12)
    # a tol stop inside a replay chunk stops every later replay
    trs = sharded_eliminate(A, 0, rp.PivotRule("rplu", rp.RngState(5)), 250, stop_tol=0.5,
                            graph=True)
    refs = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(5)), 250, stop_tol=0.5)
    assert trs.tol_stop and refs.tol_stop and trs.pivots == refs.pivots


@pytest.mark.parametrize("dtype,lazy_block", [(torch.float64, 3), (torch.float64, -1),
                                              (torch.float32, 4), (torch.complex128, 2)])
def test_world1_lazy_equals_eager(dtype, lazy_block, cuda_device):
    """Delayed-update shard loop: pivots, L, U and the final residual are
    bit-identical to the single-GPU eager loop (also after a tol stop that
    leaves pending steps for finish to apply)."""
    A = gen.c1_dense(7, n=410, m=301)
    if dtype == torch.complex128:
        A = A + 1j * gen.c1_dense(8, n=410, m=301)
    A = torch.from_numpy(A).to("cuda", dtype)
    for steps, tol in ((101, 0.0), (250, 0.45)):
        tr = sharded_eliminate(A, 0, rp.PivotRule("rplu", rp.RngState(7)), steps,
                               stop_tol=tol, update="lazy", lazy_block=lazy_block)
        ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(7)), steps, stop_tol=tol,
                           update="eager")
        assert tr.lazy_block > 0
        assert tr.pivots == ref.pivots and tr.tol_stop == ref.tol_stop
        if tol:
            assert tr.tol_stop
        assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
        assert torch.equal(tr.residual_device, ref.residual_device)
        np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-13)


@pytest.mark.parametrize("update", ["eager", "lazy"])
def test_c_group_driver_world1(update, cuda_device):
    """rplu_group_dense_run (the C loop over NCCL from ncclCommInitAll, no
    torch.distributed) at one device: bit-identical to eliminate."""
    from paper_2601_22344_b200.distributed import group_eliminate
    A = torch.from_numpy(gen.c1_dense(4, n=600, m=450)).cuda()
    ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(4)), 120, update="eager")
    rng = rp.RngState(4)
    tr = group_eliminate(A, rp.PivotRule("rplu", rng), 120, devices=[0], update=update)
    assert tr.pivots == ref.pivots
    assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
    assert torch.equal(tr.residual_device, ref.residual_device)
    np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-12)
    assert (tr.lazy_block > 0) == (update == "lazy")
    ref2 = rp.RngState(4)
    rp.eliminate(A, rp.PivotRule("rplu", ref2), 120)
    assert rng.uniform() == ref2.uniform()


@pytest.mark.parametrize("graph_env", ["0", "1"])
def test_c_group_driver_lazy_graph_and_plain_loop(graph_env, cuda_device, monkeypatch):
    """The C group driver's delayed-update loop with its multi-device block
    graph (RPLU_GROUP_GRAPH unset / 1) and with the plain step loop (0), across
    a trailing partial block and a tol stop inside a replayed block."""
    from paper_2601_22344_b200.distributed import group_eliminate
    monkeypatch.setenv("RPLU_GROUP_GRAPH", graph_env)
    A = torch.from_numpy(gen.c1_dense(13, n=520, m=400)).cuda()
    for steps, tol in ((75, 0.0), (300, 0.4)):
        ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(8)), steps, stop_tol=tol,
                           update="eager")
        tr = group_eliminate(A, rp.PivotRule("rplu", rp.RngState(8)), steps, devices=[0],
                             stop_tol=tol, update="lazy")
        assert tr.pivots == ref.pivots and tr.tol_stop == ref.tol_stop
        assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
        assert torch.equal(tr.residual_device, ref.residual_device)
        np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-12)


@pytest.mark.parametrize("dtype,lazy_block,gram", [(torch.float64, -1, True), (torch.float64, 5, True),
                                                   (torch.float64, 4, False), (torch.float32, 6, False),
                                                   (torch.complex128, 3, False)])
def test_world1_lazy_block_graph(dtype, lazy_block, gram, cuda_device, monkeypatch):
    """Delayed-update shards with one whole flush block (kernels with
    block-relative steps + collectives) captured in a CUDA graph and replayed:
    bit-identical to the eager single-GPU loop for full blocks + a trailing
    partial block, for a run shorter than two blocks, and across a tol stop
    inside a replayed block."""
    A = gen.c1_dense(11, n=390, m=305)
    if dtype == torch.complex128:
        A = A + 1j * gen.c1_dense(12, n=390, m=305)
    A = torch.from_numpy(A).to("cuda", dtype)
    for steps, tol in ((77, 0.0), (19, 0.0), (250, 0.4)):
        tr = sharded_eliminate(A, 0, rp.PivotRule("rplu", rp.RngState(3)), steps, stop_tol=tol,
                               update="lazy", lazy_block=lazy_block, graph=True)
        ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(3)), steps, stop_tol=tol,
                           update="eager")
        assert tr.lazy_block > 0
        assert tr.pivots == ref.pivots and tr.tol_stop == ref.tol_stop
        assert torch.equal(tr.L, ref.L) and torch.equal(tr.U, ref.U)
        assert torch.equal(tr.residual_device, ref.residual_device)
        np.testing.assert_allclose(tr.resid_fro, ref.resid_fro, rtol=1e-13)


def test_emulated_shards_block_positions(cuda_device):
    """3 emulated shards driven with block-relative steps (t = -1 - position,
    the form a captured block replays) after an explicit first block."""
    A = gen.c1_dense(9, n=420, m=256)
    steps, world, b, seed = 40, 3, 4, 9
    bes = []
    for r in range(world):
        lo, hi = shard_rows(A.shape[0], world, r)
        R = torch.from_numpy(np.ascontiguousarray(A[lo:hi])).cuda()
        bes.append(CudaShardBackend(R, lo, world, r, rp.PivotRule("rplu", rp.RngState(seed)),
                                    steps, ctx=_ffi.Context(0), lazy_block=b))
    assert all(be.block_len == b for be in bes)
    totals = torch.cat([be.begin().clone() for be in bes])
    for t in range(steps + 1):
        tt = t if t < b or t == steps else -1 - (t % b)
        ms = [be.select(-1 if tt < 0 else tt, totals).clone() for be in bes]
        if t == steps:
            break
        msg = ms[0]
        for x in ms[1:]:
            msg = msg + x
        totals = torch.cat([be.update(tt, msg).clone() for be in bes])
    res = [be.finish() for be in bes]
    ref = oracle.eliminate_real(A, "rplu", steps, seed=seed)
    assert res[0]["pivots"] == ref["pivots"]
    L = torch.cat([r["L_local"] for r in res], dim=0).cpu().numpy()
    np.testing.assert_array_equal(L, ref["L"])
    np.testing.assert_array_equal(res[0]["U"].cpu().numpy(), ref["U"])


@pytest.mark.parametrize("world,lazy_block", [(2, 0), (3, 0), (2, 4), (3, 5), (8, 0), (8, 6)])
def test_emulated_shards(world, lazy_block, cuda_device):
    A = gen.c1_dense(6, n=500, m=333)
    steps = 120
    seed = 6
    bes = []
    for r in range(world):
        lo, hi = shard_rows(A.shape[0], world, r)
        R = torch.from_numpy(np.ascontiguousarray(A[lo:hi])).cuda()
        vec = 2
        if R.shape[1] % vec:
            buf = torch.zeros((hi - lo, ((R.shape[1] + 1) // 2) * 2), dtype=R.dtype, device="cuda")
            buf[:, :R.shape[1]] = R
            R = buf[:, :A.shape[1]]
        bes.append(CudaShardBackend(R, lo, world, r, rp.PivotRule("rplu", rp.RngState(seed)),
                                    steps, ctx=_ffi.Context(0), lazy_block=lazy_block))
    totals = torch.cat([b.begin().clone() for b in bes])
    # exercise the device step counter (t = -1) too (eager only)
    device_t = world == 3 and lazy_block == 0
    for t in range(steps + 1):
        tt = -1 if device_t else t
        ms = [b.select(tt, totals).clone() for b in bes]
        if t == steps:
            break
        msg = ms[0]
        for x in ms[1:]:
            msg = msg + x     # the allreduce(sum) with -0.0 contributions
        totals = torch.cat([b.update(tt, msg).clone() for b in bes])
    res = [b.finish() for b in bes]
    ref = oracle.eliminate_real(A, "rplu", steps, seed=seed, margins=True)
    for r in res:
        assert r["pivots"] == res[0]["pivots"]
    piv = res[0]["pivots"]
    mism = [t for t, (a, b) in enumerate(zip(piv, ref["pivots"])) if a != b]
    if mism:
        assert ref["margins"][mism[0]] <= oracle.NEAR_REL
        return
    L = torch.cat([r["L_local"] for r in res], dim=0).cpu().numpy()
    np.testing.assert_array_equal(L, ref["L"])
    np.testing.assert_array_equal(res[0]["U"].cpu().numpy(), ref["U"])
    np.testing.assert_allclose(res[0]["resid_fro"], ref["resid_fro"], rtol=1e-12)
    Rs = torch.cat([b.R for b in bes], dim=0).cpu().numpy()
    np.testing.assert_array_equal(Rs, ref["residual"])


def _emulate_dense(A_dev, world, steps, seed, lazy_block):
    """world shards of a device matrix on one GPU (own contexts; the
    allreduce / allgather replaced by device-side sums / concatenation)."""
    n, m = A_dev.shape
    bes = []
    for r in range(world):
        lo, hi = shard_rows(n, world, r)
        bes.append(CudaShardBackend(A_dev[lo:hi].clone(), lo, world, r,
                                    rp.PivotRule("rplu", rp.RngState(seed)), steps,
                                    ctx=_ffi.Context(0), lazy_block=lazy_block))
    totals = torch.cat([b.begin().clone() for b in bes])
    for t in range(steps + 1):
        ms = [b.select(t, totals).clone() for b in bes]
        if t == steps:
            break
        msg = ms[0]
        for x in ms[1:]:
            msg = msg + x
        totals = torch.cat([b.update(t, msg).clone() for b in bes])
    return bes, [b.finish() for b in bes]


@pytest.mark.parametrize("lazy_block", [0, 6])
def test_eight_shards_reduced_c3(lazy_block, cuda_device):
    """SURVEY §8(e) at G = 8 (emulated on one GPU): the reduced C3
    construction (n = 4096, 128 pivots), eager and delayed-update shard
    steps, pivots / L / U / residual bit-identical to the single-GPU eager
    elimination (the reference's rounding)."""
    A = gen.c3_dense_device(0, n=4096)
    ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 128, update="eager")
    bes, res = _emulate_dense(A, 8, 128, 0, lazy_block)
    for r in res:
        assert r["pivots"] == ref.pivots
    L = torch.cat([r["L_local"] for r in res], dim=0)
    assert torch.equal(L, ref.L) and torch.equal(res[0]["U"], ref.U)
    assert torch.equal(torch.cat([b.R for b in bes], dim=0), ref.residual_device)
    np.testing.assert_allclose(res[0]["resid_fro"], ref.resid_fro, rtol=1e-12)


# ---------------------------------------------------------------------------
# Sharded Cauchy-like (x / G row blocks, y / B replicated)

from paper_2601_22344_b200.distributed import (  # noqa: E402
    CudaCauchyShardBackend, sharded_structured_eliminate)


@pytest.mark.parametrize("rule", ["rplu", "c2plu"])
def test_cauchy_world1_equals_structured(rule, cuda_device):
    x, y, G, B = gen.c4_cauchy_like(3, n=700, m=600, p=4)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    rng = rp.RngState(3) if rule == "rplu" else None
    tr = sharded_structured_eliminate(M.copy(), 0, rule, 60, rng=rng, keep_steps=True)
    rng2 = rp.RngState(3) if rule == "rplu" else None
    ref = rp.structured_eliminate(M, rule, 60, rng=rng2, keep_steps=True)
    assert tr.row_indices == ref.row_indices and tr.col_indices == ref.col_indices
    assert tr.bound_maxes == ref.bound_maxes and tr.bound_sums == ref.bound_sums
    assert tr.uniforms_consumed == ref.uniforms_consumed
    assert torch.equal(tr.residual.G, ref.residual.G)
    assert torch.equal(tr.residual.Bt, ref.residual.Bt)
    for a, b in zip(tr.steps_device, ref.steps_device):
        assert torch.equal(a, b)
    if rng is not None:
        assert rng.uniform() == rng2.uniform()


@pytest.mark.parametrize("world,rule,stop_tol", [(2, "rplu", 0.0), (3, "rplu", 1e-3),
                                                 (2, "c2plu", 0.0)])
def test_cauchy_emulated_shards(world, rule, stop_tol, cuda_device):
    """2 / 3 shards on one GPU (own contexts, sums of the messages in place
    of the allreduce): pivots and bounds as the oracle, generators to
    rounding, keep_steps columns of every shard."""
    x, y, G, B = gen.c4_cauchy_like(5, n=900, m=700, p=3)
    steps = 100 if stop_tol else 60
    ref = oracle.structured_eliminate(x, y, G, B, rule, steps, seed=5, stop_tol=stop_tol,
                                      keep_steps=True, margins=True)
    bes, blocks = [], []
    for r in range(world):
        lo, hi = shard_rows(x.size, world, r)
        blocks.append((lo, hi))
        Ml = rp.CauchyLikeMatrix(x[lo:hi], y, G[lo:hi], B, check_points=False)
        rng = rp.RngState(5) if rule == "rplu" else None
        bes.append(CudaCauchyShardBackend(Ml, lo, world, r, rule, rng, steps,
                                          stop_tol=stop_tol, keep_steps=True,
                                          ctx=_ffi.Context(0)))
    stats = torch.cat([b.begin().clone() for b in bes])
    for t in range(steps):
        ms = [b.select(t, stats).clone() for b in bes]
        msg = ms[0]
        for m2 in ms[1:]:
            msg = msg + m2
        stats = torch.cat([b.update(t, msg).clone() for b in bes])
    outs = [b.finish() for b in bes]
    k = int(outs[0].steps_done)
    rows = [int(v) for v in bes[0].rows[:k]]
    cols = [int(v) for v in bes[0].cols[:k]]
    for b in bes[1:]:
        assert [int(v) for v in b.rows[:k]] == rows and [int(v) for v in b.cols[:k]] == cols
    mism = [t for t, (a, c) in enumerate(zip(rows, ref["row_indices"])) if a != c]
    if mism:
        assert ref["margins"][mism[0]] <= oracle.NEAR_REL
        return
    assert rows == ref["row_indices"] and cols == ref["col_indices"]
    assert bool(outs[0].tol_stop) == ref["tol_stop"]
    nb = int(outs[0].bounds_recorded)
    np.testing.assert_allclose(bes[0].bmax[:nb], ref["bound_maxes"], rtol=1e-11)
    np.testing.assert_allclose(bes[0].bsum[:nb], ref["bound_sums"], rtol=1e-11)
    Gs = torch.cat([b.M.G for b in bes]).cpu().numpy()
    np.testing.assert_allclose(Gs, ref["G"], rtol=1e-9, atol=1e-12 * np.abs(ref["G"]).max())
    for b in bes:
        Bt = b.M.Bt.cpu().numpy()
        np.testing.assert_allclose(Bt.T, ref["B"], rtol=1e-9, atol=1e-12 * np.abs(ref["B"]).max())
    C = torch.cat([b.C[:k, :hi - lo] for b, (lo, hi) in zip(bes, blocks)], dim=1).cpu().numpy()
    for t, (c, r, a) in enumerate(ref["steps"]):
        assert np.abs(C[t] - c).max() <= 1e-10 * np.abs(c).max()
        assert np.abs(bes[0].R[t].cpu().numpy() - r).max() <= 1e-10 * np.abs(r).max()


@pytest.mark.slow
def test_cauchy_one_vs_eight_shards_full_n(cuda_device):
    """SURVEY §8(d) C4 bar "1-vs-8-GPU pivot identity at full n": the C4
    generators at n = m = 2^20, p = 4, three pivot steps, single GPU against
    8 emulated shards: identical pivots and bound sums / maxes to 1e-11."""
    x, y, G, B = gen.c4_cauchy_like(0)
    K = 3
    ref = rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B, check_points=False), "rplu",
                                  K, rng=rp.RngState(0))
    world = 8
    bes = []
    for r in range(world):
        lo, hi = shard_rows(x.size, world, r)
        Ml = rp.CauchyLikeMatrix(x[lo:hi], y, G[lo:hi], B, check_points=False)
        bes.append(CudaCauchyShardBackend(Ml, lo, world, r, "rplu", rp.RngState(0), K,
                                          ctx=_ffi.Context(0)))
    stats = torch.cat([b.begin().clone() for b in bes])
    for t in range(K):
        ms = [b.select(t, stats).clone() for b in bes]
        msg = ms[0]
        for m2 in ms[1:]:
            msg = msg + m2
        stats = torch.cat([b.update(t, msg).clone() for b in bes])
    outs = [b.finish() for b in bes]
    k = int(outs[0].steps_done)
    assert k == K
    for b in bes:
        assert [int(v) for v in b.rows[:k]] == ref.row_indices
        assert [int(v) for v in b.cols[:k]] == ref.col_indices
    np.testing.assert_allclose(bes[0].bmax[:k], ref.bound_maxes[:k], rtol=1e-11)
    np.testing.assert_allclose(bes[0].bsum[:k], ref.bound_sums[:k], rtol=1e-11)


# ---------------------------------------------------------------------------
# Sharded matrix-free CUR (C5): rows of the generated GEMV per shard

from paper_2601_22344_b200.sharded_cur import sharded_cur_build  # noqa: E402
from thread_comm import run_ranks  # noqa: E402


@pytest.mark.parametrize("world,rule", [(1, "rplu-cur"), (2, "rplu-cur"), (3, "rplu-cur"),
                                        (2, "c2plu-cur")])
def test_sharded_cur_matches_single_gpu(world, rule, cuda_device):
    """Shards emulated by threads on one GPU reproduce the single-GPU
    cur_build skeleton (index sets) and core; the local maintained norms
    concatenate to the single-GPU ones."""
    P, Q = gen.c5_points(4, n=3000, m=2500)
    A = rp.GaussianKernelOperator(P, Q, h=0.1)
    k = 40
    mk = (lambda: rp.RngState(4)) if rule == "rplu-cur" else (lambda: None)
    fact, info = rp.cur_build(A, rule, k, rng=mk())

    def one(r, comm):
        lo, hi = shard_rows(3000, world, r)
        return sharded_cur_build(A, (lo, hi), rule, k, rng=mk(), comm=comm)

    res = run_ranks(world, one)
    for f, inf in res:
        assert f.row_indices == fact.row_indices and f.col_indices == fact.col_indices
        np.testing.assert_allclose(f.core_matrix(), fact.core_matrix(), rtol=1e-12, atol=1e-15)
    rn = np.concatenate([inf.row_norms for _, inf in res])
    np.testing.assert_allclose(rn, info.row_norms, rtol=1e-7,
                               atol=1e-13 * info.total_sq_norms[0])
    np.testing.assert_allclose(res[0][1].total_sq_norms, info.total_sq_norms, rtol=1e-10)
    assert res[0][1].uniforms_consumed == info.uniforms_consumed
