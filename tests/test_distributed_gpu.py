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


@pytest.mark.parametrize("world", [2, 3])
def test_emulated_shards(world, cuda_device):
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
                                    steps, ctx=_ffi.Context(0)))
    totals = torch.cat([b.begin().clone() for b in bes])
    device_t = world == 3   # exercise the device step counter (t = -1) too
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
