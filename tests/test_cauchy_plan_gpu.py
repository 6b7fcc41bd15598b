"""Certified tree bounds (Alg C.2, device) and structured RPLU with a plan
(rejection sampling, cauchy.py:207-277) against the reference's goldens.

Bars: bounds to 1e-12 relative of the reference's and certified
(exact <= u <= nu * exact up to rounding); pivots, proposal / acceptance
counts and the uniform stream identical; bound sums / maxes to 1e-11; the
pivot rows r to 1e-10 relative.
"""

import numpy as np
import pytest

import paper_2601_22344_b200 as rp
from conftest import load_golden
from paper_2601_22344_b200 import gen

pytestmark = pytest.mark.gpu


def _cases():
    info, _ = load_golden("cauchy_plan")
    return info["cases"]


def _setup(case, arr):
    name = case["name"]
    x, y, G, B = (arr[name + k] for k in ("_x", "_y", "_G", "_B"))
    M = rp.CauchyLikeMatrix(x, y, G, B)
    plan = rp.build_plan(x, y, nu=case["nu"], leaf_size=case["leaf_size"])
    return M, plan


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_bounds_match_reference(case, cuda_device):
    _, arr = load_golden("cauchy_plan")
    M, plan = _setup(case, arr)
    name = case["name"]
    u = rp.certified_upper_bounds(plan, arr[name + "_G"], arr[name + "_B"])
    np.testing.assert_allclose(u, arr[name + "_u0"], rtol=1e-12)
    exact = arr[name + "_exact0"]
    assert np.all(u >= exact * (1 - 1e-12))
    assert np.all(u <= case["nu"] * exact * (1 + 1e-12))


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_structured_with_plan_matches_reference(case, cuda_device):
    _, arr = load_golden("cauchy_plan")
    M, plan = _setup(case, arr)
    rng = rp.RngState(case["seed"]) if case["seed"] is not None else None
    tr = rp.structured_eliminate(M, case["rule"], case["rank"], stop_tol=case["stop_tol"],
                                 nu=case["nu"], plan=plan, rng=rng, keep_steps=True)
    assert tr.row_indices == case["rows"]
    assert tr.col_indices == case["cols"]
    assert tr.proposals == case["proposals"]
    assert tr.acceptances == case["acceptances"]
    assert tr.exact_fallbacks == case["exact_fallbacks"]
    np.testing.assert_allclose(tr.bound_maxes, case["bound_maxes"], rtol=1e-11)
    np.testing.assert_allclose(tr.bound_sums, case["bound_sums"], rtol=1e-11)
    rs = arr[case["name"] + "_r"]
    for t, (c, r, a) in enumerate(tr.steps):
        assert np.abs(r - rs[t]).max() <= 1e-10 * np.abs(rs[t]).max()
    if rng is not None:
        assert rng.uniform() == case["next_uniform"]


def test_plan_bounds_certify_after_updates(cuda_device):
    """The plan is reused across generator updates: bounds stay certified."""
    x, y, G, B = gen.c4_cauchy_like(9, n=600, m=500, p=3)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    plan = rp.build_plan(x, y, nu=5.0, leaf_size=16)
    tr = rp.structured_eliminate(M, "rplu", 12, plan=plan, rng=rp.RngState(1))
    R = tr.residual
    u = rp.certified_upper_bounds(plan, R.G.cpu().numpy(), R.B.cpu().numpy())
    exact = rp.exact_row_norms(R)
    live = exact > 1e-20 * exact.max()
    assert np.all(u[live] >= exact[live] * (1 - 1e-10))
    assert np.all(u[live] <= 5.0 * exact[live] * (1 + 1e-10))
    assert tr.acceptances == len(tr.row_indices)


def test_plan_step_primitives_match_generator_formulas(cuda_device):
    """rplu_cauchy_plan_row / rplu_cauchy_plan_update (the plan path's fused
    K6 kernels) against the reference's row / column / generator-update
    formulas (cauchy.py:82-86, :247-250) evaluated in numpy."""
    import ctypes

    import torch

    from paper_2601_22344_b200 import _device, _ffi
    x, y, G, B = gen.c4_cauchy_like(7, n=300, m=260, p=3)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    n, m, p = 300, 260, 3
    dev = M.device
    c = _device.ctx(dev)
    st = _device.stream_handle(dev)
    rbuf = torch.empty(m, dtype=torch.complex128, device=dev)
    wbuf = torch.empty(m, dtype=torch.float64, device=dev)
    u = torch.rand(n, dtype=torch.float64, device=dev)
    out3 = np.zeros(3)
    i, j = 17, 41
    _ffi.check(c._lib.rplu_cauchy_plan_row(c.handle, p, n, m, M.x.data_ptr(), M.y.data_ptr(),
                                           M.G.data_ptr(), M.Bt.data_ptr(), i, rbuf.data_ptr(),
                                           wbuf.data_ptr(), u.data_ptr(), out3.ctypes.data, st))
    r = (G[i, :] @ B) / (x[i] - y)
    np.testing.assert_allclose(rbuf.cpu().numpy(), r, rtol=1e-13)
    np.testing.assert_allclose(wbuf.cpu().numpy(), np.abs(r) ** 2, rtol=1e-13)
    assert abs(out3[0] - np.sum(np.abs(r) ** 2)) <= 1e-13 * out3[0]
    assert out3[1] == np.max(np.abs(r)) and out3[2] == float(u[i])
    C = torch.empty(n, dtype=torch.complex128, device=dev)
    R = torch.empty(m, dtype=torch.complex128, device=dev)
    _ffi.check(c._lib.rplu_cauchy_plan_update(c.handle, p, n, m, M.x.data_ptr(), M.y.data_ptr(),
                                              M.G.data_ptr(), M.Bt.data_ptr(), i, j,
                                              rbuf.data_ptr(), C.data_ptr(), R.data_ptr(), st))
    a = r[j]
    col = (G @ B[:, j]) / (x - y[j])
    G1 = G - np.outer(col / a, G[i, :])
    B1 = B - np.outer(B[:, j], r / a)
    np.testing.assert_allclose(C.cpu().numpy(), col, rtol=1e-13)
    np.testing.assert_allclose(R.cpu().numpy(), r, rtol=1e-13)
    np.testing.assert_allclose(M.G.cpu().numpy(), G1, rtol=1e-12, atol=1e-14 * np.abs(G1).max())
    np.testing.assert_allclose(M.B.cpu().numpy(), B1, rtol=1e-12, atol=1e-14 * np.abs(B1).max())
    # after the update, row i and column j of the residual are (numerically) zero
    Mn = rp.CauchyLikeMatrix(x, y, M.G.cpu().numpy(), M.B.cpu().numpy(), check_points=False)
    assert np.abs(Mn.row(i)).max() <= 1e-12 * np.abs(r).max()
