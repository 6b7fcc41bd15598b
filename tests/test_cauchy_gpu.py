"""Parity of the B200 Cauchy-like path (structured_eliminate, plan=None ->
rplu_cauchy_run -> K5/K2/K6) with the reference goldens and the oracle.

Bars: pivots identical (a divergence must coincide with an oracle draw within
1e-12 relative of a CDF boundary); L/U (c/a, r) to 1e-10 relative; bound
sums/maxes to 1e-12 relative; the caller's uniform stream advanced exactly.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2601_22344_b200 as rp
from conftest import load_golden
from paper_2601_22344_b200 import gen

pytestmark = pytest.mark.gpu


def _cases():
    info, _ = load_golden("cauchy")
    return info["cases"]


def _first_mismatch(a, b):
    for t, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return t
    return None


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_cauchy_golden(case, cuda_device):
    _, arr = load_golden("cauchy")
    name = case["name"]
    x, y, G, B = (arr[name + k] for k in ("_x", "_y", "_G", "_B"))
    M = rp.CauchyLikeMatrix(x, y, G, B)
    np.testing.assert_allclose(rp.exact_row_norms(M), arr[name + "_norms0"], rtol=1e-13)
    rng = rp.RngState(case["seed"]) if case["seed"] is not None else None
    tr = rp.structured_eliminate(M, case["rule"], case["rank"], stop_tol=case["stop_tol"],
                                 rng=rng, keep_steps=True)
    assert tr.row_indices == case["rows"]
    assert tr.col_indices == case["cols"]
    assert tr.tol_stop == case["tol_stop"]
    assert tr.degenerate_stop == case["degenerate_stop"]
    np.testing.assert_allclose(tr.bound_maxes, case["bound_maxes"], rtol=1e-11)
    np.testing.assert_allclose(tr.bound_sums, case["bound_sums"], rtol=1e-11)
    k = len(case["rows"])
    if k:
        c = np.stack([s[0] for s in tr.steps])
        r = np.stack([s[1] for s in tr.steps])
        a = np.array([s[2] for s in tr.steps])
        ca, ra, aa = arr[name + "_c"], arr[name + "_r"], arr[name + "_a"]
        # L = c/a, U = r to 1e-10 relative (per step, scaled by the step's max)
        for t in range(k):
            lt, lref = c[t] / a[t], ca[t] / aa[t]
            assert np.abs(lt - lref).max() <= 1e-10 * np.abs(lref).max()
            assert np.abs(r[t] - ra[t]).max() <= 1e-10 * np.abs(ra[t]).max()
    if rng is not None:
        assert rng.uniform() == case["next_uniform"]


def test_validation(cuda_device):
    x, y, G, B = gen.c2_cauchy(0, n=32)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    with pytest.raises(ValueError):
        rp.structured_eliminate(M, "bogus", 2, rng=rp.RngState(0))
    with pytest.raises(ValueError):
        rp.structured_eliminate(M, "rplu", 2)
    with pytest.raises(ValueError):
        rp.structured_eliminate(M, "rplu", 33, rng=rp.RngState(0))
    with pytest.raises(ValueError):
        rp.structured_eliminate(M, "rplu", 2, rng=rp.RngState(0), plan=object())
    with pytest.raises(ValueError):
        rp.CauchyLikeMatrix(x, x, G, B)          # coincident points
    with pytest.raises(ValueError):
        rp.CauchyLikeMatrix(x, y, np.ones((32, 9)), np.ones((9, 32)))
    tr = rp.structured_eliminate(M, "rplu", 0, rng=rp.RngState(0))
    assert tr.rank == 0 and tr.bound_maxes == []


def test_generator_update_matches_dense_schur(cuda_device):
    """SPEC acceptance 9: generator-updated residuals equal the dense Schur
    complements entrywise to 1e-10 over 5 steps (p in {1, 2}, n = m = 40)."""
    for p in (1, 2):
        x, y, G, B = gen.c4_cauchy_like(p, n=40, p=p)
        M = rp.CauchyLikeMatrix(x, y, G, B)
        D = M.materialize()
        rs = np.random.default_rng(p)
        for _ in range(5):
            i, j = int(rs.integers(40)), int(rs.integers(40))
            while abs(D[i, j]) < 1e-3 * np.abs(D).max():
                i, j = int(rs.integers(40)), int(rs.integers(40))
            D = D - np.outer(D[:, j] / D[i, j], D[i, :])
            M = rp.generator_schur_update(M, (i, j))
            E = M.materialize()
            assert np.abs(E - D).max() <= 1e-10 * np.abs(D).max()


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_generator_schur_update_k6(p, cuda_device):
    """a11: the public single-step update runs the K6 kernels: G1, B1 equal to
    the oracle's restatement of cauchy.py:140-154 to the last few ulps (the
    reference's G[i] @ B and G @ B[:, j] are OpenBLAS zgemv calls whose
    internal FMA order is not reproduced; the quotient, the Smith division
    and the outer update follow numpy); the input generators are untouched;
    the relative zero-pivot guard raises ZeroDivisionError."""

    def close(a, b):
        assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()
    x, y, G, B = gen.c4_cauchy_like(p + 10, n=300, m=257, p=p)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    G0, Bt0 = M.G.clone(), M.Bt.clone()
    for (i, j) in [(0, 0), (17, 200), (299, 256)]:
        M1 = rp.generator_schur_update(M, (i, j))
        G1, B1 = oracle.generator_schur_update(x, y, G, B, i, j)
        close(M1.G.cpu().numpy(), G1)
        close(M1.Bt.cpu().numpy(), B1.T)
    assert torch.equal(M.G, G0) and torch.equal(M.Bt, Bt0)
    # chained: a second update on the updated generators
    M2 = rp.generator_schur_update(rp.generator_schur_update(M, (5, 9)), (40, 3))
    Ga, Ba = oracle.generator_schur_update(x, y, G, B, 5, 9)
    Gb, Bb = oracle.generator_schur_update(x, y, Ga, Ba, 40, 3)
    close(M2.G.cpu().numpy(), Gb)
    close(M2.Bt.cpu().numpy(), Bb.T)
    # eliminated row / column are numerically zero afterwards
    E = M2.materialize()
    assert np.abs(E[40]).max() <= 1e-12 * np.abs(M.materialize()).max()
    z = rp.CauchyLikeMatrix(x[:4], y[:4], np.zeros((4, 1)) + 0j, np.ones((1, 4)) + 0j)
    with pytest.raises(ZeroDivisionError):
        rp.generator_schur_update(z, (1, 2))


def test_structured_equals_dense_pivots(cuda_device):
    """With exact norms, structured RPLU picks the dense path's pivots
    (SURVEY §4 probe 2) — both sides on the GPU."""
    x, y, G, B = gen.c4_cauchy_like(7, n=300, p=2)
    M = rp.CauchyLikeMatrix(x, y, G, B)
    tr = rp.structured_eliminate(M, "rplu", 40, rng=rp.RngState(9), keep_steps=True)
    dtr = rp.eliminate(M.materialize(), rp.PivotRule("rplu", rp.RngState(9)), 40)
    got = list(zip(tr.row_indices, tr.col_indices))
    t = _first_mismatch(got, dtr.pivots)
    assert t is None or t > 30, (t, got[:5], dtr.pivots[:5])
    L, U = tr.factors()
    k = 40 if t is None else t
    np.testing.assert_allclose(L[:, :k].cpu().numpy(), dtr.L[:, :k], rtol=0, atol=1e-12 * np.abs(dtr.L).max())


@pytest.mark.parametrize("n,p,K,seed", [(4096, 1, 40, 0), (2048, 4, 24, 1)])
def test_vs_oracle_reduced(n, p, K, seed, cuda_device):
    if p == 1:
        x, y, G, B = gen.c2_cauchy(seed, n=n)
    else:
        x, y, G, B = gen.c4_cauchy_like(seed, n=n, p=p)
    ref = oracle.structured_eliminate(x, y, G, B, "rplu", K, seed=seed, keep_steps=True,
                                      margins=True)
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    tr = rp.structured_eliminate(M, "rplu", K, rng=rp.RngState(seed), keep_steps=True)
    got = list(zip(tr.row_indices, tr.col_indices))
    want = list(zip(ref["row_indices"], ref["col_indices"]))
    t = _first_mismatch(got, want)
    if t is not None:
        assert ref["margins"][t] <= oracle.NEAR_REL, f"divergence at {t} not near a boundary"
        K = t
    np.testing.assert_allclose(tr.bound_maxes[:K], ref["bound_maxes"][:K], rtol=1e-11)
    for s in range(K):
        c, r, a = tr.steps[s]
        rc, rr, ra = ref["steps"][s]
        assert np.abs(r - rr).max() <= 1e-10 * np.abs(rr).max()
        assert np.abs(c / a - rc / ra).max() <= 1e-10 * np.abs(rc / ra).max()


@pytest.mark.parametrize("n,m,p,rule,K,tol", [
    (4096, 4096, 1, "rplu", 60, 0.0), (700, 523, 2, "rplu", 48, 0.0), (300, 300, 1, "c2plu", 30, 0.0),
    (1000, 640, 1, "rplu", 200, 1e-3), (5, 9, 2, "rplu", 5, 0.0), (2600, 1500, 2, "c2plu", 16, 0.0)])
def test_resident_loop_matches_stepwise(n, m, p, rule, K, tol, cuda_device):
    """The resident cooperative loop (one launch, one grid barrier per step)
    against the per-step kernels on the same inputs: same pivots, stop flags
    and uniform consumption; columns, rows, pivot values and the final
    generators to rounding (the mass summation order differs, nothing else)."""
    if p == 1 and n == m:
        x, y, G, B = gen.c2_cauchy(4, n=n)
    else:
        x, y, G, B = gen.c4_cauchy_like(4, n=n, m=m, p=p)
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    r1, r2 = rp.RngState(11), rp.RngState(11)
    a = rp.structured_eliminate(M, rule, K, stop_tol=tol, rng=r1, keep_steps=True)
    b = rp.structured_eliminate(M, rule, K, stop_tol=tol, rng=r2, keep_steps=True,
                                persistent=False)
    assert a.row_indices == b.row_indices and a.col_indices == b.col_indices
    assert a.tol_stop == b.tol_stop and a.degenerate_stop == b.degenerate_stop
    assert r1.uniform() == r2.uniform()
    np.testing.assert_allclose(a.bound_maxes, b.bound_maxes, rtol=1e-12)
    np.testing.assert_allclose(a.bound_sums, b.bound_sums, rtol=1e-12)
    for (ca, ra, aa), (cb, rb, ab) in zip(a.steps, b.steps):
        np.testing.assert_array_equal(ra, rb)      # same generators in -> same bits
        np.testing.assert_array_equal(ca, cb)
        assert aa == ab
    np.testing.assert_array_equal(a.residual.G.cpu().numpy(), b.residual.G.cpu().numpy())
    np.testing.assert_array_equal(a.residual.Bt.cpu().numpy(), b.residual.Bt.cpu().numpy())


def test_c2plu_rule(cuda_device):
    x, y, G, B = gen.c4_cauchy_like(2, n=128, p=3)
    ref = oracle.structured_eliminate(x, y, G, B, "c2plu", 20)
    tr = rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B), "c2plu", 20)
    assert tr.row_indices == ref["row_indices"]
    assert tr.col_indices == ref["col_indices"]


def test_full_rank_drains(cuda_device):
    """SPEC: K = full rank on a 6x6 p=1 Cauchy -> final max u <= 1e-18 initial."""
    x, y, G, B = gen.c2_cauchy(3, n=6)
    tr = rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B), "rplu", 6,
                                 rng=rp.RngState(1))
    u = rp.exact_row_norms(tr.residual)
    assert u.max() <= 1e-18 * tr.bound_maxes[0]


@pytest.mark.slow
def test_c4_full_size_properties(cuda_device):
    """C4 at full size (2^20, p=4), 4 steps: eliminated rows drain to zero
    relative to the initial bound and the bound history is consistent."""
    x, y, G, B = gen.c4_cauchy_like(0)
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    tr = rp.structured_eliminate(M, "rplu", 4, rng=rp.RngState(0))
    u = rp.exact_row_norms(tr.residual)
    for i in tr.row_indices:
        assert u[i] <= 1e-20 * tr.bound_maxes[0]
    assert abs(u.sum() - tr.bound_sums[0]) > 0  # residual changed
