"""Parity of the B200 dense path (eliminate -> C-ABI -> K1/K2/K3) against the
reference goldens and the CPU oracle, on the same input bytes and the same
uniform stream.

Bars (north star): pivots identical (a mismatch is only acceptable when the
oracle marks the draw within 1e-12 relative of a CDF boundary); fp64 L/U to
1e-10 relative (observed: bit-identical); fp32 L/U to 1e-4 against the fp64
forced-pivot replay of the GPU's own pivots.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2601_22344_b200 as rp
from conftest import GOLDEN, check_dense_parity, load_golden, record_parity
from paper_2601_22344_b200 import gen

pytestmark = pytest.mark.gpu


def _cases():
    info, _ = load_golden("dense")
    return info["cases"]


def _rule(case):
    return rp.PivotRule(case["rule"], rp.RngState(case["seed"]) if case["seed"] is not None else None)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_dense_golden(case, cuda_device):
    _, arr = load_golden("dense")
    name = case["name"]
    A = arr[name + "_A"]
    rule = _rule(case)
    tr = rp.eliminate(A, rule, case["steps"], stop_tol=case["stop_tol"])
    assert [list(p) for p in tr.pivots] == case["pivots"]
    assert tr.steps == case["steps_done"]
    assert tr.clean_early_stop == case["clean_early_stop"]
    assert tr.tol_stop == case["tol_stop"]
    L, U = arr[name + "_L"], arr[name + "_U"]
    if A.dtype == np.float32:
        # float32 input is promoted to float64 as in the reference
        assert tr.L.dtype == np.float64
    np.testing.assert_array_equal(tr.L, L)      # bit-identical update arithmetic
    np.testing.assert_array_equal(tr.U, U)
    np.testing.assert_allclose(tr.resid_fro, arr[name + "_resid_fro"], rtol=1e-12,
                               atol=1e-300)
    if name + "_residual" in arr:
        np.testing.assert_array_equal(tr.residual, arr[name + "_residual"])
    if rule.rng is not None:
        assert rule.rng.uniform() == case["next_uniform"], "uniform stream not advanced exactly"


def test_sample_index_device(cuda_device):
    info, arr = load_golden("sample_index")
    for case in info["cases"]:
        w = arr[case["key"]]
        want = list(arr["idx" + case["key"][1:]])
        got = [rp.sample_index(w, u) for u in arr["us"]]
        assert got == want, case["key"]
    for bad in ([], [1.0, -2.0], [0.0, 0.0, 0.0]):
        with pytest.raises(ValueError):
            rp.sample_index(np.array(bad, dtype=float), 0.3)


def test_sample_index_boundaries(cuda_device):
    # u * total landing exactly on partial sums: side='right' semantics
    w = np.array([1.0, 2.0, 0.0, 1.0, 4.0])     # cdf 1 3 3 4 8
    for u, want in [(0.0, 0), (1 / 8, 1), (3 / 8, 3), (4 / 8, 4), (0.999, 4)]:
        assert rp.sample_index(w, u) == oracle.sample_index(w, u) == want
    big = np.random.default_rng(0).random(300_000)
    for u in (0.1, 0.5, 0.9):
        assert abs(rp.sample_index(big, u) - oracle.sample_index(big, u)) <= 1


def test_sample_index_chunked_large_n(cuda_device):
    """n >= 131072 uses the two-level (chunked) CDF: same semantics as the
    reference's sample_index (first running sum > u*total, clamp, zero
    walk-back), draws equal to the oracle's except within 1e-12 of a CDF
    boundary; zero runs across chunk boundaries, leading zero chunks and a
    zero tail exercise the walk-back and the clamp."""
    g = np.random.default_rng(3)
    n = 5 * 32768 + 123
    cases = []
    w = g.random(n)
    cases.append(w)
    w = g.random(n)
    w[: 2 * 32768 + 7] = 0.0                  # leading zero chunks
    cases.append(w)
    w = g.random(n)
    w[32768 - 50: 2 * 32768 + 50] = 0.0       # zero run across two chunk boundaries
    w[-1000:] = 0.0                           # zero tail (clamp + walk-back)
    cases.append(w)
    w = np.zeros(n)
    w[[5, 40000, 150000]] = [1.0, 2.0, 3.0]   # sparse
    cases.append(w)
    us = list(g.random(40)) + [0.0, 1.0 - 2 ** -53, 0.5]
    for w in cases:
        tot = float(np.sum(w))
        for u in us:
            got = rp.sample_index(w, u)
            want = oracle.sample_index(w, u)
            if got != want:
                c = np.cumsum(w)
                lo = c[min(got, want)]
                assert abs(lo - u * c[-1]) <= 1e-12 * tot, (u, got, want)
            assert w[got] > 0.0
    with pytest.raises(ValueError):
        bad = g.random(n)
        bad[100000] = -1.0
        rp.sample_index(bad, 0.3)
    with pytest.raises(ValueError):
        rp.sample_index(np.zeros(n), 0.3)


def test_sample_target_and_cdf_total(cuda_device):
    """The owner-shard draw against an absolute target and the per-shard CDF
    totals (rplu_sample_target / rplu_cdf_total) keep sample_index's
    semantics: first running sum > target, clamp, zero walk-back."""
    import torch

    from paper_2601_22344_b200.sharded_cur import CudaCurOps
    ops = CudaCurOps(torch.device("cuda"))
    w = torch.tensor([1.0, 2.0, 0.0, 1.0, 4.0, 0.0], dtype=torch.float64, device="cuda")
    assert ops.cdf_total(w) == 8.0
    for target, want in [(0.0, 0), (0.999, 0), (1.0, 1), (3.0, 3), (4.0, 4), (7.9, 4),
                         (8.0, 4), (9.0, 4)]:
        assert ops.sample_target(w, target) == want, target
    big = torch.from_numpy(np.random.default_rng(1).random(200_001)).cuda()
    tot = ops.cdf_total(big)
    assert abs(tot - float(big.sum())) <= 1e-9 * tot
    for u in (0.05, 0.5, 0.95):
        assert ops.sample_target(big, u * tot) == rp.sample_index(big, u)
    assert ops.cdf_total(torch.zeros(0, dtype=torch.float64, device="cuda")) == 0.0


def test_errors_and_validation(cuda_device):
    with pytest.raises(ValueError):
        rp.eliminate(np.eye(3), rp.PivotRule("rplu", rp.RngState(0)), 4)
    with pytest.raises(ValueError):
        rp.eliminate(np.eye(3), rp.PivotRule("rplu", rp.RngState(0)), 1, stop_tol=-1.0)
    tr = rp.eliminate(np.ones((3, 4)), "cplu", 0)
    assert tr.steps == 0 and tr.L.shape == (3, 0) and tr.U.shape == (0, 4)
    assert tr.resid_fro[0] == pytest.approx(np.sqrt(12.0))


def test_zero_residual_clean_stop(cuda_device):
    tr = rp.eliminate(np.zeros((4, 4)), rp.PivotRule("rplu", rp.RngState(0)), 3)
    assert tr.steps == 0 and tr.clean_early_stop


def test_c1_all_30_seeds_exact(cuda_device):
    """C1 2000^2, r=100, seeds 0..29 (BASELINE configs[0]):

    * the generated input bytes equal the ones the reference was run on
      (sha256 recorded by tests/golden/make_golden.py) -- a mismatch fails;
    * pivots identical to the reference's recorded pivots for every seed
      (a divergence is accepted only at a draw the oracle marks within 1e-12
      of a CDF boundary, and L/U are still checked up to that step);
    * L, U bit-identical to the C oracle on the same bytes, resid_fro to
      1e-12 relative of the reference's;
    * ||A-LU||_F/||A||_F equal to the reference's seed by seed (1e-8) and so
      are the 30-seed statistics.
    """
    from oracle import c_oracle
    runs = {r["seed"]: r for r in json.load(open(os.path.join(GOLDEN, "c1_reference.json")))["runs"]}
    errs, near, divergences = [], 0, {}
    for s in range(30):
        A = gen.c1_dense(s)
        assert hashlib.sha256(A.tobytes()).hexdigest() == runs[s]["sha256"], (
            f"seed {s}: C1 input bytes differ from the reference run's")
        ref = c_oracle.eliminate_c(A, "rplu", 100, seed=s, margins=True)
        tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(s)), 100)
        near += tr.near_boundary_draws
        t = check_dense_parity(tr, ref)
        want = [tuple(p) for p in runs[s]["pivots"]]
        tr_ref = next((q for q, (a, b) in enumerate(zip(tr.pivots, want)) if a != b), None)
        if tr_ref is not None:
            assert ref["margins"][tr_ref] <= oracle.NEAR_REL, (s, tr_ref)
            divergences[s] = tr_ref
        k = 100 if tr_ref is None else tr_ref
        np.testing.assert_allclose(tr.resid_fro[:k + 1], runs[s]["resid_fro"][:k + 1],
                                   rtol=1e-12)
        assert t == tr_ref
        err = float(np.linalg.norm(A - tr.L @ tr.U) / np.linalg.norm(A))
        errs.append(err)
        if tr_ref is None:
            assert abs(err - runs[s]["rel_err"]) <= 1e-8 * runs[s]["rel_err"], s
    errs = np.array(errs)
    ref_errs = np.array([runs[s]["rel_err"] for s in range(30)])
    record_parity("c1_all_30_seeds", divergences=divergences, near_boundary_draws=near,
                  mean=errs.mean(), min=errs.min(), max=errs.max(),
                  ref_mean=ref_errs.mean(), ref_min=ref_errs.min(), ref_max=ref_errs.max())
    assert abs(errs.mean() - ref_errs.mean()) <= 1e-8 * ref_errs.mean()


def test_fp32_against_forced_replay(cuda_device):
    """fp32 residual: L/U within 1e-4 of the fp64 forced-pivot replay of the
    GPU's own pivots (no fp32 reference exists)."""
    A = gen.c3_dense_host(0, n=1024, reflectors=16)
    tr = rp.eliminate(A.astype(np.float32), rp.PivotRule("rplu", rp.RngState(0)), 128,
                      compute_dtype=torch.float32)
    assert tr.L.dtype == np.float32
    rep = oracle.replay_pivots(A.astype(np.float32).astype(np.float64), tr.pivots)
    scale_l = np.abs(rep["L"]).max()
    scale_u = np.abs(rep["U"]).max()
    assert np.abs(tr.L - rep["L"]).max() <= 1e-4 * scale_l
    assert np.abs(tr.U - rep["U"]).max() <= 1e-4 * scale_u
    # and it reproduces a sensible error
    err = np.linalg.norm(A - tr.L.astype(np.float64) @ tr.U.astype(np.float64)) / np.linalg.norm(A)
    err64 = oracle.lu_error(A, rep["L"], rep["U"])
    assert abs(err - err64) <= 1e-3 * err64 + 1e-6


def test_c3_reduced_parity(cuda_device):
    """C3 construction at n=4096, r=128: pivots and factors vs the oracle."""
    A = gen.c3_dense_host(0, n=4096)
    ref = oracle.eliminate_real(A, "rplu", 128, seed=0, margins=True)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 128)
    check_dense_parity(tr, ref)


def test_complex_dense_parity(cuda_device):
    A = gen.planted_spectrum(300, 200, 0.9, 5)
    ref = oracle.eliminate_c128(A, "rplu", 80, seed=5, margins=True)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(5)), 80)
    check_dense_parity(tr, ref, exact=False, rtol=1e-12)


@pytest.mark.parametrize("rule", ["c2plu", "cplu"])
def test_greedy_rules_parity(rule, cuda_device):
    A = gen.c1_dense(3, n=500, m=433)
    ref = oracle.eliminate_real(A, rule, 60)
    tr = rp.eliminate(A, rule, 60)
    assert tr.pivots == ref["pivots"]
    np.testing.assert_array_equal(tr.L, ref["L"])


def test_ragged_shapes_and_stride(cuda_device):
    # odd m (scalar tail path), n < block rows, tall and wide
    for n, m in [(1, 7), (3, 1), (5, 3), (257, 129), (130, 1025)]:
        A = np.random.default_rng(n * 1000 + m).standard_normal((n, m))
        k = min(n, m)
        ref = oracle.eliminate_real(A, "rplu", k, seed=n + m)
        tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(n + m)), k)
        assert tr.pivots == ref["pivots"], (n, m)
        np.testing.assert_array_equal(tr.U, ref["U"])


@pytest.mark.parametrize("shape,dtype", [((1449, 1450), np.float64), ((3001, 2999), np.float32),
                                         ((1100, 1001), np.complex128), ((20_000_003,), np.float64)])
def test_pageable_upload_ring(shape, dtype, cuda_device, monkeypatch):
    """rplu_upload (worker pool, streaming stores, pinned ring): pageable
    arrays above the direct-copy threshold arrive bit for bit, for sizes that
    do not divide into the 64-byte granules / pieces, unaligned sources and
    every staging thread count."""
    from paper_2601_22344_b200 import _device
    rs = np.random.default_rng(5)
    n = int(np.prod(shape))
    raw = rs.standard_normal(2 * n + 3)
    a = (raw[:n] + 1j * raw[n:2 * n]).astype(dtype) if np.issubdtype(dtype, np.complexfloating) \
        else raw[:n].astype(dtype)
    a = a.reshape(shape)
    assert a.nbytes >= 16 << 20
    dev = torch.device("cuda", 0)
    for threads in ("1", "3", "8", "16"):
        monkeypatch.setenv("RPLU_UPLOAD_THREADS", threads)
        t = _device.upload(a, dev)
        torch.cuda.synchronize()
        assert torch.equal(t.cpu(), torch.from_numpy(a))
    # a source that is not 16-byte aligned (a view one element into a buffer)
    buf = np.empty(n + 1, dtype=dtype)
    v = buf[1:]
    v[:] = a.reshape(-1)
    t = _device.upload(v, dev)
    torch.cuda.synchronize()
    assert torch.equal(t.cpu(), torch.from_numpy(v))


def test_device_tensor_inputs_stay_on_device(cuda_device):
    A = torch.from_numpy(gen.c1_dense(0, n=256)).cuda()
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 32)
    assert isinstance(tr.L, torch.Tensor) and tr.L.is_cuda
    # identity A = L U + residual
    resid = tr.residual
    err = torch.linalg.norm(A - tr.L @ tr.U - resid) / torch.linalg.norm(A)
    assert float(err) <= 1e-13


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.complex128])
@pytest.mark.parametrize("n,m,steps", [(700, 530, 97), (257, 1024, 40)])
def test_lazy_update_is_bit_identical(dtype, n, m, steps, cuda_device):
    """Delayed updates (R read per step, written every few steps) reproduce
    the eager path's residual, L, U and pivots bit for bit."""
    rs = np.random.default_rng(n + m)
    A = rs.standard_normal((n, m)) @ np.diag(0.97 ** np.arange(m))
    if dtype == torch.complex128:
        A = A + 1j * rs.standard_normal((n, m)) @ np.diag(0.97 ** np.arange(m))
    At = torch.from_numpy(A).to("cuda", dtype)
    e = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(3)), steps, update="eager")
    z = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(3)), steps, update="lazy",
                     time_kernels=True, fused_updates=False)
    assert z.kernel_stats["lazy_block"] > 0 and e.kernel_stats["lazy_block"] == 0
    assert z.pivots == e.pivots
    assert torch.equal(z.L, e.L) and torch.equal(z.U, e.U)
    assert torch.equal(z.residual, e.residual)
    # masses are summed in a different order by the two passes
    np.testing.assert_allclose(z.resid_fro, e.resid_fro, rtol=1e-13)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.complex128])
@pytest.mark.parametrize("block", [1, 2, 7, 11, 16])
def test_lazy_every_flush_interval_is_bit_identical(dtype, block, cuda_device, monkeypatch):
    """Every pending-term count q = 1..16 of the TMA-fed pass (one kernel
    instantiation per q) against the eager loop, on a ragged shape (row
    count not a multiple of the 32-row block, odd column count: scalar tail,
    partial last column chunk); fp64 runs the Gram-mass loop (its flushes
    are the q = block instantiations) and the applied-term loop."""
    monkeypatch.setenv("RPLU_LAZY_BLOCK", str(block))
    monkeypatch.setenv("RPLU_LAZY_BLOCK_GRAM", str(block))
    n, m, steps = 1001, 1153, 70
    rs = np.random.default_rng(block)
    A = rs.standard_normal((n, m)) @ np.diag(0.98 ** np.arange(m))
    if dtype == torch.complex128:
        A = A + 1j * rs.standard_normal((n, m)) @ np.diag(0.98 ** np.arange(m))
    At = torch.from_numpy(A).to("cuda", dtype)
    e = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(5)), steps, update="eager")
    for gram in ((True, False) if dtype == torch.float64 else (True,)):
        z = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(5)), steps, update="lazy",
                         time_kernels=True, gram_masses=gram)
        assert z.kernel_stats["lazy_block"] == block
        assert z.pivots == e.pivots
        assert torch.equal(z.L, e.L) and torch.equal(z.U, e.U)
        assert torch.equal(z.residual, e.residual)
        np.testing.assert_allclose(z.resid_fro, e.resid_fro, rtol=1e-13)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.complex128])
@pytest.mark.parametrize("block", [1, 3, 8, 12, 16])
def test_lazy_fused_every_flush_interval(dtype, block, cuda_device, monkeypatch):
    """The optional fused delayed-update arithmetic (one FMA per pending
    term) for every instantiated pending-term count: pivots equal to the eager loop's
    (reference rounding), L / U / residual to 1e-12 of their scale (fp64,
    complex128) or 1e-5 (fp32)."""
    monkeypatch.setenv("RPLU_LAZY_BLOCK_FUSED", str(block))
    n, m, steps = 1001, 1153, 70
    rs = np.random.default_rng(block + 100)
    A = rs.standard_normal((n, m)) @ np.diag(0.98 ** np.arange(m))
    if dtype == torch.complex128:
        A = A + 1j * rs.standard_normal((n, m)) @ np.diag(0.98 ** np.arange(m))
    At = torch.from_numpy(A).to("cuda", dtype)
    e = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(6)), steps, update="eager")
    z = rp.eliminate(At, rp.PivotRule("rplu", rp.RngState(6)), steps, update="lazy",
                     time_kernels=True, fused_updates=True)
    assert z.kernel_stats["lazy_block"] == block
    assert z.pivots == e.pivots
    tol = 1e-5 if dtype == torch.float32 else 1e-12
    for a, b in ((z.L, e.L), (z.U, e.U), (z.residual, e.residual)):
        assert float((a - b).abs().max()) <= tol * float(b.abs().max())
    np.testing.assert_allclose(z.resid_fro, e.resid_fro, rtol=1e-10 if tol < 1e-6 else 1e-4)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.complex128])
@pytest.mark.parametrize("rule", ["rplu", "c2plu"])
@pytest.mark.parametrize("n,m,steps", [(2000, 2000, 100), (1001, 1153, 80), (37, 1500, 30),
                                       (1500, 41, 41)])
def test_persistent_loop_matches_stepwise(dtype, rule, n, m, steps, cuda_device):
    """The one-launch persistent loop (L2-resident residuals) against the
    per-step K2/K3 launches: same pivots, bit-identical L, U and residual."""
    rs = np.random.default_rng(n * 7 + m)
    A = rs.standard_normal((n, m)) @ np.diag(0.99 ** np.arange(m))
    if dtype == torch.complex128:
        A = A + 1j * rs.standard_normal((n, m))
    At = torch.from_numpy(A).to("cuda", dtype)

    def mk():
        return rp.PivotRule("rplu", rp.RngState(9)) if rule == "rplu" else "c2plu"

    s = rp.eliminate(At, mk(), steps, persistent=False)
    z = rp.eliminate(At, mk(), steps, time_kernels=True)
    vec = {torch.float64: 2, torch.float32: 4, torch.complex128: 1}[dtype]
    if m <= 1024 * vec and n * m * At.element_size() <= 30e6:  # fits the SMs' shared memory
        assert z.kernel_stats["kernel_launches"] <= 3  # init + one loop launch
    assert z.pivots == s.pivots and z.steps == s.steps
    assert torch.equal(z.L, s.L) and torch.equal(z.U, s.U)
    assert torch.equal(z.residual, s.residual)
    np.testing.assert_allclose(z.resid_fro, s.resid_fro, rtol=1e-13)
    assert z.uniforms_consumed == s.uniforms_consumed


def test_persistent_loop_stops(cuda_device):
    A = torch.from_numpy(gen.c1_dense(2, n=600, m=512)).cuda()
    for tol in (0.3, 0.05):
        e = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(2)), 300, stop_tol=tol,
                         persistent=False)
        z = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(2)), 300, stop_tol=tol)
        assert e.tol_stop and z.tol_stop and z.steps == e.steps and z.pivots == e.pivots
        assert torch.equal(z.residual, e.residual)
    B = torch.from_numpy(np.diag(np.arange(1.0, 31.0))).cuda()
    z = rp.eliminate(B, rp.PivotRule("rplu", rp.RngState(0)), 30)
    e = rp.eliminate(B, rp.PivotRule("rplu", rp.RngState(0)), 30, persistent=False)
    assert z.pivots == e.pivots and z.clean_early_stop == e.clean_early_stop


@pytest.mark.parametrize("rule", ["rplu", "c2plu"])
def test_lazy_early_stops_flush_the_residual(rule, cuda_device):
    A = torch.from_numpy(gen.c1_dense(2, n=600, m=512)).cuda()
    mk = (lambda: rp.PivotRule("rplu", rp.RngState(2))) if rule == "rplu" else (lambda: "c2plu")
    e = rp.eliminate(A, mk(), 300, stop_tol=0.3, update="eager")
    z = rp.eliminate(A, mk(), 300, stop_tol=0.3, update="lazy", fused_updates=False)
    assert e.tol_stop and z.tol_stop and z.steps == e.steps
    assert torch.equal(z.residual, e.residual) and torch.equal(z.L, e.L)
    f = rp.eliminate(A, mk(), 300, stop_tol=0.3, update="lazy", fused_updates=True)
    assert f.tol_stop and f.steps == e.steps and f.pivots == e.pivots
    assert float((f.residual - e.residual).abs().max()) <= 1e-12 * float(A.abs().max())
    # clean stop on an exactly low-rank matrix
    B = torch.from_numpy(np.diag(np.arange(1.0, 31.0))).cuda()
    e = rp.eliminate(B, rp.PivotRule("rplu", rp.RngState(0)), 30, update="eager")
    z = rp.eliminate(B, rp.PivotRule("rplu", rp.RngState(0)), 30, update="lazy",
                     fused_updates=False)
    assert z.pivots == e.pivots and torch.equal(z.residual, e.residual)


def test_lazy_matches_oracle_c3_reduced(cuda_device):
    A = gen.c3_dense_host(1, n=4096)
    ref = oracle.eliminate_real(A, "rplu", 128, seed=1, margins=True)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(1)), 128, update="lazy",
                      fused_updates=False)
    check_dense_parity(tr, ref)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(1)), 128, update="lazy",
                      fused_updates=True)
    check_dense_parity(tr, ref, exact=False, rtol=1e-12)


@pytest.mark.slow
def test_c3_full_size_properties(cuda_device):
    """Full C3 (32768^2 fp64, r=512): size-independent identities.

    A = L U + R to 1e-10 relative; L[i_t, t] == R_t[i_t,j_t]*(1/a) (~1);
    pivots distinct rows/cols; resid_fro[k] == ||R||_F; non-increasing-ish
    (the RPLU residual is not monotone in general, so only the final value is
    compared with torch's norm).
    """
    A = gen.c3_dense_device(0, n=32768)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512)
    R = tr.residual
    rel = torch.linalg.norm(A - tr.L @ tr.U - R) / torch.linalg.norm(A)
    assert float(rel) <= 1e-10
    rows = [p[0] for p in tr.pivots]
    cols = [p[1] for p in tr.pivots]
    assert len(set(rows)) == 512 and len(set(cols)) == 512
    assert abs(float(torch.linalg.norm(R)) - tr.resid_fro[-1]) <= 1e-10 * tr.resid_fro[0]
    Li = tr.L[torch.tensor(rows, device=A.device), torch.arange(512, device=A.device)]
    assert float((Li - 1).abs().max()) <= 1e-12


def test_error_evaluation_matches_reference_measures(cuda_device):
    """§8(f2): device ||A-LU||_F/||A||_F, power-iteration spectral error and
    optimal SVD errors agree with the host computations."""
    from paper_2601_22344_b200 import errors
    A = gen.c1_dense(1, n=400, m=300)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(1)), 40)
    fro = errors.lu_error(A, tr.L, tr.U)
    assert abs(fro - oracle.lu_error(A, tr.L, tr.U)) <= 1e-12 * fro
    # power iteration restated on the host (cli.py:86-99)
    R = A - tr.L @ tr.U
    g = rp.RngState(77)
    v = g.complex_normal(300)
    v /= np.linalg.norm(v)
    est = 0.0
    for _ in range(20):
        w = R.conj().T @ (R @ v)
        est = float(np.linalg.norm(w))
        v = w / est
    spec = errors.residual_spectral(A, tr.L, tr.U, seed=77)
    assert abs(spec - np.sqrt(est)) <= 1e-10 * spec
    s = np.linalg.svd(A, compute_uv=False)
    f, sp = errors.truncated_svd_error(A, 40)
    assert abs(f - np.sqrt((s[40:] ** 2).sum())) <= 1e-10 * f and abs(sp - s[40]) <= 1e-10 * sp


@pytest.mark.parametrize("n,m,k,dtype", [(1000, 777, 37, np.float64), (129, 1031, 16, np.float64),
                                         (700, 500, 60, np.complex128), (513, 257, 8, np.float32),
                                         (300, 200, 0, np.float64), (1, 5, 1, np.float64)])
def test_k11_lu_error_kernel(n, m, k, dtype, cuda_device):
    """K11 (rplu_lu_error, DMMA tensor cores, fused subtract + Frobenius) on
    ragged shapes, complex, fp32 and k = 0 against numpy: ||A - L U||_F to
    1e-12 relative, ||A||_F to 1e-13."""
    from paper_2601_22344_b200 import errors
    rs = np.random.default_rng(n + m + k)
    A = rs.standard_normal((n, m))
    L = rs.standard_normal((n, k))
    U = rs.standard_normal((k, m))
    if dtype == np.complex128:
        A = A + 1j * rs.standard_normal((n, m))
        L = L + 1j * rs.standard_normal((n, k))
        U = U + 1j * rs.standard_normal((k, m))
    A, L, U = A.astype(dtype), L.astype(dtype), U.astype(dtype)
    e, a, ms = errors.lu_error_sq(A, L, U)
    A64, L64, U64 = (x.astype(np.complex128 if dtype == np.complex128 else np.float64)
                     for x in (A, L, U))
    want_e = np.linalg.norm(A64 - L64 @ U64) ** 2
    want_a = np.linalg.norm(A64) ** 2
    assert abs(e - want_e) <= 1e-12 * want_e
    assert abs(a - want_a) <= 1e-13 * want_a
    assert ms > 0


def test_k11_on_elimination_factors(cuda_device):
    """K11 on the factors of a real elimination (L from Lt, no transpose
    copy) at 8192^2, r = 512: equal to the oracle's host computation."""
    from paper_2601_22344_b200 import errors
    A = gen.c3_dense_device(0, n=8192)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512)
    e, a, ms = errors.lu_error_sq(A, tr.L, tr.U)
    Ah, Lh, Uh = A.cpu().numpy(), tr.L.cpu().numpy(), tr.U.cpu().numpy()
    want = oracle.lu_error(Ah, Lh, Uh)
    assert abs(np.sqrt(e / a) - want) <= 1e-11 * want
    # the eliminate identity: ||A - LU|| = ||R_k|| = resid_fro[k]
    assert abs(np.sqrt(e) - tr.resid_fro[-1]) <= 1e-9 * tr.resid_fro[-1]
    record_parity("k11_8192", tflops=2.0 * 8192 * 8192 * 512 / (ms * 1e-3) / 1e12, ms=ms)
