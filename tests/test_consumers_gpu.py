"""§8(f4) downstream consumers on the device against the reference's goldens
(tests/golden/rational.*, precond.*) and the pinned oracle.

Bars:
* Loewner generators bit-identical to the reference's;
* AAA / CUR-AAA: support indices (and CUR-AAA's side and the caller's
  uniform stream) identical; AAA error histories to 1e-4 relative or
  1e-12 max|f| (the final rounds are at rounding level); the fitted rational on off-sample points within
  1e-9 of max|f|; CUR-AAA weights equal up to one unit-modulus phase
  (1e-6); inputs whose reference result is itself unstable under 1e-15
  perturbations (rejection-test ties) get a fit-quality bar instead;
* barycentric evaluation: values to 1e-13 relative, pole / hit flags equal;
* SMW apply to 1e-10 relative; GMRES iteration counts and flags identical,
  residual histories to 1e-5 relative (entries down to 1e-13), solutions
  to 1e-8;
* the MGS Arnoldi kernel against numpy MGS to 1e-12.
"""

import warnings

import numpy as np
import pytest
import torch

import oracle
import paper_2601_22344_b200 as rp
from conftest import load_golden
from consumer_cases import band_system
from paper_2601_22344_b200 import gen

pytestmark = pytest.mark.gpu

NAMES = ["tanh_line", "circle_log", "spiral_mero"]


def _case(name):
    info, arr = load_golden("rational")
    return next(c for c in info["cases"] if c["name"] == name), arr


def _phase_close(w, ref, tol):
    ph = np.vdot(w, ref)
    ph = ph / abs(ph)
    np.testing.assert_allclose(w * ph, ref, rtol=0, atol=tol)


@pytest.mark.parametrize("name", NAMES)
def test_loewner_build_matches_reference(name, cuda_device):
    case, arr = _case(name)
    z, f = arr[name + "_z"], arr[name + "_f"]
    perm = rp.RngState(case["seed"]).permutation(z.size)
    h = (z.size + 1) // 2
    L = rp.loewner_build(z[perm[:h]], f[perm[:h]], z[perm[h:]], f[perm[h:]])
    np.testing.assert_array_equal(L.G.cpu().numpy(), arr[name + "_loewner_G"])
    np.testing.assert_array_equal(L.B.cpu().numpy(), arr[name + "_loewner_B"])


@pytest.mark.parametrize("name", NAMES)
def test_aaa_matches_reference(name, cuda_device):
    case, arr = _case(name)
    z, f = arr[name + "_z"], arr[name + "_f"]
    r, errs = rp.aaa(rp.SampleSet(z, f), tol=1e-13, max_degree=60)
    idx = [int(np.nonzero(z == t)[0][0]) for t in r.support]
    assert idx == case["aaa_support_idx"]
    fs = np.abs(f).max()
    # the last rounds sit at rounding level: absolute 1e-12 max|f| there
    np.testing.assert_allclose(errs, arr[name + "_aaa_errors"], rtol=1e-4, atol=1e-12 * fs)
    np.testing.assert_allclose(r(arr[name + "_zt"]), arr[name + "_aaa_eval"], rtol=0,
                               atol=1e-9 * fs)
    # no weight check: at AAA convergence sigma_min / sigma_{k-1} ~ 1e-2 with
    # sigma ~ 1e-12, so a 1e-16 perturbation of L moves the weights by ~1e-4
    # (the reference's own weights included); the rational is what is pinned


@pytest.mark.parametrize("tag", ["_cur", "_cur8"])
@pytest.mark.parametrize("name", NAMES)
def test_cur_aaa_matches_reference(name, tag, cuda_device):
    case, arr = _case(name)
    cc = case["cur"][tag]
    z, f = arr[name + "_z"], arr[name + "_f"]
    rng = rp.RngState(case["seed"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r, side = rp.cur_aaa(rp.SampleSet(z, f), tol=case["tol"], rng=rng,
                             leaf_size=cc["leaf_size"])
    assert rng.uniform() == cc["next_uniform"]     # one permutation drawn, as the reference
    fs = np.abs(f).max()
    err = float(np.max(np.abs(r(z) - f)))
    ref_err = float(arr[name + tag + "_err"][0])
    if not cc["stable"]:
        # the reference's own pivots move under 1e-15 perturbations (rejection
        # test ties, see make_golden._cur_aaa_stable): fit-quality bar only
        assert err <= max(10.0 * ref_err, 10.0 * case["tol"] * fs)
        assert abs(r.degree - cc["degree"]) <= 1
        return
    assert side == cc["side"]
    idx = [int(np.nonzero(z == t)[0][0]) for t in r.support]
    assert idx == cc["support_idx"]
    np.testing.assert_allclose(r(arr[name + "_zt"]), arr[name + tag + "_eval"], rtol=0,
                               atol=1e-9 * fs)
    _phase_close(r.weights, arr[name + tag + "_weights"], 1e-6)
    assert err <= max(2.0 * ref_err, 1e-12 * fs)


def test_bary_eval_edge_cases(cuda_device):
    _, arr = load_golden("rational")
    r = rp.BarycentricRational(arr["bary_t"], arr["bary_f"], arr["bary_w"])
    out, flags = r.eval_flagged(arr["bary_z"])
    ref = arr["bary_out"]
    fin = np.isfinite(ref)
    np.testing.assert_allclose(out[fin], ref[fin], rtol=1e-13)
    np.testing.assert_array_equal(flags, arr["bary_flags"])
    v, fl = r.eval_flagged(arr["bary_t"][1])          # scalar input -> (complex, bool)
    assert v == complex(arr["bary_f"][1]) and fl is False
    # device input stays on the device
    zt = torch.from_numpy(arr["bary_z"]).cuda()
    dv = r(zt)
    assert isinstance(dv, torch.Tensor) and dv.is_cuda


def test_bary_eval_large_matches_oracle(cuda_device):
    g = np.random.default_rng(7)
    k = 700                                        # > one shared-memory tile (512)
    t = g.standard_normal(k) + 1j * g.standard_normal(k)
    f = np.exp(t)
    w = g.standard_normal(k) + 1j * g.standard_normal(k)
    z = 3 * (g.standard_normal(5000) + 1j * g.standard_normal(5000))
    z[:3] = t[[5, 600, 699]]                       # exact hits across tiles
    r = rp.BarycentricRational(t, f, w)
    got, gflags = r.eval_flagged(z)
    want, wflags = oracle.consumers.bary_eval_flagged(t, f, w, z)
    np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12 * np.abs(want).max())
    np.testing.assert_array_equal(gflags, wflags)


def test_rational_errors(cuda_device):
    with pytest.raises(ValueError):
        rp.BarycentricRational([1.0, 1.0], [1.0, 2.0], [1.0, 1.0])
    with pytest.raises(ValueError):
        rp.BarycentricRational([1.0, 2.0], [1.0, 2.0], [0.0, 0.0])
    with pytest.raises(ValueError):
        rp.BarycentricRational([], [], [])
    S = rp.SampleSet(np.arange(6) + 0j, np.arange(6) + 0j)
    with pytest.raises(ValueError):
        rp.cur_aaa(S, rng=None)
    with pytest.raises(ValueError):
        rp.cur_aaa(rp.SampleSet([0j, 1, 2], [0j, 1, 2]), rng=rp.RngState(0))
    with pytest.raises(ValueError):
        rp.aaa(S, tol=0.0)
    with pytest.raises(ValueError):
        rp.SampleSet([0j, 0j], [1.0, 2.0])
    # constant samples: cur_aaa falls back to greedy AAA with a warning
    with pytest.warns(UserWarning):
        r, side = rp.cur_aaa(rp.SampleSet(np.arange(8) + 0j, np.ones(8)), rng=rp.RngState(1))
    assert side == "fallback"


# ---------------------------------------------------------------------------
# SMW + GMRES

def _precond(idx):
    info, arr = load_golden("precond")
    case = info["cases"][idx]
    return case, arr, band_system(case["n"], case["seed"])


@pytest.mark.parametrize("idx", [0, 1])
def test_smw_and_gmres_match_reference(idx, cuda_device):
    case, arr, (A, _, b_inv, K_apply, K) = _precond(idx)
    name = case["name"]
    fact, _ = rp.cur_build(rp.DenseMatrix(A), "rplu-cur", case["k"],
                           rng=rp.RngState(case["seed"] ^ 1))
    assert list(fact.row_indices) == case["I"] and list(fact.col_indices) == case["J"]
    pre = rp.smw_build(b_inv, rp.DenseMatrix(A), fact)
    pv = pre.apply(arr[name + "_v"])
    np.testing.assert_allclose(pv, arr[name + "_pre_v"], rtol=1e-10,
                               atol=1e-12 * np.abs(pv).max())
    b = arr[name + "_b"]
    res = rp.gmres(K_apply, b, M_inv=pre, restart=20, tol=1e-10, max_restarts=200)
    assert (res.iterations, res.converged, res.stagnated) == (
        case["pre"]["iterations"], case["pre"]["converged"], case["pre"]["stagnated"])
    np.testing.assert_allclose(res.residuals, arr[name + "_hist_pre"], rtol=1e-5)
    np.testing.assert_allclose(res.x, arr[name + "_x_pre"], rtol=1e-8, atol=1e-10)
    # unpreconditioned with restarts; the operator as a device matrix
    res = rp.gmres(torch.from_numpy(K).cuda(), b, restart=10, tol=1e-8, max_restarts=300)
    assert (res.iterations, res.converged) == (case["plain"]["iterations"],
                                               case["plain"]["converged"])
    np.testing.assert_allclose(res.residuals, arr[name + "_hist_plain"], rtol=1e-6)
    np.testing.assert_allclose(res.x, arr[name + "_x_plain"], rtol=1e-7, atol=1e-9)


def test_gmres_device_callables_and_tensor_rhs(cuda_device):
    case, arr, (A, ab, b_inv, K_apply, K) = _precond(1)
    Kd = torch.from_numpy(K).to("cuda", torch.complex128)
    k_dev = rp.device_callable(lambda v: Kd @ v)
    b = torch.from_numpy(arr[case["name"] + "_b"]).cuda()
    res = rp.gmres(k_dev, b, restart=10, tol=1e-8, max_restarts=300)
    assert isinstance(res.x, torch.Tensor) and res.x.is_cuda
    np.testing.assert_allclose(res.x.cpu().numpy(), arr[case["name"] + "_x_plain"], rtol=1e-7,
                               atol=1e-9)
    assert res.iterations == case["plain"]["iterations"]


def test_mgs_arnoldi_kernel_matches_numpy(cuda_device):
    import ctypes
    from paper_2601_22344_b200 import _device, _ffi
    g = np.random.default_rng(3)
    n, j = 100_003, 6
    Q = np.linalg.qr(g.standard_normal((n, j + 1)) + 1j * g.standard_normal((n, j + 1)))[0]
    w0 = g.standard_normal(n) + 1j * g.standard_normal(n)
    V = torch.zeros((j + 2, n), dtype=torch.complex128, device="cuda")
    V[:j + 1] = torch.from_numpy(Q.T.copy()).cuda()
    w = torch.from_numpy(w0).cuda()
    h = torch.zeros(j + 2, dtype=torch.complex128, device="cuda")
    c = _device.ctx(torch.device("cuda", 0))
    _ffi.check(c._lib.rplu_mgs_arnoldi(c.handle, V.data_ptr(), n, j, w.data_ptr(),
                                       V[j + 1].data_ptr(), h.data_ptr(),
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    ww = w0.copy()
    hr = np.zeros(j + 2, np.complex128)
    for t in range(j + 1):
        hr[t] = np.vdot(Q[:, t], ww)
        ww = ww - hr[t] * Q[:, t]
    hr[j + 1] = np.linalg.norm(ww)
    np.testing.assert_allclose(h.cpu().numpy(), hr, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(w.cpu().numpy(), ww, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(V[j + 1].cpu().numpy(), ww / hr[j + 1].real, rtol=1e-12,
                               atol=1e-14)


def test_smw_gaussian_operator_matches_dense(cuda_device):
    P, Q = gen.c5_points(2, n=3000, m=3000)
    op = rp.GaussianKernelOperator(P, Q)
    dense = rp.DenseMatrix(op.materialize())
    fact, _ = rp.cur_build(op, "rplu-cur", 12, rng=rp.RngState(5))
    shift = 2.0
    b_inv = rp.device_callable(lambda v: v / shift)
    pre_g = rp.smw_build(b_inv, op, fact)
    pre_d = rp.smw_build(b_inv, dense, fact)
    v = torch.from_numpy(rp.RngState(9).complex_normal(3000)).cuda()
    a, b = pre_g.apply(v), pre_d.apply(v)
    torch.testing.assert_close(a, b, rtol=1e-10, atol=1e-12 * float(b.abs().max()))
    # GMRES on (shift I + A) with the SMW preconditioner converges fast
    K = rp.device_callable(lambda x: shift * x + torch.complex(
        op.apply_dev(x.real.contiguous()), op.apply_dev(x.imag.contiguous())))
    res = rp.gmres(K, v, M_inv=pre_g, restart=20, tol=1e-10)
    assert res.converged
    plain = rp.gmres(K, v, restart=20, tol=1e-10)
    assert res.iterations <= plain.iterations


def test_precond_errors(cuda_device):
    A = gen.planted_spectrum(20, 30, 0.5, 1)
    fact, _ = rp.cur_build(rp.DenseMatrix(A), "rplu-cur", 3, rng=rp.RngState(0))
    with pytest.raises(ValueError):
        rp.smw_build(lambda v: v, rp.DenseMatrix(A), fact)
    with pytest.raises(ValueError):
        rp.gmres(np.eye(3), np.ones(3), restart=0)
    r = rp.gmres(np.eye(3), np.zeros(3))
    assert r.converged and r.iterations == 0
    # singular inner matrix W + A[I,:] B^{-1} A[:,J] = 1 - 1 raises LinAlgError
    A2 = np.zeros((6, 6))
    A2[0, 0] = 1.0
    fact2, _ = rp.cur_build(rp.DenseMatrix(A2), "rplu-cur", 1, rng=rp.RngState(0))
    with pytest.raises(np.linalg.LinAlgError):
        rp.smw_build(lambda v: -v, rp.DenseMatrix(A2), fact2)


def test_gmres_x0_and_restart_edge_cases(cuda_device):
    """x0 start, restart = 1, and a singular system that stagnates, each
    against the pinned oracle's MGS-GMRES."""
    g = np.random.default_rng(11)
    n = 120
    K = np.eye(n) * 3 + g.standard_normal((n, n)) * 0.05
    b = g.standard_normal(n) + 1j * g.standard_normal(n)
    x0 = g.standard_normal(n) + 0j
    res = rp.gmres(K, b, restart=7, tol=1e-11, x0=x0)
    Kf = lambda v: K @ v  # noqa: E731
    assert res.converged
    np.testing.assert_allclose(K @ res.x, b, rtol=0, atol=1e-9 * np.linalg.norm(b))
    r1 = rp.gmres(Kf, b, restart=1, tol=1e-8, max_restarts=500)
    o1 = oracle.consumers.gmres_mgs(Kf, b, restart=1, tol=1e-8, max_restarts=500)
    assert (r1.iterations, r1.converged) == (o1[2], o1[3])
    np.testing.assert_allclose(r1.residuals, o1[1], rtol=1e-6)
    S = np.diag(np.r_[np.ones(n - 1), 0.0])          # singular: b has a null-space part
    with pytest.warns(UserWarning):
        rs = rp.gmres(S, np.ones(n), restart=5, tol=1e-12, max_restarts=20)
    assert rs.stagnated and not rs.converged


class _RefDense:
    """Stand-in with the reference rplu.DenseMatrix's surface
    (accessors.py:93-131: complex128 ``.array``, host apply/adjoint_apply);
    /root/reference is not on the GPU box, so the tests use a duck type."""

    def __init__(self, a):
        self.array = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
        self.shape = self.array.shape

    def apply(self, v):
        return self.array @ v

    def adjoint_apply(self, v):
        return self.array.conj().T @ v


class _RefCallable:
    """Stand-in for rplu.CallableOperator (host callables only)."""

    def __init__(self, K):
        self.K = K
        self.shape = K.shape

    def apply(self, v):
        return self.K @ v


def test_reference_objects_cross_the_boundary(cuda_device):
    """the reference's DenseMatrix (``.array``) and host
    accessors are accepted by eliminate / smw_build / gmres, and accessor
    inputs get numpy results as in the reference (cli.py:150-157)."""
    A = gen.c1_dense(4, n=300, m=240)
    want = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(4)), 30)
    got = rp.eliminate(_RefDense(A), rp.PivotRule("rplu", rp.RngState(4)), 30)
    assert isinstance(got.L, np.ndarray) and isinstance(got.U, np.ndarray)
    assert got.pivots == want.pivots
    np.testing.assert_array_equal(got.L, want.L)
    np.testing.assert_array_equal(got.U, want.U)
    assert isinstance(got.residual, np.ndarray)
    # this package's DenseMatrix: numpy results, the accessor's buffer untouched
    D = rp.DenseMatrix(A)
    before = D.tensor.clone()
    mine = rp.eliminate(D, rp.PivotRule("rplu", rp.RngState(4)), 30)
    assert isinstance(mine.L, np.ndarray) and mine.pivots == want.pivots
    np.testing.assert_array_equal(mine.U, want.U)
    assert torch.equal(D.tensor, before)
    # smw_build / gmres with the reference types
    case, arr, (Ab, _, b_inv, K_apply, K) = _precond(0)
    fact, _ = rp.cur_build(rp.DenseMatrix(Ab), "rplu-cur", case["k"],
                           rng=rp.RngState(case["seed"] ^ 1))
    ref_fact, _ = rp.cur_build(_RefDense(Ab), "rplu-cur", case["k"],
                               rng=rp.RngState(case["seed"] ^ 1))
    assert list(ref_fact.row_indices) == list(fact.row_indices)
    pre = rp.smw_build(b_inv, _RefDense(Ab), fact)
    pv = pre.apply(arr[case["name"] + "_v"])
    np.testing.assert_allclose(pv, arr[case["name"] + "_pre_v"], rtol=1e-10,
                               atol=1e-12 * np.abs(pv).max())
    b = arr[case["name"] + "_b"]
    res = rp.gmres(_RefCallable(K), b, M_inv=pre, restart=20, tol=1e-10, max_restarts=200)
    assert res.iterations == case["pre"]["iterations"] and res.converged
    res2 = rp.gmres(_RefDense(K), b, restart=10, tol=1e-8, max_restarts=300)
    assert res2.iterations == case["plain"]["iterations"]
