"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py [--c1]

It imports ``rplu`` from /root/reference/pkg/src, runs its public entry
points (eliminate, structured_eliminate, cur_build, sample_index) on seeded
desk-size inputs and writes the inputs and outputs as small fixtures next to
this script.  The fixtures pin the oracle (tests/test_oracle_golden.py) and
the GPU path (tests/test_*_gpu.py).  ``--c1`` also records the reference's
C1 run (2000 x 2000, r = 100, seeds 0..29): pivots, residual norms and
||A - LU||_F / ||A||_F, plus a hash of the input bytes (the 32 MB inputs are
regenerated from the seed, not committed).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import rplu  # noqa: E402  (the reference)
import scipy  # noqa: E402

from paper_2601_22344_b200 import gen  # noqa: E402  (input constructors only)


def meta():
    return {"numpy": np.__version__, "scipy": scipy.__version__, "rplu": rplu.__version__}


def _compact(a):
    a = np.asarray(a)
    if np.iscomplexobj(a) and not np.any(a.imag):
        return np.ascontiguousarray(a.real)  # reference complex128 with zero imaginary part
    return a


def save(name, arrays, info):
    arrays = {k: _compact(v) for k, v in arrays.items()}
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump({"meta": meta(), "cases": info}, f, indent=1)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_index_cases():
    arrays, info = {}, []
    rs = np.random.default_rng(5)
    vecs = [
        np.array([1.0]),
        np.array([0.0, 1.0, 0.0, 2.0, 0.0]),
        np.array([3.0, 0.0, 0.0]),
        np.array([0.0, 0.0, 5.0]),
        np.array([1.0, 1.0, 1.0, 1.0]),
        rs.random(1000) * (rs.random(1000) > 0.3),
        rs.random(5000) ** 8,
        np.concatenate([np.zeros(700), rs.random(3000), np.zeros(300)]),
    ]
    us = [0.0, 0.25, 0.5, 0.75, 1.0 - 2.0 ** -53, 0.123456789, 0.999999]
    for k, w in enumerate(vecs):
        out = []
        for u in us:
            out.append(rplu.sample_index(w, u))
        # exact boundary draws: u*total == c_k for a few k
        c = np.cumsum(w)
        arrays[f"w{k}"] = w
        arrays[f"idx{k}"] = np.array(out)
        info.append({"key": f"w{k}", "us": us, "n": int(w.size), "total": float(c[-1])})
    arrays["us"] = np.array(us)
    save("sample_index", arrays, info)


def dense_cases():
    arrays, info = {}, []
    cases = []
    rs = np.random.default_rng(11)
    cases.append(("diag2", np.eye(2), "rplu", 2, 3, 0.0))
    cases.append(("cplu2", np.array([[1.0, 3.0], [2.0, 0.0]]), "cplu", 1, None, 0.0))
    cases.append(("c8x6", rs.standard_normal((8, 6)) + 1j * rs.standard_normal((8, 6)), "rplu", 6, 1, 0.0))
    cases.append(("real40x30", rs.standard_normal((40, 30)), "rplu", 30, 2, 0.0))
    cases.append(("planted60", gen.planted_spectrum(60, 60, 0.3, 100), "rplu", 10, 7, 0.0))
    cases.append(("planted60c2", gen.planted_spectrum(60, 60, 0.3, 101), "c2plu", 12, None, 0.0))
    cases.append(("planted60cplu", gen.planted_spectrum(60, 60, 0.3, 102), "cplu", 12, None, 0.0))
    cases.append(("rank3_clean", rs.standard_normal((20, 3)) @ rs.standard_normal((3, 25)),
                  "rplu", 10, 4, 0.0))
    cases.append(("diag5_clean", np.diag([5.0, 4.0, 3.0, 2.0, 1.0]), "rplu", 5, 9, 0.0))
    cases.append(("tol_stop", gen.c1_dense(3, n=200), "rplu", 150, 3, 1e-2))
    cases.append(("c1_small_real", gen.c1_dense(0, n=300, m=257), "rplu", 60, 0, 0.0))
    cases.append(("c3_small_real", gen.c3_dense_host(0, n=512, m=384, reflectors=8), "rplu", 96, 0, 0.0))
    cases.append(("c3_small_f32src", gen.c3_dense_host(1, n=256, reflectors=8).astype(np.float32),
                  "rplu", 64, 1, 0.0))
    for name, A, tag, steps, seed, tol in cases:
        rule = rplu.PivotRule(tag, rplu.RngState(seed) if seed is not None else None)
        tr = rplu.eliminate(A, rule, steps, stop_tol=tol)
        after = rule.rng.uniform() if rule.rng is not None else None
        arrays[name + "_A"] = A
        arrays[name + "_L"] = tr.L
        arrays[name + "_U"] = tr.U
        arrays[name + "_resid_fro"] = tr.resid_fro
        if tr.residual.size <= 4096:
            arrays[name + "_residual"] = tr.residual
        info.append({"name": name, "rule": tag, "steps": steps, "seed": seed, "stop_tol": tol,
                     "pivots": [list(map(int, p)) for p in tr.pivots], "steps_done": tr.steps,
                     "clean_early_stop": bool(tr.clean_early_stop), "tol_stop": bool(tr.tol_stop),
                     "next_uniform": after})
    save("dense", arrays, info)


def cauchy_cases():
    arrays, info = {}, []
    rs = np.random.default_rng(21)
    cases = []
    x, y, G, B = gen.c2_cauchy(0, n=300)
    cases.append(("c2_300", x, y, G, B, "rplu", 40, 9, 0.0))
    x, y, G, B = gen.c4_cauchy_like(0, n=256, p=4)
    cases.append(("c4_256", x, y, G, B, "rplu", 32, 3, 0.0))
    x, y, G, B = gen.c4_cauchy_like(1, n=200, m=150, p=2)
    cases.append(("c4_200x150_p2", x, y, G, B, "rplu", 30, 5, 0.0))
    x, y, G, B = gen.c4_cauchy_like(2, n=128, p=3)
    cases.append(("c4_128_c2plu", x, y, G, B, "c2plu", 20, None, 0.0))
    x, y, G, B = gen.c2_cauchy(4, n=64)
    cases.append(("c2_64_full", x, y, G, B, "rplu", 64, 4, 1e-9))
    for name, x, y, G, B, rule, rank, seed, tol in cases:
        M = rplu.CauchyLikeMatrix(x, y, G, B)
        rng = rplu.RngState(seed) if seed is not None else None
        tr = rplu.structured_eliminate(M, rule, rank, stop_tol=tol, rng=rng, keep_steps=True)
        after = rng.uniform() if rng is not None else None
        arrays[name + "_x"], arrays[name + "_y"] = x, y
        arrays[name + "_G"], arrays[name + "_B"] = G, B
        k = len(tr.row_indices)
        if k:
            arrays[name + "_c"] = np.stack([s[0] for s in tr.steps])
            arrays[name + "_r"] = np.stack([s[1] for s in tr.steps])
            arrays[name + "_a"] = np.array([s[2] for s in tr.steps])
        arrays[name + "_norms0"] = rplu.exact_row_norms(M)
        info.append({"name": name, "rule": rule, "rank": rank, "seed": seed, "stop_tol": tol,
                     "rows": tr.row_indices, "cols": tr.col_indices,
                     "bound_sums": tr.bound_sums, "bound_maxes": tr.bound_maxes,
                     "tol_stop": tr.tol_stop, "degenerate_stop": tr.degenerate_stop,
                     "next_uniform": after})
    save("cauchy", arrays, info)


def _plan_signature(plan):
    """Per target leaf (keyed by its smallest point index): sorted aggregated
    alphas and the sorted point sets of the exact source leaves — a
    numbering-independent description of an InteractionPlan."""
    tgt, src = plan.target_tree, plan.source_tree
    sig = {}
    for leaf in tgt.leaves:
        key = int(np.min(tgt.nodes[leaf].points))
        alphas = sorted(float(a) for _, a in plan.aggregated[leaf])
        exact = sorted(sorted(int(i) for i in src.nodes[s].points) for s in plan.exact[leaf])
        sig[str(key)] = {"alphas": alphas, "exact": exact,
                         "points": sorted(int(i) for i in tgt.nodes[leaf].points)}
    return sig


def cauchy_plan_cases():
    """structured_eliminate WITH a plan (certified bounds + rejection
    sampling), the path every in-package Cauchy caller takes."""
    arrays, info = {}, []
    cases = []
    x, y, G, B = gen.c2_cauchy(0, n=300)
    cases.append(("c2_300_plan", x, y, G, B, "rplu", 40, 9, 0.0, 5.0, 32))
    x, y, G, B = gen.c4_cauchy_like(3, n=400, m=350, p=2)
    cases.append(("c4_400x350_p2_plan", x, y, G, B, "rplu", 30, 5, 0.0, 5.0, 16))
    x, y, G, B = gen.c4_cauchy_like(4, n=256, p=4)
    cases.append(("c4_256_c2plu_plan", x, y, G, B, "c2plu", 20, None, 0.0, 3.0, 32))
    for name, x, y, G, B, rule, rank, seed, tol, nu, leaf in cases:
        M = rplu.CauchyLikeMatrix(x, y, G, B)
        plan = rplu.build_plan(x, y, nu=nu, leaf_size=leaf)
        u0 = rplu.certified_upper_bounds(plan, M.G, M.B)
        rng = rplu.RngState(seed) if seed is not None else None
        tr = rplu.structured_eliminate(M, rule, rank, stop_tol=tol, nu=nu, plan=plan, rng=rng,
                                       keep_steps=True)
        after = rng.uniform() if rng is not None else None
        arrays[name + "_x"], arrays[name + "_y"] = x, y
        arrays[name + "_G"], arrays[name + "_B"] = G, B
        arrays[name + "_u0"] = u0
        arrays[name + "_exact0"] = rplu.exact_row_norms(M)
        if tr.steps:
            arrays[name + "_r"] = np.stack([s[1] for s in tr.steps])
        info.append({"name": name, "rule": rule, "rank": rank, "seed": seed, "stop_tol": tol,
                     "nu": nu, "leaf_size": leaf, "rows": tr.row_indices,
                     "cols": tr.col_indices, "proposals": tr.proposals,
                     "acceptances": tr.acceptances, "exact_fallbacks": tr.exact_fallbacks,
                     "bound_sums": tr.bound_sums, "bound_maxes": tr.bound_maxes,
                     "tol_stop": tr.tol_stop, "degenerate_stop": tr.degenerate_stop,
                     "next_uniform": after, "plan": _plan_signature(plan)})
    save("cauchy_plan", arrays, info)


class _Gauss(rplu.CallableOperator):
    def __init__(self, P, Q, h=0.1):
        d2 = ((P[:, None, :] - Q[None, :, :]) ** 2).sum(-1)
        K = np.exp(-d2 / (2 * h * h))
        self.K = K
        super().__init__(K.shape, lambda v: K @ v, lambda v: K.conj().T @ v,
                         row_norms_fn=lambda: np.einsum("ij,ij->i", K, K))


def cur_cases():
    arrays, info = {}, []
    cases = []
    A = gen.planted_spectrum(60, 60, 0.3, 100)
    cases.append(("planted60", rplu.DenseMatrix(A), A, "rplu-cur", 10, 7))
    P, Q = gen.c5_points(0, n=400, m=300)
    op = _Gauss(P, Q)
    cases.append(("gauss400x300", op, op.K, "rplu-cur", 24, 3))
    arrays["gauss400x300_P"], arrays["gauss400x300_Q"] = P, Q
    A2 = gen.c1_dense(5, n=120, m=90)
    cases.append(("c1_120x90", rplu.DenseMatrix(A2), A2, "rplu-cur", 30, 5))
    cases.append(("c1_120x90_c2", rplu.DenseMatrix(A2), A2, "c2plu-cur", 20, None))
    for name, acc, dense, rule, k, seed in cases:
        rng = rplu.RngState(seed) if seed is not None else None
        fact, inf = rplu.cur_build(acc, rule, k, rng=rng)
        after = rng.uniform() if rng is not None else None
        arrays[name + "_dense"] = dense
        arrays[name + "_W"] = fact.core_matrix()
        arrays[name + "_row_norms"] = inf.row_norms
        info.append({"name": name, "rule": rule, "rank": k, "seed": seed,
                     "I": fact.row_indices, "J": fact.col_indices,
                     "total_sq_norms": inf.total_sq_norms, "clamped": inf.clamped,
                     "rebuilds": inf.rebuilds, "degenerate_stop": inf.degenerate_stop,
                     "tol_stop": inf.tol_stop, "next_uniform": after})
    save("cur", arrays, info)


def c1_runs(seeds=range(30), steps=100):
    out = []
    for s in seeds:
        A = gen.c1_dense(s)
        tr = rplu.eliminate(A, rplu.PivotRule("rplu", rplu.RngState(s)), steps)
        err = float(np.linalg.norm(A - tr.L @ tr.U) / np.linalg.norm(A))
        out.append({"seed": s, "sha256": sha(A), "pivots": [list(map(int, p)) for p in tr.pivots],
                    "resid_fro": [float(v) for v in tr.resid_fro], "rel_err": err})
        print("c1 seed", s, err, tr.pivots[:2], flush=True)
    with open(os.path.join(HERE, "c1_reference.json"), "w") as f:
        json.dump({"meta": meta(), "n": 2000, "steps": steps, "runs": out}, f)


def _aaa_samples(name):
    """Seeded desk-size sample sets for the rational consumers (§8(f4))."""
    g = np.random.default_rng(len(name) * 7919)
    if name == "tanh_line":        # real segment, a function with nearby poles
        z = np.linspace(-1.0, 1.0, 240) + 0j
        return z, np.tanh(6.0 * z)
    if name == "circle_log":       # jittered unit circle, a branch point outside
        t = np.sort(g.uniform(0.0, 2 * np.pi, 300))
        z = np.exp(1j * t) * (1.0 + 0.01 * g.standard_normal(300))
        return z, np.log(2.5 - z)
    if name == "spiral_mero":      # C2-like spiral point set, a meromorphic function
        t = g.uniform(0.0, 1.0, 360)
        z = (0.1 + t) * np.exp(1j * 4 * np.pi * t) + 0.01 * (g.standard_normal(360)
                                                         + 1j * g.standard_normal(360))
        return z, np.exp(z) / (z - 1.7) + 1.0 / (z + 1.6j)
    raise KeyError(name)


def _cur_aaa_stable(S, tol, seed, leaf, result, trials=3):
    """Whether the reference's cur_aaa result survives 1e-15 relative
    perturbations of the generated rows / columns.  With exact-interaction
    leaves the certified bound equals ||r_i||^2 in exact arithmetic, so the
    rejection test rho >= u_i (which decides whether an acceptance uniform is
    drawn) is a rounding-level tie and the whole stream can shift; such
    inputs only get the fit-quality bar in the GPU test."""
    import warnings
    C = rplu.cauchy.CauchyLikeMatrix
    row, col = C.row, C.column
    g = np.random.default_rng(1)
    try:
        C.row = lambda self, i: row(self, i) * (1 + 1e-15 * g.standard_normal(self.shape[1]))
        C.column = lambda self, j: col(self, j) * (1 + 1e-15 * g.standard_normal(self.shape[0]))
        for _ in range(trials):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                rc, side = rplu.cur_aaa(S, tol=tol, rng=rplu.RngState(seed), leaf_size=leaf)
            if side != result[0] or not np.array_equal(rc.support, result[1]):
                return False
        return True
    finally:
        C.row, C.column = row, col


def rational_cases():
    """aaa / cur_aaa / bary_eval / loewner_build (rational.py, cauchy.py:280-306)."""
    import warnings
    arrays, info = {}, []
    for name, tol, seed in (("tanh_line", 1e-11, 3), ("circle_log", 1e-11, 5),
                            ("spiral_mero", 1e-10, 11)):
        z, f = _aaa_samples(name)
        S = rplu.SampleSet(z, f)
        arrays[name + "_z"], arrays[name + "_f"] = z, f
        r, errs = rplu.aaa(S, tol=1e-13, max_degree=60)
        zt = z[:-1] + 0.37 * np.diff(z)              # off-sample evaluation points
        arrays[name + "_zt"] = zt
        arrays[name + "_aaa_support"] = r.support
        arrays[name + "_aaa_weights"] = r.weights
        arrays[name + "_aaa_errors"] = errs
        arrays[name + "_aaa_eval"] = r(zt)
        cur = {}
        for leaf in (None, 8):
            tag = "_cur" if leaf is None else "_cur8"
            rng = rplu.RngState(seed)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                rc, side = rplu.cur_aaa(S, tol=tol, rng=rng, leaf_size=leaf)
            after = rng.uniform()
            arrays[name + tag + "_support"] = rc.support
            arrays[name + tag + "_weights"] = rc.weights
            arrays[name + tag + "_eval"] = rc(zt)
            arrays[name + tag + "_err"] = np.array([np.max(np.abs(rc(z) - f))])
            cur[tag] = {"leaf_size": leaf, "side": side, "next_uniform": after,
                        "support_idx": [int(np.nonzero(z == t)[0][0]) for t in rc.support],
                        "degree": int(rc.degree),
                        "stable": _cur_aaa_stable(S, tol, seed, leaf, (side, rc.support))}
        # the split Loewner generators cur_aaa eliminates
        perm = rplu.RngState(seed).permutation(z.size)
        half = (z.size + 1) // 2
        L = rplu.cauchy.loewner_build(z[perm[:half]], f[perm[:half]], z[perm[half:]],
                                      f[perm[half:]])
        arrays[name + "_loewner_G"], arrays[name + "_loewner_B"] = L.G, L.B
        info.append({"name": name, "tol": tol, "seed": seed, "cur": cur,
                     "aaa_support_idx": [int(np.nonzero(z == t)[0][0]) for t in r.support],
                     "aaa_degree": int(r.degree)})
    # bary_eval edge cases: exact support hits, a point on a pole
    t = np.array([0.0, 1.0, 1j, -1.0 + 0.5j])
    fv = np.array([1.0, 2.0 - 1j, 0.5j, -3.0])
    w = np.array([1.0, -2.0, 1.5j, 0.25 - 0.25j])
    r = rplu.BarycentricRational(t, fv, w)
    ze = np.array([0.0, 1.0 + 1e-16, 0.3 + 0.2j, 2.0, 1j, 5.0 - 5j])
    out, flags = r.eval_flagged(ze)
    arrays["bary_t"], arrays["bary_f"], arrays["bary_w"] = t, fv, w
    arrays["bary_z"], arrays["bary_out"], arrays["bary_flags"] = ze, out, flags
    save("rational", arrays, info)


def precond_cases():
    """smw_build + gmres (precond.py) on a banded-plus-low-rank system."""
    import scipy.linalg as sla
    arrays, info = {}, []
    for name, n, k, seed in (("band_lowrank300", 300, 20, 4), ("band_lowrank200_k8", 200, 8, 9)):
        A = gen.planted_spectrum(n, n, 0.5, seed) * 40.0
        main = np.full(n, 4.0)
        off = np.full(n - 1, -1.0)
        ab = np.zeros((3, n))
        ab[0, 1:], ab[1, :], ab[2, :-1] = off, main, off

        def b_inv(v, ab=ab):
            return sla.solve_banded((1, 1), ab, v)

        def K_apply(v, A=A, main=main, off=off):
            out = A @ v
            out = out + main * v
            out[:-1] += off * v[1:]
            out[1:] += off * v[:-1]
            return out

        rng = rplu.RngState(seed)
        b = rng.complex_normal(n)
        fact, _ = rplu.cur_build(rplu.DenseMatrix(A), "rplu-cur", k, rng=rplu.RngState(seed ^ 1))
        pre = rplu.smw_build(b_inv, rplu.DenseMatrix(A), fact)
        v = rplu.RngState(seed + 100).complex_normal(n)
        res_pre = rplu.gmres(K_apply, b, M_inv=pre, restart=20, tol=1e-10, max_restarts=200)
        res_plain = rplu.gmres(K_apply, b, restart=10, tol=1e-8, max_restarts=300)
        arrays[name + "_b"], arrays[name + "_v"] = b, v   # A regenerated from gen (seeded)
        arrays[name + "_pre_v"] = pre.apply(v)
        arrays[name + "_x_pre"], arrays[name + "_hist_pre"] = res_pre.x, res_pre.residuals
        arrays[name + "_x_plain"], arrays[name + "_hist_plain"] = res_plain.x, res_plain.residuals
        info.append({"name": name, "n": n, "k": k, "seed": seed,
                     "I": [int(i) for i in fact.row_indices],
                     "J": [int(j) for j in fact.col_indices],
                     "pre": {"iterations": res_pre.iterations, "converged": res_pre.converged,
                             "stagnated": res_pre.stagnated},
                     "plain": {"iterations": res_plain.iterations,
                               "converged": res_plain.converged,
                               "stagnated": res_plain.stagnated}})
    save("precond", arrays, info)


def sweep_cases():
    """The reference's error sweep (cli._sweep_rows, cli.py:100-138) over the
    hot-path methods: rows (rank, method, seed, frob_err/||A||_F,
    spec_err/||A||_2, seconds, applies, adjoints)."""
    from rplu import cli
    info = []
    for name, A, methods, ranks, trials, seed in (
            ("planted120x100", gen.planted_spectrum(120, 100, 0.8, 3),
             ["rplu", "cplu", "c2plu", "rplu-cur", "c2plu-cur", "svd-oracle"], [4, 8, 16], 3, 11),
            ("c1_300x250", gen.c1_dense(2, n=300, m=250), ["rplu", "rplu-cur", "svd-oracle"],
             [10, 40], 2, 5)):
        rows = cli._sweep_rows(rplu.DenseMatrix(A), methods, ranks, trials, seed)
        info.append({"name": name, "sha256": sha(A), "methods": methods, "ranks": ranks,
                     "trials": trials, "seed": seed,
                     "rows": [[int(k), m, int(sd), float(ef), float(es), 0.0, int(na), int(nat)]
                              for (k, m, sd, ef, es, _sec, na, nat) in rows]})
    with open(os.path.join(HERE, "sweep.json"), "w") as f:
        json.dump({"meta": meta(), "cases": info}, f, indent=1)


if __name__ == "__main__":
    if "--sweep" in sys.argv:
        sweep_cases()
        sys.exit(0)
    if "--consumers" not in sys.argv:
        sample_index_cases()
        dense_cases()
        cauchy_cases()
        cauchy_plan_cases()
        cur_cases()
    rational_cases()
    precond_cases()
    if "--c1" in sys.argv:
        c1_runs()
