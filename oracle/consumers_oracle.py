"""numpy restatement of the reference's downstream consumers of the pivots
 — TEST INFRASTRUCTURE ONLY.

* barycentric rationals and greedy AAA (rplu/rational.py:25-175),
* the Loewner generators of CUR-AAA (rplu/cauchy.py:280-306),
* the SMW preconditioner and restarted MGS-GMRES (rplu/precond.py:30-192).

Pinned against the reference's own outputs in tests/golden/rational.* and
tests/golden/precond.* (tests/test_oracle_golden.py).  ``cur_aaa`` itself is
not restated here (it needs the certified-bound plan path); its GPU parity
test compares against the reference's goldens directly.
"""

import numpy as np
import scipy.linalg

__all__ = ["loewner_generators", "loewner_matrix", "loewner_weights", "bary_eval_flagged",
           "aaa", "smw_apply_factory", "gmres_mgs"]

HIT_TOL = 1e-14   # rational.py:22


def loewner_generators(x, fx, y, fy):
    """G = [fx/a, a], B = [a; -fy/a], a = sqrt(max|f|) or 1 (cauchy.py:296-305)."""
    fx = np.asarray(fx, np.complex128).ravel()
    fy = np.asarray(fy, np.complex128).ravel()
    top = max(np.abs(fx).max(initial=0.0), np.abs(fy).max(initial=0.0))
    a = 1.0 if top == 0.0 else float(np.sqrt(top))
    G = np.empty((fx.size, 2), np.complex128)
    G[:, 0], G[:, 1] = fx / a, a
    B = np.empty((2, fy.size), np.complex128)
    B[0], B[1] = a, -fy / a
    return G, B


def loewner_matrix(zs, fs, zo, fo):
    """Divided differences (fo_i - fs_j) / (zo_i - zs_j) (rational.py:126-127)."""
    return np.subtract.outer(fo, fs) / np.subtract.outer(zo, zs)


def loewner_weights(zs, fs, zo, fo):
    """Conjugated last right singular vector (rational.py:128-130)."""
    L = loewner_matrix(zs, fs, zo, fo)
    Vh = np.linalg.svd(L)[2]
    return Vh[-1].conj()


def bary_eval_flagged(t, f, w, z):
    """(values, near_pole) of sum c w f / sum c w, c = 1/(z - t)
    (rational.py:63-80), with the exact-hit override."""
    t, f, w = (np.asarray(a, np.complex128).ravel() for a in (t, f, w))
    w = w / np.linalg.norm(w)
    z = np.atleast_1d(np.asarray(z, np.complex128)).ravel()
    with np.errstate(divide="ignore", invalid="ignore"):
        C = 1.0 / np.subtract.outer(z, t)
        den = C @ w
        val = (C @ (w * f)) / den
    flag = (np.abs(den) < 1e3 * np.finfo(float).tiny) | ~np.isfinite(val)
    lim = HIT_TOL * max(float(np.abs(t).max()), 1.0)
    for j in range(t.size):
        on = np.abs(z - t[j]) <= lim
        val[on] = f[j]
        flag[on] = False
    return val, flag


def aaa(z, f, tol=1e-13, max_degree=100):
    """Greedy AAA (rational.py:134-175): support indices, weights, errors."""
    z = np.asarray(z, np.complex128).ravel()
    f = np.asarray(f, np.complex128).ravel()
    top = float(np.abs(f).max())
    alive = np.ones(z.size, bool)
    sup, errs = [], []
    approx = np.full(z.size, np.mean(f), np.complex128)
    w = np.ones(1, np.complex128)
    for _ in range(min(max_degree, z.size - 1)):
        cand = np.nonzero(alive)[0]
        pick = int(cand[np.argmax(np.abs(f[cand] - approx[cand]))])
        sup.append(pick)
        alive[pick] = False
        rest = np.nonzero(alive)[0]
        w = loewner_weights(z[sup], f[sup], z[rest], f[rest])
        with np.errstate(divide="ignore", invalid="ignore"):
            C = 1.0 / np.subtract.outer(z[rest], z[sup])
            vals = (C @ (w * f[sup])) / (C @ w)
        vals[~np.isfinite(vals)] = 0.0
        approx = f.copy()
        approx[rest] = vals
        errs.append(float(np.abs(f - approx).max()))
        if errs[-1] <= tol * max(top, np.finfo(float).tiny):
            break
    return sup, w / np.linalg.norm(w), np.array(errs)


def smw_apply_factory(b_inv, A, I, J):
    """v -> (B + A[:,J] W^{-1} A[I,:])^{-1} v with W = A[I,J] (precond.py:48-94),
    dense A."""
    A = np.asarray(A, np.complex128)
    I, J = list(I), list(J)
    X = np.column_stack([b_inv(A[:, j]) for j in J])
    inner = A[np.ix_(I, J)] + A[I, :] @ X
    lu = scipy.linalg.lu_factor(inner)

    def apply(v):
        u = b_inv(np.asarray(v, np.complex128))
        q = scipy.linalg.lu_solve(lu, (A @ u)[I])
        return u - b_inv(A[:, J] @ q)
    return apply


def gmres_mgs(K, b, M=None, restart=20, tol=1e-10, max_restarts=200):
    """Right-preconditioned restarted GMRES, MGS Arnoldi, Givens on the
    Hessenberg column (precond.py:137-192).  Returns (x, history, iters,
    converged, stagnated)."""
    M = (lambda v: v) if M is None else M
    b = np.asarray(b, np.complex128)
    n = b.size
    x = np.zeros(n, np.complex128)
    bn = float(np.linalg.norm(b))
    hist, iters = [], 0
    best, best_res = x.copy(), np.inf
    for _ in range(max_restarts):
        r = b - K(x)
        beta = float(np.linalg.norm(r))
        if beta / bn <= tol:
            return x, np.array(hist), iters, True, False
        start = beta / bn
        V = np.zeros((n, restart + 1), np.complex128)
        H = np.zeros((restart + 1, restart), np.complex128)
        cs = np.zeros(restart, np.complex128)
        sn = np.zeros(restart, np.complex128)
        g = np.zeros(restart + 1, np.complex128)
        V[:, 0], g[0] = r / beta, beta
        done = 0
        for j in range(restart):
            w = K(M(V[:, j]))
            for t in range(j + 1):
                H[t, j] = np.vdot(V[:, t], w)
                w = w - H[t, j] * V[:, t]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 0:
                V[:, j + 1] = w / H[j + 1, j]
            for t in range(j):
                a, c = H[t, j], H[t + 1, j]
                H[t, j] = cs[t] * a + sn[t] * c
                H[t + 1, j] = -np.conj(sn[t]) * a + np.conj(cs[t]) * c
            d = np.sqrt(abs(H[j, j]) ** 2 + abs(H[j + 1, j]) ** 2)
            cs[j], sn[j] = (1.0, 0.0) if d == 0.0 else (np.conj(H[j, j]) / d,
                                                       np.conj(H[j + 1, j]) / d)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1], g[j] = -np.conj(sn[j]) * g[j], cs[j] * g[j]
            iters += 1
            done = j + 1
            hist.append(float(abs(g[j + 1])) / bn)
            if hist[-1] <= tol:
                break
        y = scipy.linalg.solve_triangular(H[:done, :done], g[:done])
        x = x + M(V[:, :done] @ y)
        rel = float(np.linalg.norm(b - K(x))) / bn
        if rel < best_res:
            best_res, best = rel, x.copy()
        if rel <= tol:
            return x, np.array(hist), iters, True, False
        if start - rel < 1e-14 * start:
            return best, np.array(hist), iters, False, True
    return best, np.array(hist), iters, False, False
