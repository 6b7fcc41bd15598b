"""numpy restatement of the reference RPLU loops (TEST INFRASTRUCTURE ONLY).

Every routine cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/rplu).  Two flavours of dense Alg 1:

* ``eliminate_c128`` follows the reference arithmetic literally (complex128
  residual, einsum row masses, np.abs column weights, R - outer(col, row)),
  so it reproduces the golden vectors bit for bit;
* ``eliminate_real`` is a real-fp64 restatement (different row-mass
  reduction order, in-place blocked update) used for the large configs; it
  is pinned to the reference through the same goldens (pivots identical,
  factors equal to rounding).

Also: ``sample_index`` / ``draw_margin`` (inverse-CDF draw and its distance to
the nearest CDF boundary), forced-pivot replay, the Cauchy-like exact-norm
loop, the CUR-form Alg 2 and a host Gaussian-kernel operator.
"""

import numpy as np
import scipy.linalg

__all__ = [
    "NEAR_REL", "PIVOT_REL_TOL", "sample_index", "draw_margin", "uniform_stream",
    "eliminate_c128", "eliminate_real", "replay_pivots",
    "cauchy_row", "cauchy_column", "exact_row_norms", "structured_eliminate",
    "generator_schur_update", "GaussianKernelHost", "DenseHost", "cur_build",
    "lu_error",
]

NEAR_REL = 1e-12  # north star: draws within 1e-12 relative of a CDF boundary


def uniform_stream(seed):
    """The reference stream: numpy Generator(Philox(key=seed)) (rng.py:25-33)."""
    return np.random.Generator(np.random.Philox(key=int(seed)))


# ---------------------------------------------------------------------------
# rng.py:50-74

def sample_index(weights, u):
    """First index whose cumulative weight exceeds u*total, with the
    reference's top clamp and zero-weight walk-back (rng.py:50-74)."""
    w = np.asarray(weights, dtype=float)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("weights must be a nonempty 1-D array")
    if (w < 0).any():
        raise ValueError("weights must be nonnegative")
    cdf = np.cumsum(w)
    if not cdf[-1] > 0:
        raise ValueError("all weights are zero; nothing to sample")
    k = min(int(np.searchsorted(cdf, u * cdf[-1], side="right")), w.size - 1)
    while k > 0 and not w[k] > 0:
        k -= 1
    if not w[k] > 0:
        k = int(np.argmax(w > 0))
    return k


def draw_margin(weights, u):
    """Relative distance of u*total to the nearest CDF boundary of the draw."""
    w = np.asarray(weights, dtype=float)
    cdf = np.cumsum(w)
    total = cdf[-1]
    target = u * total
    k = min(int(np.searchsorted(cdf, target, side="right")), w.size - 1)
    lo = cdf[k - 1] if k > 0 else 0.0
    return min(abs(target - lo), abs(cdf[k] - target)) / total


# ---------------------------------------------------------------------------
# dense_pivots.py:103-209

def _rank1_draw(R, tag, gen, masses_fn, weights_fn, margins):
    """One pivot for rules rplu / c2plu / cplu (dense_pivots.py:103-126)."""
    if tag == "cplu":
        flat = int(np.argmax(np.abs(R)))
        return divmod(flat, R.shape[1])
    masses = masses_fn(R)
    if tag == "c2plu":
        i = int(np.argmax(masses))
        return i, int(np.argmax(np.abs(R[i])))
    u1 = float(gen.random())
    i = sample_index(masses, u1)
    w = weights_fn(R[i])
    u2 = float(gen.random())
    j = sample_index(w, u2)
    if margins is not None:
        margins.append(min(draw_margin(masses, u1), draw_margin(w, u2)))
    return i, j


def _run_alg1(R, tag, steps, gen, stop_tol, masses_fn, weights_fn, update_fn, norm_fn,
              margins=None):
    n, m = R.shape
    if not 0 <= steps <= min(n, m):
        raise ValueError(f"steps {steps} out of range [0, {min(n, m)}]")
    if stop_tol < 0:
        raise ValueError("stop_tol must be nonnegative")
    L = np.zeros((n, steps), dtype=R.dtype)
    U = np.zeros((steps, m), dtype=R.dtype)
    piv = []
    resid = [norm_fn(R)]
    fro0 = resid[0]
    clean = tol = False
    for t in range(steps):
        if resid[-1] == 0.0:          # dense_pivots.py:162-164
            clean = True
            break
        i, j = _rank1_draw(R, tag, gen, masses_fn, weights_fn, margins)
        a = R[i, j]
        if a == 0:                     # one resample, then error (:178-184)
            i, j = _rank1_draw(R, tag, gen, masses_fn, weights_fn, margins)
            a = R[i, j]
            if a == 0:
                raise ZeroDivisionError(
                    f"pivot ({i}, {j}) has exactly zero value after resampling")
        col, row = update_fn(R, i, j, a)
        L[:, t] = col
        U[t, :] = row
        piv.append((int(i), int(j)))
        resid.append(norm_fn(R))
        if stop_tol > 0 and resid[-1] <= stop_tol * fro0:   # :195-197
            tol = True
            break
    k = len(piv)
    return dict(pivots=piv, L=L[:, :k], U=U[:k], resid_fro=np.array(resid), residual=R,
                steps=k, clean_early_stop=clean, tol_stop=tol,
                margins=None if margins is None else np.array(margins))


def eliminate_c128(A, tag, steps, seed=None, gen=None, stop_tol=0.0, margins=False):
    """Alg 1 with the reference's complex128 arithmetic (dense_pivots.py:129-209)."""
    if tag not in ("rplu", "cplu", "c2plu"):
        raise ValueError(f"unknown pivot rule {tag!r}")
    if gen is None and tag == "rplu":
        gen = uniform_stream(seed)
    state = {"R": np.array(A, dtype=np.complex128)}

    def masses_fn(R):
        return np.einsum("ij,ij->i", R, R.conj()).real

    def weights_fn(r):
        return np.abs(r) ** 2

    def update_fn(R, i, j, a):
        col = R[:, j] / a
        row = R[i, :].copy()
        state["R"] = R - np.outer(col, row)
        return col, row

    R = state["R"]
    n, m = R.shape
    if not 0 <= steps <= min(n, m):
        raise ValueError(f"steps {steps} out of range [0, {min(n, m)}]")
    if stop_tol < 0:
        raise ValueError("stop_tol must be nonnegative")
    # the residual is rebound each step (R - outer), so drive the loop here
    L = np.zeros((n, steps), dtype=np.complex128)
    U = np.zeros((steps, m), dtype=np.complex128)
    piv, mg = [], ([] if margins else None)
    resid = [float(np.linalg.norm(R))]
    clean = tol = False
    for t in range(steps):
        if resid[-1] == 0.0:
            clean = True
            break
        i, j = _rank1_draw(R, tag, gen, masses_fn, weights_fn, mg)
        a = R[i, j]
        if a == 0:
            i, j = _rank1_draw(R, tag, gen, masses_fn, weights_fn, mg)
            a = R[i, j]
            if a == 0:
                raise ZeroDivisionError(
                    f"pivot ({i}, {j}) has exactly zero value after resampling")
        col, row = update_fn(R, i, j, a)
        R = state["R"]
        L[:, t] = col
        U[t, :] = row
        piv.append((int(i), int(j)))
        resid.append(float(np.linalg.norm(R)))
        if stop_tol > 0 and resid[-1] <= stop_tol * resid[0]:
            tol = True
            break
    k = len(piv)
    return dict(pivots=piv, L=L[:, :k], U=U[:k], resid_fro=np.array(resid), residual=R,
                steps=k, clean_early_stop=clean, tol_stop=tol,
                margins=None if mg is None else np.array(mg))


def eliminate_real(A, tag, steps, seed=None, gen=None, stop_tol=0.0, dtype=np.float64,
                   margins=False, block_rows=1024, threads=1, copy=True):
    """Real restatement of Alg 1 for large inputs (same semantics as
    dense_pivots.py:129-209 restricted to real data; arithmetic of the update
    identical to the reference's zero-imaginary complex128 path: col =
    R[:,j]*(1/a), R -= col (x) row with one rounding per operation)."""
    if tag not in ("rplu", "cplu", "c2plu"):
        raise ValueError(f"unknown pivot rule {tag!r}")
    if gen is None and tag == "rplu":
        gen = uniform_stream(seed)
    R = np.array(A, dtype=dtype) if copy else np.asarray(A, dtype=dtype)
    one = dtype(1.0)
    pool = None
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        pool = ThreadPoolExecutor(threads)
    blocks = [(lo, min(lo + block_rows, R.shape[0])) for lo in range(0, R.shape[0], block_rows)]

    def each_block(fn):
        if pool is None:
            for b in blocks:
                fn(*b)
        else:
            list(pool.map(lambda b: fn(*b), blocks))

    def masses_fn(R):
        out = np.empty(R.shape[0])

        def blk(lo, hi):
            out[lo:hi] = np.einsum("ij,ij->i", R[lo:hi], R[lo:hi], dtype=np.float64)
        each_block(blk)
        return out

    def weights_fn(r):
        r64 = r.astype(np.float64)
        return r64 * r64

    def update_fn(R, i, j, a):
        col = R[:, j] * (one / a)
        row = R[i, :].copy()

        def blk(lo, hi):
            R[lo:hi] -= np.outer(col[lo:hi], row)
        each_block(blk)
        return col, row

    def norm_fn(R):
        parts = np.zeros(len(blocks))

        def blk(lo, hi):
            parts[blocks.index((lo, hi))] = np.einsum("ij,ij->", R[lo:hi], R[lo:hi],
                                                      dtype=np.float64)
        each_block(blk)
        return float(np.sqrt(parts.sum()))

    try:
        return _run_alg1(R, tag, steps, gen, stop_tol, masses_fn, weights_fn, update_fn, norm_fn,
                         [] if margins else None)
    finally:
        if pool is not None:
            pool.shutdown()


def replay_pivots(A, pivots, dtype=np.float64):
    """Forced-pivot replay of Alg 1 (dense_pivots.py:185-191) with given
    pivots; the fp64 replay grades fp32 factors (north star: 1e-4)."""
    R = np.array(A, dtype=dtype)
    n, m = R.shape
    k = len(pivots)
    L = np.zeros((n, k), dtype=dtype)
    U = np.zeros((k, m), dtype=dtype)
    resid = [float(np.linalg.norm(R))]
    for t, (i, j) in enumerate(pivots):
        a = R[i, j]
        col = R[:, j] * (dtype(1.0) / a) if not np.iscomplexobj(R) else R[:, j] / a
        row = R[i].copy()
        R -= np.outer(col, row)
        L[:, t] = col
        U[t] = row
        resid.append(float(np.linalg.norm(R)))
    return dict(L=L, U=U, residual=R, resid_fro=np.array(resid))


def lu_error(A, L, U):
    """||A - L U||_F / ||A||_F (cli.py:151-157 error evaluation)."""
    A = np.asarray(A)
    return float(np.linalg.norm(A - L @ U) / np.linalg.norm(A))


# ---------------------------------------------------------------------------
# cauchy.py:39-256 (plan=None exact-norm path)

def cauchy_row(x, y, G, B, i):
    """Row i: (G_i . B) / (x_i - y) (cauchy.py:82-83)."""
    return (G[i, :] @ B) / (x[i] - y)


def cauchy_column(x, y, G, B, j):
    """Column j: (G . B_:,j) / (x - y_j) (cauchy.py:85-86)."""
    return (G @ B[:, j]) / (x - y[j])


def exact_row_norms(x, y, G, B, block_entries=2_000_000):
    """u_i = sum_j |G_i B_:,j / (x_i - y_j)|^2 in row blocks (cauchy.py:129-137)."""
    n, m = G.shape[0], B.shape[1]
    out = np.empty(n)
    rows = max(1, block_entries // max(m, 1))
    for lo in range(0, n, rows):
        hi = min(lo + rows, n)
        K = (G[lo:hi] @ B) / (x[lo:hi, None] - y[None, :])
        out[lo:hi] = np.einsum("ij,ij->i", K, K.conj()).real
    return out


PIVOT_REL_TOL = 1e-14  # cauchy.py:33


def generator_schur_update(x, y, G, B, i, j):
    """One generator update (cauchy.py:140-154); returns (G1, B1)."""
    r = cauchy_row(x, y, G, B, i)
    a = r[j]
    if abs(a) <= PIVOT_REL_TOL * float(np.max(np.abs(r))):
        raise ZeroDivisionError(f"pivot ({i}, {j}) is numerically zero")
    c = cauchy_column(x, y, G, B, j)
    return G - np.outer(c / a, G[i, :]), B - np.outer(B[:, j], r / a)


def structured_eliminate(x, y, G, B, rule, rank, seed=None, gen=None, stop_tol=0.0,
                         keep_steps=False, margins=False):
    """Alg 3 with exact row norms (cauchy.py:177-256, plan=None branch)."""
    if rule not in ("rplu", "c2plu"):
        raise ValueError(f"unknown structured rule {rule!r}")
    if rule == "rplu" and gen is None:
        if seed is None:
            raise ValueError("structured rplu needs an RngState")
        gen = uniform_stream(seed)
    x = np.asarray(x, dtype=np.complex128).ravel()
    y = np.asarray(y, dtype=np.complex128).ravel()
    G = np.ascontiguousarray(np.asarray(G, dtype=np.complex128))
    B = np.asarray(B, dtype=np.complex128, order="F")
    n, m = G.shape[0], B.shape[1]
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    out = dict(row_indices=[], col_indices=[], steps=[], bound_sums=[], bound_maxes=[],
               tol_stop=False, degenerate_stop=False, margins=[] if margins else None)
    u0 = None
    for _ in range(rank):
        u = exact_row_norms(x, y, G, B)
        umax, usum = float(np.max(u)), float(np.sum(u))
        out["bound_maxes"].append(umax)
        out["bound_sums"].append(usum)
        u0 = umax if u0 is None else u0
        if umax <= 0.0:
            out["degenerate_stop"] = True
            break
        if stop_tol > 0 and umax <= stop_tol ** 2 * u0:
            out["tol_stop"] = True
            break
        if rule == "c2plu":
            i = int(np.argmax(u))
        else:
            u1 = float(gen.random())
            i = sample_index(u, u1)
        r = cauchy_row(x, y, G, B, i)
        w = np.abs(r) ** 2
        if rule == "c2plu":
            j = int(np.argmax(np.abs(r)))
        else:
            u2 = float(gen.random())
            j = sample_index(w, u2)
            if margins:
                out["margins"].append(min(draw_margin(u, u1), draw_margin(w, u2)))
        a = r[j]
        thr = PIVOT_REL_TOL * float(np.max(np.abs(r)))
        if abs(a) <= thr:
            if rule == "c2plu":
                raise ZeroDivisionError(f"pivot ({i}, {j}) is numerically zero")
            j = sample_index(w, float(gen.random()))
            a = r[j]
            if abs(a) <= thr:
                raise ZeroDivisionError(
                    f"pivot ({i}, {j}) is numerically zero after resampling")
        c = cauchy_column(x, y, G, B, j)
        G = G - np.outer(c / a, G[i, :])
        B = np.asfortranarray(B - np.outer(B[:, j], r / a))
        out["row_indices"].append(int(i))
        out["col_indices"].append(int(j))
        if keep_steps:
            out["steps"].append((c.copy(), r.copy(), complex(a)))
    out["G"], out["B"] = G, B
    return out


# ---------------------------------------------------------------------------
# lowmem_cur.py:161-312 (Alg 2, CUR form, QR core)

class DenseHost:
    """Host dense operator with the accessor calls cur_build uses."""

    def __init__(self, A):
        self.A = np.asarray(A, dtype=np.complex128)
        self.shape = self.A.shape

    def apply(self, v):
        return self.A @ v

    def adjoint_apply(self, v):
        return self.A.conj().T @ v

    def row_norms(self):
        return np.einsum("ij,ij->i", self.A, self.A.conj()).real


class GaussianKernelHost:
    """A_ij = exp(-|p_i - q_j|^2 / (2 h^2)) applied in row blocks (C5)."""

    def __init__(self, P, Q, h=0.1, block_entries=4_000_000):
        self.P = np.ascontiguousarray(P, dtype=np.float64)
        self.Q = np.ascontiguousarray(Q, dtype=np.float64)
        self.h = float(h)
        self.shape = (self.P.shape[0], self.Q.shape[0])
        self.rows = max(1, block_entries // max(self.shape[1], 1))

    def block(self, lo, hi):
        d2 = np.zeros((hi - lo, self.shape[1]))
        for c in range(3):
            diff = self.P[lo:hi, c, None] - self.Q[None, :, c]
            d2 += diff * diff
        return np.exp(-d2 / (2.0 * self.h * self.h))

    def apply(self, v):
        v = np.asarray(v)
        out = np.zeros(self.shape[0], dtype=np.result_type(v.dtype, np.float64))
        for lo in range(0, self.shape[0], self.rows):
            hi = min(lo + self.rows, self.shape[0])
            out[lo:hi] = self.block(lo, hi) @ v
        return out

    def adjoint_apply(self, v):
        v = np.asarray(v)
        out = np.zeros(self.shape[1], dtype=np.result_type(v.dtype, np.float64))
        for lo in range(0, self.shape[0], self.rows):
            hi = min(lo + self.rows, self.shape[0])
            out += self.block(lo, hi).T @ v[lo:hi]
        return out

    def row_norms(self):
        out = np.empty(self.shape[0])
        for lo in range(0, self.shape[0], self.rows):
            hi = min(lo + self.rows, self.shape[0])
            K = self.block(lo, hi)
            out[lo:hi] = np.einsum("ij,ij->i", K, K)
        return out

    def materialize(self):
        return self.block(0, self.shape[0])


class _QrCore:
    """Core A[I,J] with a QR recomputed at every extension (lowmem_cur.py:43-133)."""

    def __init__(self):
        self.I, self.J = [], []
        self.W = np.zeros((0, 0), dtype=np.complex128)
        self.Q = self.R = None

    def solve(self, v):                      # :72-79  W x = v
        if not self.I:
            return np.zeros(0, dtype=np.complex128)
        return scipy.linalg.solve_triangular(self.R, self.Q.conj().T @ v)

    def solve_t(self, v):                    # :81-88  W^T x = v
        if not self.I:
            return np.zeros(0, dtype=np.complex128)
        return self.Q.conj() @ scipy.linalg.solve_triangular(self.R, v, trans="T")

    def extend(self, i, j, w, z, omega):     # :90-133
        k = len(self.I)
        W = np.zeros((k + 1, k + 1), dtype=np.complex128)
        W[:k, :k] = self.W
        W[:k, k] = w
        W[k, :k] = z
        W[k, k] = omega
        self.W = W
        self.I.append(int(i))
        self.J.append(int(j))
        self.Q, self.R = scipy.linalg.qr(W)


def _unit(n, i):
    e = np.zeros(n, dtype=np.complex128)
    e[i] = 1.0
    return e


def cur_build(A, rule, rank, seed=None, gen=None, stop_tol=0.0, margins=False):
    """Alg 2 in CUR form driven by applies (lowmem_cur.py:212-300), QR core."""
    if rule not in ("rplu-cur", "c2plu-cur"):
        raise ValueError(f"unknown CUR rule {rule!r}")
    if rule == "rplu-cur" and gen is None:
        if seed is None:
            raise ValueError("rplu-cur needs an RngState")
        gen = uniform_stream(seed)
    n, m = A.shape
    if not 0 <= rank <= min(n, m):
        raise ValueError(f"rank {rank} out of range [0, {min(n, m)}]")
    core = _QrCore()
    info = dict(total_sq_norms=[], clamped=[], rebuilds=0, degenerate_stop=False,
                tol_stop=False, margins=[] if margins else None)
    nrow = np.asarray(A.row_norms(), dtype=float).copy()
    total0 = float(np.sum(nrow))
    info["total_sq_norms"].append(total0)
    if total0 == 0.0:
        info["degenerate_stop"] = True
        info["row_norms"] = nrow
        return core, info
    eps = np.finfo(float).eps

    def cols_apply(w):                       # A[:, J] w   (:174-179)
        v = np.zeros(m, dtype=np.complex128)
        if core.J:
            v[core.J] = w
        return A.apply(v)

    def rows_tapply(w):                      # A[I, :]^T w (:182-187)
        v = np.zeros(n, dtype=np.complex128)
        if core.I:
            v[core.I] = w
        return np.conj(A.adjoint_apply(np.conj(v)))

    def draw_row():                          # :303-312
        if rule == "rplu-cur":
            u1 = float(gen.random())
            i = sample_index(nrow, u1)
            if margins:
                info["margins"].append(draw_margin(nrow, u1))
        else:
            i = int(np.argmax(nrow))
        r = np.conj(A.adjoint_apply(_unit(n, i)))
        rhat = r - rows_tapply(core.solve_t(r[core.J]))
        return i, rhat, r

    for _ in range(rank):
        if np.sum(nrow) <= 0.0:
            info["degenerate_stop"] = True
            break
        i, rhat, r = draw_row()
        energy = float(np.sum(np.abs(rhat) ** 2))
        if energy <= eps ** 2 * total0:
            i, rhat, r = draw_row()
            energy = float(np.sum(np.abs(rhat) ** 2))
            if energy <= eps ** 2 * total0:
                info["degenerate_stop"] = True
                break
        w = np.abs(rhat) ** 2
        if rule == "rplu-cur":
            u2 = float(gen.random())
            j = sample_index(w, u2)
            if margins:
                info["margins"].append(draw_margin(w, u2))
        else:
            j = int(np.argmax(np.abs(rhat)))
        a = rhat[j]
        c = A.apply(_unit(m, j))
        chat = c - cols_apply(core.solve(c[core.I]))
        l = np.conj(rhat) / np.conj(a)
        g = A.apply(l)
        v = cols_apply(core.solve(g[core.I]))
        prev = info["total_sq_norms"][-1]
        nrow -= 2.0 * np.real((g - v) * np.conj(chat))
        nrow += float(np.real(np.vdot(l, l))) * (np.abs(chat) ** 2)
        floor = eps * prev / n
        clamped = int(np.count_nonzero(nrow < -floor))
        np.clip(nrow, 0.0, None, out=nrow)
        info["clamped"].append(clamped)
        core.extend(i, j, c[core.I], r[core.J], r[j])
        if clamped > 0.01 * n:                # :290-292 rebuild from m residual columns
            nrow[:] = 0.0
            for jj in range(m):
                cc = A.apply(_unit(m, jj))
                rc = cc - cols_apply(core.solve(cc[core.I]))
                nrow += np.abs(rc) ** 2
            info["rebuilds"] += 1
        info["total_sq_norms"].append(float(np.sum(nrow)))
        if stop_tol > 0 and info["total_sq_norms"][-1] <= stop_tol ** 2 * total0:
            info["tol_stop"] = True
            break
    info["row_norms"] = nrow
    return core, info
