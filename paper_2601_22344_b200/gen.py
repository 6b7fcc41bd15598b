"""Seeded synthetic inputs for the BASELINE.json configurations (C1..C5).

The reference ships no datasets for this path; BASELINE.json describes each
input in words and SURVEY §8(d) fixes the concrete draw order used here.
Every generator takes a seed, draws from ``RngState(seed)`` (Philox, the
reference's stream) on the host, and returns numpy arrays, so the oracle and
the GPU consume the same bytes.  The large configs have device-side builders
(``*_device``) that reproduce the same construction with torch GEMMs on the
GPU (input construction only; not part of any timed region).
"""

import numpy as np

from .rng import RngState


def _blas_threads(k):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=k, user_api="blas")
    except ImportError:  # pragma: no cover - threadpoolctl ships with the image
        import contextlib
        return contextlib.nullcontext()

__all__ = ["c1_dense", "c2_cauchy", "c3_householder", "c3_dense_host", "c3_dense_host_wy",
           "c3_dense_device",
           "c4_cauchy_like", "c5_points", "planted_spectrum"]


def c1_dense(seed, n=2000, m=None):
    """C1: A = Q1 diag(sigma) Q2^T, Q from numpy QR of Gaussian matrices,
    sigma_i = 10^(-i/40), i = 1..min(n,m) (BASELINE configs[0])."""
    m = n if m is None else m
    g = RngState(seed)
    # LAPACK's blocked QR splits its panels by BLAS thread count: pin it to the
    # 8 threads of the container that recorded the reference runs, so the
    # input bytes (and the reference's recorded pivots) are reproduced on any
    # host (measured: 16 threads on the GPU box give different bytes).
    with _blas_threads(8):
        Q1 = np.linalg.qr(g.standard_normal((n, n)))[0]
        Q2 = np.linalg.qr(g.standard_normal((m, m)))[0]
        r = min(n, m)
        s = 10.0 ** (-np.arange(1, r + 1) / 40.0)
        return (Q1[:, :r] * s) @ Q2[:, :r].T


def c2_cauchy(seed, n=4096, m=None, cluster_frac=0.2):
    """C2: p=1 Cauchy matrix 1/(x_i - y_j); x, y on two interleaved
    Archimedean spirals (radius 0.1+t, angle 4*pi*t (+pi for y), jitter
    0.01 per real component) plus a Gaussian cluster (0.05 per component)
    holding 20% of the points.  Draw order: x-spiral, x-cluster, y-spiral,
    y-cluster; within each block t (spiral only), then real noise, then
    imaginary noise.  Returns (x, y, G, B) with G = ones(n,1), B = ones(1,m).
    """
    m = n if m is None else m
    g = RngState(seed)

    def points(k, phase):
        kc = int(round(cluster_frac * k))
        ks = k - kc
        t = g.uniforms(ks)
        nr = g.standard_normal(ks)
        ni = g.standard_normal(ks)
        spiral = (0.1 + t) * np.exp(1j * (4 * np.pi * t + phase)) + 0.01 * (nr + 1j * ni)
        cr = g.standard_normal(kc)
        ci = g.standard_normal(kc)
        cluster = 0.05 * (cr + 1j * ci)
        return np.concatenate([spiral, cluster])

    x = points(n, 0.0)
    y = points(m, np.pi)
    G = np.ones((n, 1), dtype=np.complex128)
    B = np.ones((1, m), dtype=np.complex128)
    return x, y, G, B


def c3_householder(seed, n=32768, m=None, reflectors=64):
    """Reflector vectors V1 (k x n), V2 (k x m) and sigma_i = 0.98^i for C3."""
    m = n if m is None else m
    g = RngState(seed)
    V1 = g.standard_normal((reflectors, n))
    V2 = g.standard_normal((reflectors, m))
    s = 0.98 ** np.arange(1, min(n, m) + 1)
    return V1, V2, s


def _apply_reflectors_left(V, M):
    # Q M with Q = H_1 H_2 ... H_k, H_t = I - 2 v v^T / |v|^2: apply H_k first.
    for t in range(V.shape[0] - 1, -1, -1):
        v = V[t]
        M -= np.outer(v, (2.0 / (v @ v)) * (v @ M))
    return M


def c3_dense_host(seed, n=4096, m=None, reflectors=64, dtype=np.float64):
    """C3 at desk size on the host: A = Q1 diag(sigma) Q2^T (Householder products)."""
    m = n if m is None else m
    V1, V2, s = c3_householder(seed, n, m, reflectors)
    r = min(n, m)
    M = np.zeros((n, m))
    M[np.arange(r), np.arange(r)] = s
    M = _apply_reflectors_left(V1, M)              # Q1 Sigma
    M = _apply_reflectors_left(V2, M.T.copy()).T  # (Q2 (Q1 Sigma)^T)^T = Q1 Sigma Q2^T
    return np.ascontiguousarray(M, dtype=dtype)


def _wy_factor(V):
    """Compact-WY factor T of Q = H_1 ... H_k = I - Y T Y^T, Y = V^T
    (LAPACK larft forward recurrence, tau_t = 2/|v_t|^2)."""
    G = V @ V.T
    k = V.shape[0]
    tau = 2.0 / np.diag(G)
    T = np.zeros((k, k))
    for t in range(k):
        T[t, t] = tau[t]
        if t:
            T[:t, t] = -tau[t] * (T[:t, :t] @ G[:t, t])
    return T


def c3_dense_host_wy(seed, n=32768, m=None, reflectors=64, dtype=np.float64, block_rows=4096):
    """C3 on the host with BLAS (compact WY, row-blocked); the same
    construction as c3_dense_device, for the CPU baseline at full size."""
    m = n if m is None else m
    V1, V2, s = c3_householder(seed, n, m, reflectors)
    T1, T2 = _wy_factor(V1), _wy_factor(V2)
    r = min(n, m)
    # A = Q1 S Q2^T; Q1 S = S - V1^T T1 (V1 S) where V1 S only touches r columns
    W1 = T1 @ (V1[:, :r] * s)                  # k x r : T1 V1 S
    A = np.zeros((n, m), dtype=np.float64)
    A[np.arange(r), np.arange(r)] = s
    A[:, :r] -= V1.T @ W1
    # A <- A - ((A V2^T) T2^T) V2, in row blocks to bound temporaries
    for lo in range(0, n, block_rows):
        hi = min(lo + block_rows, n)
        blk = A[lo:hi]
        blk -= ((blk @ V2.T) @ T2.T) @ V2
    return A.astype(dtype, copy=False)


def c3_dense_device(seed, n=32768, m=None, reflectors=64, dtype=None, device="cuda"):
    """C3 built on the GPU with the compact-WY form (torch/cuBLAS, fp64).

    Q = I - V^T T V with T from the reflector Gram matrix; A = Q1 S Q2^T
    formed as two rank-64 corrections of the diagonal.  Input construction
    only (not timed).
    """
    import torch
    m = n if m is None else m
    V1, V2, s = c3_householder(seed, n, m, reflectors)
    dev = torch.device(device)

    def wy(V):
        return torch.from_numpy(V).to(dev), torch.from_numpy(_wy_factor(V)).to(dev)

    V1t, T1 = wy(V1)
    V2t, T2 = wy(V2)
    r = min(n, m)
    A = torch.zeros((n, m), dtype=torch.float64, device=dev)
    sd = torch.from_numpy(s).to(dev)
    A[torch.arange(r, device=dev), torch.arange(r, device=dev)] = sd
    # A <- Q1 A = A - V1^T (T1 (V1 A))
    A -= V1t.T @ (T1 @ (V1t @ A))
    # A <- A Q2^T = A - ((A V2^T) T2^T) V2
    A -= ((A @ V2t.T) @ T2.T) @ V2t
    if dtype is not None and dtype != torch.float64:
        A = A.to(dtype)
    return A


def c4_cauchy_like(seed, n=1 << 20, m=None, p=4):
    """C4: x = e^{2 pi i u} (unit circle), y = 1.5 e^{2 pi i u}, G n x p and
    B p x m unit-variance complex Gaussian (BASELINE configs[3])."""
    m = n if m is None else m
    g = RngState(seed)
    x = np.exp(2j * np.pi * g.uniforms(n))
    y = 1.5 * np.exp(2j * np.pi * g.uniforms(m))
    G = g.complex_normal((n, p))
    B = g.complex_normal((p, m))
    return x, y, G, B


def c5_points(seed, n=2_000_000, m=None):
    """C5: Gaussian-kernel points. P uniform in [0,1]^3 (n x 3); Q from a
    3-component mixture with means uniform in [0,1]^3 and sigma 0.08 (m x 3).
    A_ij = exp(-|p_i - q_j|^2 / (2 * 0.1^2))."""
    m = n if m is None else m
    g = RngState(seed)
    P = g.uniforms((n, 3))
    mu = g.uniforms((3, 3))
    comp = np.floor(3 * g.uniforms(m)).astype(np.int64)
    Q = mu[comp] + 0.08 * g.standard_normal((m, 3))
    return P, Q


def planted_spectrum(n, m, rho, seed):
    """Complex dense matrix with singular values rho**j (the reference's
    io.planted_spectrum family, io.py:126-132), for desk-scale tests."""
    g = RngState(seed)
    r = min(n, m)
    s = rho ** np.arange(1, r + 1)

    def unitary(k):
        q, rr = np.linalg.qr(g.complex_normal((k, k)))
        return q * (np.diag(rr) / np.abs(np.diag(rr)))

    with _blas_threads(8):     # input bytes independent of the host's thread count
        U = unitary(n)[:, :r]
        V = unitary(m)[:, :r]
        return (U * s) @ V.conj().T
