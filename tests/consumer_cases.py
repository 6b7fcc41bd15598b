"""Shared inputs of the §8(f4) consumer tests (rational / precond goldens).

The banded-plus-low-rank systems are regenerated from the seeded generator
used by tests/golden/make_golden.py (precond_cases), so the goldens only
hold the right-hand sides and outputs."""

import numpy as np
import scipy.linalg as sla

from paper_2601_22344_b200 import gen


def band_system(n, seed):
    """(A, ab, b_inv, K_apply, K_dense): A low-rank-ish dense, B = tridiag(-1, 4, -1)."""
    A = gen.planted_spectrum(n, n, 0.5, seed) * 40.0
    main = np.full(n, 4.0)
    off = np.full(n - 1, -1.0)
    ab = np.zeros((3, n))
    ab[0, 1:], ab[1, :], ab[2, :-1] = off, main, off

    def b_inv(v):
        return sla.solve_banded((1, 1), ab, v)

    def K_apply(v):
        out = A @ v
        out = out + main * v
        out[:-1] += off * v[1:]
        out[1:] += off * v[:-1]
        return out

    K = A + np.diag(main) + np.diag(off, 1) + np.diag(off, -1)
    return A, ab, b_inv, K_apply, K
