"""Tiny runs of every device path, for compute-sanitizer (one tool per call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = gen.c1_dense(0, n=150, m=131)
for dt in (None, "float32"):
    rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 20, compute_dtype=dt)
rp.eliminate(A + 1j * A[::-1], rp.PivotRule("rplu", rp.RngState(1)), 10)
rp.eliminate(A, "cplu", 10)
rp.eliminate(A, "c2plu", 10)
x, y, G, B = gen.c4_cauchy_like(0, n=300, m=257, p=3)
rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B), "rplu", 12, rng=rp.RngState(0),
                        keep_steps=True)
P, Q = gen.c5_points(0, n=700, m=500)
rp.cur_build(rp.GaussianKernelOperator(P, Q), "rplu-cur", 8, rng=rp.RngState(0))
rp.sample_index(np.array([0.0, 1.0, 0.0, 2.0]), 0.7)
print("sanitize_small: ok")
