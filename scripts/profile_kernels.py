"""Small fixed workloads for ncu captures of each hot kernel (one path per run).

python scripts/profile_kernels.py dense|cauchy|gauss
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

which = sys.argv[1]
if which == "dense":
    A = gen.c3_dense_device(0, n=32768)
    rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 4)
elif which == "cauchy":
    x, y, G, B = gen.c4_cauchy_like(0, n=1 << 17, p=4)
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    rp.structured_eliminate(M, "rplu", 2, rng=rp.RngState(0))
elif which == "gauss":
    P, Q = gen.c5_points(0, n=200_000)
    op = rp.GaussianKernelOperator(P, Q)
    rp.cur_build(op, "rplu-cur", 2, rng=rp.RngState(0))
torch.cuda.synchronize()
print("profile_kernels:", which, "ok")
