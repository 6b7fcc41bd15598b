import sys, warnings, time
import torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
n = 1 << int(sys.argv[1]); rank = int(sys.argv[2])
x, y, G, B = gen.c4_cauchy_like(0, n=n, p=4)
plan = rp.build_plan(x, y, nu=5.0)
M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    rp.structured_eliminate(M, "rplu", 2, plan=plan, rng=rp.RngState(0), host_steps=False)
    torch.cuda.synchronize(); t = time.time()
    tr = rp.structured_eliminate(M, "rplu", rank, plan=plan, rng=rp.RngState(0), host_steps=False)
    torch.cuda.synchronize(); print("wall ms", (time.time() - t) * 1e3)
