import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
from paper_2601_22344_b200.cauchy import tree_bounds_device
n = 1 << int(sys.argv[1])
x, y, G, B = gen.c4_cauchy_like(0, n=n, p=4)
plan = rp.build_plan(x, y, nu=5.0)
M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
for _ in range(2):
    tree_bounds_device(plan, M)
torch.cuda.synchronize()
