"""One K7 generated GEMV (C5 points, n = m = 200000) for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
P, Q = gen.c5_points(0, n=n)
op = rp.GaussianKernelOperator(P, Q)
v = torch.ones(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    op.apply_dev(v, timed=True)
torch.cuda.synchronize()
print("kernel ms", op.last_kernel_ms, "evals/s", n * n / (op.last_kernel_ms / 1e3))
