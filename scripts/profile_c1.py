"""C1 2000^2 fp64 r=100 elimination (persistent loop by default): for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = torch.from_numpy(gen.c1_dense(0)).cuda()
persistent = os.environ.get("PROFILE_STEPWISE") is None
for _ in range(2):
    rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 100, persistent=persistent)
torch.cuda.synchronize()
print("profile_c1 ok")
