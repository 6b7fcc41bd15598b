"""C3 fp64 delayed-update run of 12 steps (default flush interval): for ncu of the lazy pass."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

dt = torch.float32 if (len(sys.argv) > 1 and sys.argv[1] == "f32") else torch.float64
A = gen.c3_dense_device(0, n=32768, dtype=dt)
rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 12, update="lazy")
torch.cuda.synchronize()
print("profile_lazy ok")
