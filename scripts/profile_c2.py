"""C2 Cauchy 4096^2 p=1 r=200 structured_eliminate (exact norms): for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

x, y, G, B = gen.c2_cauchy(0, n=4096)
M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
steps = int(os.environ.get("PROFILE_STEPS", "20"))
for _ in range(2):
    rp.structured_eliminate(M, "rplu", steps, rng=rp.RngState(0),
                            time_kernels=os.environ.get("PROFILE_NOGRAPH") is not None)
torch.cuda.synchronize()
print("profile_c2 ok")
