"""C3 delayed-update run for ncu of the lazy pass: argv[1] = f64|f32|c128,
PROFILE_STEPS steps (default 12) at the flush interval RPLU_LAZY_BLOCK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "f64"
dt = {"f64": torch.float64, "f32": torch.float32, "c128": torch.complex128}[name]
n = int(os.environ.get("PROFILE_N", "32768"))
A = gen.c3_dense_device(0, n=n, dtype=torch.float64).to(dt)
steps = int(os.environ.get("PROFILE_STEPS", "12"))
rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), steps, update="lazy")
torch.cuda.synchronize()
print("profile_lazy ok")
