"""Per-call timing of C1 eliminate (graph path) to diagnose launch/graph costs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = torch.from_numpy(gen.c1_dense(0)).cuda()
for k in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 100)
    torch.cuda.synchronize()
    print(f"call {k}: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 100, time_kernels=True)
    torch.cuda.synchronize()
    print(f"timed call {k}: {1e3 * (time.perf_counter() - t0):.3f} ms {tr.kernel_stats}", flush=True)
