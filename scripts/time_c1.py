"""C1 per-elimination timing: persistent loop vs per-step launches (graph)."""
import os
import sys

sys.path.insert(0, os.environ.get("RPLU_TREE", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = torch.from_numpy(gen.c1_dense(0)).cuda()
for persistent in (True, False):
    for _ in range(3):
        rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 100, persistent=persistent)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 100, persistent=persistent)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"persistent={persistent}: {ms:.3f} ms per elimination, {100 / ms * 1e3:.0f} steps/s",
          flush=True)
