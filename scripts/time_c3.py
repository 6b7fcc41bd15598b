"""C3 per-run timing: plain stream vs per-kernel events vs CUDA graph, and
the per-run fixed cost (512 vs 256 pivots)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = gen.c3_dense_device(0, n=32768)
torch.cuda.synchronize()


def run(k, tk=False, reps=3):
    rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), k, time_kernels=tk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), k, time_kernels=tk)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, tr


mode = os.environ.get("RPLU_GRAPH", "auto")
for k in (256, 512):
    ms, tr = run(k)
    print(f"[{mode}] k={k}: {ms:.2f} ms/run, {k / ms * 1e3:.1f} steps/s", flush=True)
ms, tr = run(512, tk=True)
st = tr.kernel_stats
print(f"[{mode}] k=512 timed: {ms:.2f} ms/run; sweep avg {st['sweep_ms'] / st['sweep_launches']:.4f} ms,"
      f" select total {st['select_ms']:.2f} ms", flush=True)
