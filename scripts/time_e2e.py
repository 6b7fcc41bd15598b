"""C3 e2e breakdown: pinned H2D bandwidth, device-resident eliminate, host eliminate."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

n = 32768
A = gen.c3_dense_device(0, n=n)
host = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
host.copy_(A)
torch.cuda.synchronize()


def timed(fn, reps=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


dev = torch.empty_like(A)
print("h2d copy_ pinned (ms, wall ms):", timed(lambda: dev.copy_(host, non_blocking=True)), flush=True)
print("h2d .to(cuda) via from_numpy:", timed(lambda: torch.from_numpy(host.numpy()).to("cuda")), flush=True)
print("device eliminate:", timed(lambda: rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512)), flush=True)
An = host.numpy()
print("host eliminate:", timed(lambda: rp.eliminate(An, rp.PivotRule("rplu", rp.RngState(0)), 512)), flush=True)
tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512)
print("d2h Lt,U contiguous:", timed(lambda: (tr.L.T.contiguous().cpu(), tr.U.cpu())), flush=True)

from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    tr = rp.eliminate(An, rp.PivotRule("rplu", rp.RngState(0)), 512)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25), flush=True)
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25), flush=True)
