"""C1 e2e breakdown: where the host-buffer eliminate call spends its time
beyond the device-resident loop (pinned H2D, wrapper, copy-back)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

n, rank, seed = 2000, 100, 0
A = torch.from_numpy(gen.c1_dense(seed)).cuda()
host = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
host.copy_(A)
A_host = host.numpy()
torch.cuda.synchronize()


def timed(name, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:40s} dev {e0.elapsed_time(e1) / reps:8.3f} ms  wall "
          f"{(time.perf_counter() - t0) * 1e3 / reps:8.3f} ms", flush=True)


def run(src, **kw):
    return lambda: rp.eliminate(src, rp.PivotRule("rplu", rp.RngState(seed)), rank, **kw)


timed("h2d 32 MB pinned", lambda: host.to("cuda", non_blocking=True))
timed("eliminate device-resident", run(A))
timed("eliminate device, return host", run(A, return_device=False))
timed("eliminate host in, device out", run(A_host, return_device=True))
timed("eliminate host in, host out", run(A_host))



def keep_alive(reps):
    f = run(A_host)
    tr = f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        tr = f()
    e1.record()
    torch.cuda.synchronize()
    print(f"host in/out, trace kept, reps={reps:3d}        dev {e0.elapsed_time(e1) / reps:8.3f} ms  "
          f"wall {(time.perf_counter() - t0) * 1e3 / reps:8.3f} ms", flush=True)
    return tr


for r in (1, 3, 3, 20):
    keep_alive(r)

from torch.profiler import ProfilerActivity, profile  # noqa: E402
f = run(A_host)
f()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        f()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
