"""Pageable-host -> device staging rate of rplu_upload (C3-size fp64 array)
against a pinned-host copy, for several staging thread counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_22344_b200 import _device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
a = np.empty((n, n))
a[:] = 1.5          # touch every page
dev = torch.device("cuda", 0)
pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
pin.copy_(torch.from_numpy(a))
out = torch.empty((n, n), dtype=torch.float64, device=dev)
for _ in range(2):
    out.copy_(pin, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
out.copy_(pin, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"pinned copy: {dt * 1e3:.1f} ms = {a.nbytes / dt / 1e9:.1f} GB/s", flush=True)
for th in (4, 8, 12, 16):
    os.environ["RPLU_UPLOAD_THREADS"] = str(th)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = _device.upload(a, dev)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
        ok = bool((t[::4097, ::4097] == 1.5).all())
        del t
    print(f"rplu_upload threads={th}: {best * 1e3:.1f} ms = {a.nbytes / best / 1e9:.1f} GB/s ok={ok}",
          flush=True)
