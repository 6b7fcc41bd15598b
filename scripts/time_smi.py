"""C3 fp64 elimination timing with and without a concurrent nvidia-smi
sampler (-lms 200), alternating, same process."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

A = gen.c3_dense_device(0, n=32768)


def run(k=3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


run(2)
for rep in range(2):
    print(f"no sampler: {run():.1f} ms/run", flush=True)
    for lms in (200, 1000):
        p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits", "-lms", str(lms)],
                             stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        print(f"sampler -lms {lms}: {run():.1f} ms/run", flush=True)
        p.terminate()
        p.wait()
