"""Per-rank step time of the sharded C3 loop at 1/G of the rows.

One GPU cannot run G ranks that wait on one another, so this times what ONE
rank of a G-GPU run computes per pivot step: the sharded delayed-update loop
(captured flush blocks, world-1 NCCL collectives standing in for the G-rank
ones) on a row block of 32768/G rows x 32768 columns, 512 steps.  The pivots
are this block's own (the data differ from a real shard's mid-run state, the
work per step does not).  Strong-scaling projection: t(1) / (t(G) + c) with c
the added latency of the two G-rank collectives per step.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402
from paper_2601_22344_b200.distributed import sharded_eliminate  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
n, k = 32768, 512
A = gen.c3_dense_device(0, n=n, dtype=torch.float64, device=torch.device("cuda", 0))
base = None
for G in (1, 2, 4, 8):
    rows = n // G
    blk = A[:rows].clone()
    for _ in range(3):   # warm: allocator, graph pool, kernel attributes
        sharded_eliminate(blk, 0, rp.PivotRule("rplu", rp.RngState(0)), k, graph=True, update="lazy")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    for _ in range(reps):
        tr = sharded_eliminate(blk, 0, rp.PivotRule("rplu", rp.RngState(0)), k, graph=True,
                               update="lazy")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * tr.steps)
    base = ms if base is None else base
    proj = {c: base / (ms + c * 1e-3) for c in (0, 20, 40)}
    print(f"G={G}: {rows} rows per rank, {ms * 1e3:.1f} us per pivot step "
          f"(includes world-1 collectives); projected speed-up with +0/+20/+40 us of "
          f"collective latency per step: {proj[0]:.2f} / {proj[20]:.2f} / {proj[40]:.2f}",
          flush=True)
    del blk
dist.destroy_process_group()
