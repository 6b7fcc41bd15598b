"""Plan-path (certified bounds + rejection sampling) timing at C4 shapes."""
import sys, time, warnings
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
for logn in [int(a) for a in sys.argv[1:]] or [16, 18, 20]:
    n = 1 << logn
    x, y, G, B = gen.c4_cauchy_like(0, n=n, p=4)
    t0 = time.time(); plan = rp.build_plan(x, y, nu=5.0); tp = time.time() - t0
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    rank = 16
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        rp.structured_eliminate(M, "rplu", 2, plan=plan, rng=rp.RngState(0), host_steps=False)
        torch.cuda.synchronize()
        t0 = time.time()
        tr = rp.structured_eliminate(M, "rplu", rank, plan=plan, rng=rp.RngState(0), host_steps=False)
        torch.cuda.synchronize()
        dt = time.time() - t0
    print(f"n=2^{logn} plan build {tp:.2f}s  {rank} steps {dt*1e3:.1f} ms = {rank/dt:.1f} steps/s "
          f"props {tr.proposals} acc {tr.acceptances} fb {tr.exact_fallbacks} ties {tr.near_tie_acceptances}", flush=True)
    # bounds kernel alone
    from paper_2601_22344_b200.cauchy import tree_bounds_device
    torch.cuda.synchronize(); t0 = time.time()
    for _ in range(5):
        u = tree_bounds_device(plan, M)
    torch.cuda.synchronize(); print(f"   tree bounds {(time.time()-t0)/5*1e3:.2f} ms")
