import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
x, y, G, B = gen.c2_cauchy(0)
M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
for _ in range(3):
    rp.structured_eliminate(M, "rplu", 200, rng=rp.RngState(0), keep_steps=True)
torch.cuda.synchronize()
def t(label, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter()-t0)*1e3:8.2f} ms"); return r
Mh = t("CauchyLikeMatrix(host arrays)", lambda: rp.CauchyLikeMatrix(x, y, G, B, check_points=False))
t("structured_eliminate device-only", lambda: rp.structured_eliminate(M, "rplu", 200, rng=rp.RngState(0)))
t("  ... keep_steps, host_steps=False", lambda: rp.structured_eliminate(M, "rplu", 200, rng=rp.RngState(0), keep_steps=True, host_steps=False))
t("  ... keep_steps host", lambda: rp.structured_eliminate(M, "rplu", 200, rng=rp.RngState(0), keep_steps=True))
t("  ... new matrix, keep_steps host", lambda: rp.structured_eliminate(Mh, "rplu", 200, rng=rp.RngState(0), keep_steps=True))
t("  ... new matrix again", lambda: rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B, check_points=False), "rplu", 200, rng=rp.RngState(0), keep_steps=True))
