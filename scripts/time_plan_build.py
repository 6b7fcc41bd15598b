"""build_plan wall time at C4 size (2^20 points per side), best and median of 7."""
import sys
import time

sys.path.insert(0, ".")
from paper_2601_22344_b200 import gen  # noqa: E402
import paper_2601_22344_b200.treebounds as tb  # noqa: E402

x, y, G, B = gen.c4_cauchy_like(0, n=1 << 20, p=1)
ts = []
for _ in range(7):
    t0 = time.perf_counter()
    tb.build_plan(x, y, nu=5.0, leaf_size=32)
    ts.append(time.perf_counter() - t0)
print("build_plan best %.3f s, median %.3f s" % (min(ts), sorted(ts)[3]))
