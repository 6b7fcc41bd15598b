"""C3 delayed-update loop: steps/s and mean pass time per flush interval b.

    python scripts/sweep_lazy_block.py [f64|f32|c128] [b,b,...] [exact|fused]

exact: the reference's multiply-then-subtract per pending term
(RPLU_LAZY_BLOCK, fused_updates=False; pivots and U checked identical to the
eager loop); fused (default arithmetic): one FMA per term
(RPLU_LAZY_BLOCK_FUSED; pivots identical, U to 1e-12 of its scale)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_22344_b200 as rp  # noqa: E402
from paper_2601_22344_b200 import gen  # noqa: E402

dtn = sys.argv[1] if len(sys.argv) > 1 else "f64"
blocks = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [5, 6, 8, 10, 12, 14, 16]
mode = sys.argv[3] if len(sys.argv) > 3 else "fused"
exact = mode == "exact"
env = "RPLU_LAZY_BLOCK" if exact else "RPLU_LAZY_BLOCK_FUSED"
n = int(os.environ.get("SWEEP_N", "32768"))
steps = int(os.environ.get("SWEEP_STEPS", "512"))
dt = {"f64": torch.float64, "f32": torch.float32, "c128": torch.complex128}[dtn]
A = gen.c3_dense_device(0, n=n, dtype=torch.float64).to(dt)


def run(update, timed=False):
    return rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), steps, update=update,
                        time_kernels=timed, fused_updates=not exact)


ref = run("eager")
refU = ref.U.clone()
pivots_ref = ref.pivots
del ref
scale = float(refU.abs().max())
print(f"{dtn} n={n} steps={steps} mode={mode}", flush=True)
for b in blocks:
    os.environ[env] = str(b)
    tr = run("lazy")
    if exact:
        same = tr.pivots == pivots_ref and torch.equal(tr.U, refU)
    else:
        tol = 1e-5 if dt == torch.float32 else 1e-12
        same = tr.pivots == pivots_ref and float((tr.U - refU).abs().max()) <= tol * scale
    del tr
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(3):
        tr = run("lazy")
        del tr
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 3
    tt = run("lazy", timed=True)
    ks = tt.kernel_stats
    del tt
    print(f"b={b:2d} {'identical' if exact else 'agrees'}={same} {steps / ms * 1e3:8.1f} steps/s  "
          f"run {ms:8.2f} ms  pass {ks['sweep_ms'] / max(1, ks['sweep_launches']):.4f} ms  "
          f"select {ks['select_ms'] / max(1, ks['sweep_launches']):.4f} ms  "
          f"GB/s {ks['sweep_bytes'] / ks['sweep_ms'] / 1e6:.0f}", flush=True)
