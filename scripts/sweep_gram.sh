#!/bin/bash
# C3 fp64: Gram-mass delayed updates per flush interval vs the applied-term loop.
python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2601_22344_b200 as rp
from paper_2601_22344_b200 import gen
A = gen.c3_dense_device(0, n=32768)
ref = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512, update="eager")
def run(gram, timed=False):
    return rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(0)), 512, update="lazy",
                        gram_masses=gram, time_kernels=timed)
for gram, blocks in ((True, [8, 12, 16]), (False, [6, 8])):
    for b in blocks:
        os.environ["RPLU_LAZY_BLOCK_GRAM" if gram else "RPLU_LAZY_BLOCK"] = str(b)
        tr = run(gram)
        same = tr.pivots == ref.pivots and torch.equal(tr.U, ref.U) and torch.equal(tr.L, ref.L)
        del tr
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(3):
            tr = run(gram); del tr
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        ks = run(gram, True).kernel_stats
        print(f"gram={gram} b={b:2d} identical_to_eager={same} {512 / ms * 1e3:7.1f} steps/s "
              f"pass {ks['sweep_ms'] / max(1, ks['sweep_launches']):.4f} ms", flush=True)
PY
