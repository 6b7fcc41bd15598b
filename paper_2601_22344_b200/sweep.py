"""Error-sweep harness on the device — the hot-path methods
of the reference's ``rplu sweep`` (cli.py:100-206).

``sweep_rows(A, methods, ranks, trials, seed)`` returns the reference's row
tuples ``(rank, method, trial_seed, frob_err / ||A||_F, spec_err / ||A||_2,
seconds, applies, adjoints)`` in its order and seeding (trial seeds
``seed ^ trial``; deterministic methods run once and are replicated,
cli.py:119-136), for

* ``rplu`` / ``cplu`` / ``c2plu`` — one ``eliminate`` to the largest rank on
  the device; frob_err = resid_fro[k] (cli.py:150-157), spec_err = the
  20-step power iteration on A - L[:, :k] U[:k] with seed ``tseed ^ (k*1009)``
  (``errors.residual_spectral``, GEMVs on HBM-resident factors);
* ``rplu-cur`` / ``c2plu-cur`` — ``cur_build`` per rank; frob_err =
  ||A - C W^{-1} R||_F by the K11 kernel (cli.py:159-169, _cur_dense
  :200-206), spec_err by power iteration on the CUR residual operator;
* ``svd-oracle`` — the optimal rank-k errors (core.py:66-76).

``applies`` / ``adjoints`` report this implementation's own full
O(n m) operator passes (the reference's column counts its CountingAccessor
calls, 4 applies + 2 adjoints per CUR step, which the device path does not
make).  The PSD / QR / randomized-SVD methods of the sweep are outside the
hot path and raise CapabilityError.

``seed_statistics`` is the 30-seed ||A - LU||_F / ||A||_F protocol of
SURVEY §8(d) on the device (K11 per seed).
"""

import time

import numpy as np
import torch

from . import _device, errors
from .accessors import CapabilityError, DenseMatrix
from .dense_pivots import PivotRule, eliminate
from .lowmem_cur import cur_build
from .rng import RngState

__all__ = ["SWEEP_METHODS", "sweep_rows", "seed_statistics", "results_csv"]

SWEEP_METHODS = ("rplu", "cplu", "c2plu", "rplu-cur", "c2plu-cur", "svd-oracle")
_DENSE = ("rplu", "cplu", "c2plu")
_DETERMINISTIC = ("cplu", "c2plu", "svd-oracle")          # cli.py:41 (hot-path subset)
_OUT_OF_SCOPE = ("rpcholesky", "srplu", "cpqr", "rpqr", "rsvd")
RESULT_HEADER = ("rank", "method", "seed", "frob_err", "spec_err", "seconds", "applies",
                 "adjoints")


def _spectral(apply, apply_h, m, seed, iters=20, dev=None):
    """The reference's power iteration (cli.py:86-99) for an operator given
    by device applies; start vector RngState(seed).complex_normal(m)."""
    v0 = RngState(seed).complex_normal(m)
    v0 = v0 / np.linalg.norm(v0)
    v = torch.from_numpy(v0).to(dev)
    est = 0.0
    for _ in range(iters):
        w = apply_h(apply(v))
        est = float(torch.linalg.norm(w))
        if est == 0.0:
            return 0.0
        v = w / est
    return float(np.sqrt(est))


def _cur_errors(Ad, fact, seed):
    """(||A - C W^{-1} R||_F, ||.||_2) for a CUR skeleton over a dense A."""
    ef, _ = errors.cur_error(Ad, fact)
    if fact.rank == 0:
        Ac = Ad.to(torch.complex128)
        return ef, _spectral(lambda x: Ac @ x, lambda y: Ac.conj().T @ y, Ad.shape[1], seed,
                             dev=Ad.device)
    dev = Ad.device
    Ac = Ad.to(torch.complex128)
    I = torch.as_tensor(list(fact.row_indices), dtype=torch.int64, device=dev)
    J = torch.as_tensor(list(fact.col_indices), dtype=torch.int64, device=dev)
    C, R = Ac[:, J], Ac[I, :]
    M = fact.core_solve_block(R).to(torch.complex128)        # W^{-1} R, k x m

    def apply(x):
        return Ac @ x - C @ (M @ x)

    def apply_h(y):
        return Ac.conj().T @ y - M.conj().T @ (C.conj().T @ y)
    return ef, _spectral(apply, apply_h, Ad.shape[1], seed, dev=dev)


def _run_method(Ad, method, ranks, kmax, tseed):
    """Per-rank (frob_err, spec_err, applies, adjoints), unnormalized
    (cli.py:140-198 for the hot-path methods)."""
    out = []
    if method in _DENSE:
        rule = PivotRule(method, RngState(tseed)) if method == "rplu" else PivotRule(method)
        tr = eliminate(Ad, rule, kmax)
        for k in ranks:
            steps = min(k, tr.steps)
            ef = float(tr.resid_fro[steps])
            es = errors.residual_spectral(Ad, tr.L[:, :steps], tr.U[:steps], tseed ^ (k * 1009))
            out.append((ef, es, 0, 0))
        return out
    if method in ("rplu-cur", "c2plu-cur"):
        D = DenseMatrix.__new__(DenseMatrix)      # wrap the device matrix without a copy
        D.tensor, D.shape = Ad, tuple(Ad.shape)
        for k in ranks:
            rng = RngState(tseed) if method == "rplu-cur" else None
            fact, info = cur_build(D, method, k, rng=rng)
            ef, es = _cur_errors(Ad, fact, tseed ^ (k * 1009))
            out.append((ef, es, fact.rank + info.rebuilds * Ad.shape[1], 0))
        return out
    if method == "svd-oracle":
        for k in ranks:
            ef, es = errors.truncated_svd_error(Ad, k)
            out.append((ef, es, 0, 0))
        return out
    raise ValueError(f"unhandled method {method!r}")


def sweep_rows(A, methods, ranks, trials, seed):
    """One row per (method, rank, trial) in the reference's order and seeding
    (cli.py:100-138), errors normalised by ||A||_F and ||A||_2."""
    if isinstance(methods, str):
        methods = methods.split(",")
    ranks = [int(k) for k in ranks]
    for mth in methods:
        if mth in _OUT_OF_SCOPE:
            raise CapabilityError(f"sweep method {mth!r} is outside the B200 RPLU hot path")
        if mth not in SWEEP_METHODS:
            raise ValueError(f"unknown sweep method {mth!r}")
    if isinstance(A, DenseMatrix):
        Ad = A.tensor
    else:
        Ad = _device.as_device_matrix(A)
    kmax = max(ranks)
    n, m = Ad.shape
    if kmax > min(n, m):
        raise ValueError(f"max rank {kmax} exceeds min(n, m) = {min(n, m)}")
    Ac = Ad if Ad.is_complex() else Ad.to(torch.float64)
    fro0 = float(torch.linalg.norm(Ac))
    spec0 = float(torch.linalg.matrix_norm(Ac, ord=2))
    rows = []
    for method in methods:
        n_trials = 1 if method in _DETERMINISTIC else trials
        for trial in range(n_trials):
            tseed = seed ^ trial
            torch.cuda.synchronize(Ad.device)
            t0 = time.perf_counter()
            per_rank = _run_method(Ad, method, ranks, kmax, tseed)
            torch.cuda.synchronize(Ad.device)
            elapsed = time.perf_counter() - t0
            for k, (ef, es, na, nat) in zip(ranks, per_rank):
                rows.append((k, method, tseed, ef / fro0, es / spec0, elapsed / len(ranks), na,
                             nat))
        if method in _DETERMINISTIC and trials > 1:
            base = rows[-len(ranks):]
            for trial in range(1, trials):
                for (k, mth, _s, ef, es, sec, na, nat) in base:
                    rows.append((k, mth, seed ^ trial, ef, es, sec, na, nat))
    rows.sort(key=lambda r: (methods.index(r[1]), r[0], r[2]))
    return rows


def results_csv(rows):
    """The rows in the reference's results format (io.py:361-370, header
    and number formatting), without the config echo."""
    lines = [",".join(RESULT_HEADER)]
    for (k, mth, sd, ef, es, sec, na, nat) in rows:
        lines.append(f"{int(k)},{mth},{int(sd)},{ef:.17g},{es:.17g},{sec:.6f},{int(na)},{int(nat)}")
    return "\n".join(lines) + "\n"


def seed_statistics(make_input, seeds, rank, rule="rplu"):
    """||A - L U||_F / ||A||_F over seeds (SURVEY §8(d) protocol): one
    eliminate and one K11 evaluation per seed on the device.  ``make_input``
    maps a seed to the (host or device) matrix.  Returns (errors, stats)."""
    errs = []
    for s in seeds:
        A = _device.as_device_matrix(make_input(s))
        tr = eliminate(A, PivotRule(rule, RngState(s)) if rule == "rplu" else rule, rank)
        errs.append(errors.lu_error(A, tr.L, tr.U))
    e = np.array(errs)
    return e, {"mean": float(e.mean()), "min": float(e.min()), "max": float(e.max()),
               "std": float(e.std(ddof=1)) if e.size > 1 else 0.0, "seeds": len(e)}
