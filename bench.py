"""Benchmark of the B200 RPLU pivot loop (BASELINE.json metric).

Default workload (N=1): BASELINE configs[2], dense fp64 32768 x 32768, rank
512 — the config the metric's "dense Schur step HBM GB/s vs B200 peak" is
quoted on (configs[0] is the reference's CPU-sized case, configs[1] a
latency-bound Cauchy case; both are parity-test cases).

One bench "step" = one full RPLU run of `rank` pivot steps on the resident
input (eliminate(): copy A into the residual buffer, then the device loop).
value = pivot steps / s over the K timed runs (inputs in HBM, CUDA events);
e2e   = the same metric through the public drop-in call with HOST buffers
        (a plain pageable numpy A in, numpy L/U/pivots out, copies inside the
        region; the pinned-input figure is reported beside it).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                [--config c3f64|c3f32|c1] [--n N] [--rank R]
Under torchrun (N>1) the residual is row-block sharded across ranks
(paper_2601_22344_b200.distributed); rank 0 prints one JSON line.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "c3f64": dict(desc="C3 dense fp64 32768x32768 rank 512 (BASELINE configs[2])",
                  n=32768, rank=512, dtype="f64", seed=0),
    "c3f32": dict(desc="C3 dense fp32 32768x32768 rank 512 (BASELINE configs[2])",
                  n=32768, rank=512, dtype="f32", seed=0),
    "c1": dict(desc="C1 dense fp64 2000x2000 rank 100 (BASELINE configs[0])",
               n=2000, rank=100, dtype="f64", seed=0, kind="c1"),
    "c2": dict(desc="C2 Cauchy c128 4096x4096 p=1 rank 200, exact norms (BASELINE configs[1])",
               n=4096, rank=200, dtype="c128", seed=0, kind="cauchy", p=1),
    "c4": dict(desc="C4 Cauchy-like c128 2^20 x 2^20 p=4 (BASELINE configs[3]); bench step = "
                    "`rank` pivot steps of the rank-256 run",
               n=1 << 20, rank=4, dtype="c128", seed=0, kind="cauchy", p=4),
    "c5": dict(desc="C5 matrix-free Gaussian kernel fp64 2e6 x 2e6 (BASELINE configs[4]); bench "
                    "step = `rank` pivot steps of the rank-1024 cur_build",
               n=2_000_000, rank=2, dtype="f64", seed=0, kind="cur"),
    "c5full": dict(desc="C5-construction matrix-free Gaussian kernel fp64 at n = m = 5e5, the "
                        "full rank-1024 cur_build (BASELINE configs[4] at reduced n: a full "
                        "rank-1024 run at 2e6 is ~1.5 h of K7); bench step = the whole run",
                   n=500_000, rank=1024, dtype="f64", seed=0, kind="cur"),
    "c4plan": dict(desc="C4 Cauchy-like c128 2^20 x 2^20 p=4 rank 256 (BASELINE configs[3]) "
                        "through the certified-bound plan path (build_plan + rejection "
                        "sampling), as every in-package Cauchy caller runs it",
                   n=1 << 20, rank=256, dtype="c128", seed=0, kind="cauchy_plan", p=4),
    "luerr": dict(desc="SURVEY 8(a) a17 / K11: ||A - L U||_F / ||A||_F of the C3 fp64 "
                       "32768^2 rank-512 elimination (FP64 tensor cores, fused); bench step = "
                       "one error evaluation",
                  n=32768, rank=512, dtype="f64", seed=0, kind="luerr"),
    # §8(f4) consumers (not BASELINE configs: supplementary measurement lines)
    "gmres": dict(desc="SURVEY 8(f4) restarted GMRES: one 20-step MGS Arnoldi cycle on n=2^24 "
                       "complex128 (stencil operator); bench step = one restart cycle",
                  n=1 << 24, rank=20, dtype="c128", seed=0, kind="gmres"),
    "bary": dict(desc="SURVEY 8(f4) barycentric evaluation: degree-256 rational at 2^24 points "
                      "(+ one cur_aaa fit on 20000 samples); bench step = one evaluation",
                 n=1 << 24, rank=256, dtype="c128", seed=0, kind="bary"),
}
METRIC = "RPLU pivot steps/sec at rank k; dense Schur step HBM GB/s vs B200 peak"
UNIT = "pivot steps/s"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(cfg, n, lazy_frac_flush=None):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_traffic.json), when it matches; for the
    delayed-update loop the read-pass / flush captures weighted by the timed
    launch mix (lazy_frac_flush = share of flush launches)."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        key = "c3" + cfg["dtype"]
        if lazy_frac_flush is not None:
            e = t.get(key + "_lazy")
            if e and e["n"] == n:
                return ((1.0 - lazy_frac_flush) * e["read_pass_traffic_bytes"]
                        + lazy_frac_flush * e["flush_traffic_bytes"])
            return None
        if key in t and t[key]["n"] == n:
            return t[key]["traffic_bytes"]
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1 or os.environ.get("RPLU_FORCE_SHARDED") == "1":
        import torch.distributed as dist
        backend = os.environ.get("RPLU_DIST_BACKEND", "nccl")
        dist.init_process_group(backend)
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, len(os.sched_getaffinity(0))


def cpu_baseline(A_host, rank, seed, n_steps, threads):
    """Oracle port (TEST INFRASTRUCTURE; timed here as the CPU baseline only):
    `n_steps` pivot steps of the real-fp64 restatement of Alg 1 on the same
    bytes, `threads` host threads over row blocks."""
    import oracle
    t0 = time.perf_counter()
    oracle.eliminate_real(A_host, "rplu", n_steps, seed=seed, threads=threads,
                          block_rows=max(256, A_host.shape[0] // (4 * threads)), copy=False)
    dt = time.perf_counter() - t0
    return n_steps / dt, dt


def run_reference_arm(args, cfg, rank_id):
    """--impl reference: the reference's algorithm on the host cores (oracle
    port; the reference is pure Python/numpy and cannot travel to the box)."""
    if rank_id != 0:
        return
    from paper_2601_22344_b200 import gen
    n, rank = cfg["n"], cfg["rank"]
    model, cores = _cpu_info()
    t0 = time.perf_counter()
    if cfg["n"] <= 4096 and cfg.get("kind") == "c1":
        A = gen.c1_dense(cfg["seed"], n=n)
    else:
        A = gen.c3_dense_host_wy(cfg["seed"], n=n)
    gen_s = time.perf_counter() - t0
    import oracle
    g = oracle.uniform_stream(cfg["seed"])
    dtype = np.float32 if cfg["dtype"] == "f32" else np.float64
    R = A.astype(dtype, copy=False)
    # W warm-up pivot steps, then K timed pivot steps, continuing one elimination
    oracle.eliminate_real(R, "rplu", args.warmup, gen=g, threads=cores, dtype=dtype,
                          block_rows=max(256, n // (4 * cores)), copy=False)
    t0 = time.perf_counter()
    oracle.eliminate_real(R, "rplu", args.steps, gen=g, threads=cores, dtype=dtype,
                          block_rows=max(256, n // (4 * cores)), copy=False)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": cfg["dtype"], "data": "synthetic (seeded, BASELINE construction)",
        "config": {"workload": cfg["desc"], "n": n, "rank": rank, "seed": cfg["seed"],
                   "step": "one pivot step of the full-size elimination (bounded sample)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{args.steps} timed pivot steps after {args.warmup} warm-up "
                                   f"steps at full size n={n} (input build {gen_s:.1f}s untimed); "
                                   f"CPU: {model}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _cauchy_input(cfg):
    from paper_2601_22344_b200 import gen
    if cfg["p"] == 1:
        return gen.c2_cauchy(cfg["seed"], n=cfg["n"])
    return gen.c4_cauchy_like(cfg["seed"], n=cfg["n"], p=cfg["p"])


def run_cauchy_arm(args, cfg):
    """Cauchy-like exact-norm path (structured_eliminate, plan=None)."""
    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _ffi
    torch.cuda.set_device(0)
    n, rank, seed, p = cfg["n"], cfg["rank"], cfg["seed"], cfg["p"]
    x, y, G, B = _cauchy_input(cfg)
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)

    def one_run(tk=False, mat=M):
        return rp.structured_eliminate(mat, "rplu", rank, rng=rp.RngState(seed),
                                       time_kernels=tk)
    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    # small sizes run the resident loop (one cooperative launch) or a
    # graph-captured step loop; K5 durations then come from the resident
    # loop's phase stamps or from a second, per-launch-evented pass
    graphable = float(n) * n * p <= 256.0 * 1024 * 1024
    ev0.record()
    for _ in range(args.steps):
        tr = one_run(not graphable)
        stats.append(tr.kernel_stats)
    ev1.record()
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    launches = sum(s["kernel_launches"] for s in stats)
    resident = graphable and all(s["kernel_launches"] == 2 for s in stats)
    clk = clocks.stop()
    k = tr.rank
    value = args.steps * k / (total_ms / 1e3)
    flops = float(n) * n * (8 * p + 8)
    peak = _ffi.fp64_peak_tflops(0)
    phases = None
    if resident:
        phases = _trace_phases(
            "import sys; sys.path.insert(0, %r); import torch; import bench;"
            "import paper_2601_22344_b200 as rp;"
            "x, y, G, B = bench._cauchy_input(%r);"
            "M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False);"
            "[rp.structured_eliminate(M, 'rplu', %d, rng=rp.RngState(%d)) for _ in range(3)];"
            "torch.cuda.synchronize()" % (REPO, cfg, rank, seed), "resident cauchy loop")
        mass_ms, mass_n = phases.get("masses", float("nan")) * 1e-3, 1
    else:
        if graphable:
            stats = [one_run(True).kernel_stats for _ in range(args.steps)]
        mass_ms = sum(s["masses_ms"] for s in stats)
        mass_n = sum(s["masses_launches"] for s in stats)
    avg_s = mass_ms / mass_n / 1e3
    achieved = flops / avg_s / 1e12
    # e2e: host generators in, host trace out (the reference-facing call);
    # one untimed call first, as for `value` (the kept-steps configuration
    # captures its own CUDA graph on first use)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if float(n) * n * p <= 2.0 ** 28:   # graph-captured sizes (seconds-long runs need none)
        rp.structured_eliminate(rp.CauchyLikeMatrix(x, y, G, B, check_points=False), "rplu",
                                rank, rng=rp.RngState(seed), keep_steps=True)
    torch.cuda.synchronize()
    e0.record()
    Mh = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    trh = rp.structured_eliminate(Mh, "rplu", rank, rng=rp.RngState(seed), keep_steps=True)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    h2d = 16 * (n + n + n * p + n * p)
    d2h = 16 * trh.rank * (2 * n + 1) + 16 * trh.rank + 16 * trh.rank
    # CPU baseline: oracle port, bounded sample of pivot steps on the same bytes
    model, cores = _cpu_info()
    cpu_k = 3 if n > 8192 else 10
    if n > 65536:
        # a full-size oracle step is ~2e4 s: time exact_row_norms on a row
        # sample and extrapolate per step (labelled)
        rows = 64
        t0 = time.perf_counter()
        oracle.exact_row_norms(x[:rows], y, G[:rows], B)
        dt = time.perf_counter() - t0
        cb_v = 1.0 / (dt * n / rows)
        sample = (f"exact_row_norms on {rows} of {n} rows ({dt:.1f}s), extrapolated to one "
                  f"full step (the step is 99.8% row norms); 1 thread (numpy)")
    else:
        t0 = time.perf_counter()
        oracle.structured_eliminate(x, y, G, B, "rplu", cpu_k, seed=seed)
        dt = time.perf_counter() - t0
        cb_v = cpu_k / dt
        sample = f"{cpu_k} pivot steps of the oracle port on the same bytes ({dt:.1f}s)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE construction)",
        "config": {"workload": cfg["desc"], "n": n, "m": n, "p": p, "rank": rank, "seed": seed,
                   "step": f"one structured_eliminate run of {rank} pivot steps",
                   "l2": "generated entries; no matrix in HBM"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": ("cauchy_resident_kernel, mass phase (K5 arithmetic on the CTA's "
                                "resident rows; one cooperative launch per run, latency-bound "
                                "step: see phases_us_per_step)" if resident else
                                "cauchy_mass_kernel (K5 generated-entry row masses)"),
                     "algorithmic_flops_per_launch": flops, "avg_launch_ms": avg_s * 1e3,
                     "peak_source": "measured FP64 DFMA probe (rplu_diag_fp64_peak)",
                     **({"phases_us_per_step": phases,
                         "launch_timing": "CTA 0's globaltimer stamps of the same run in a child "
                                          "process (RPLU_PERSIST_TRACE=1)"} if resident else {})},
        "step_breakdown_ms": {"masses_per_pivot": mass_ms / mass_n,
                              "total_per_pivot": total_ms / (args.steps * k)},
        "cpu_baseline": {"value": cb_v, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": sample + f"; CPU: {model}"},
        "e2e": {"value": trh.rank / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "near_boundary_draws": tr.near_boundary_draws,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def run_cur_arm(args, cfg):
    """Matrix-free CUR path (cur_build on the Gaussian-kernel operator)."""
    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _ffi, gen
    torch.cuda.set_device(0)
    n, rank, seed = cfg["n"], cfg["rank"], cfg["seed"]
    P, Q = gen.c5_points(seed, n=n)
    op = rp.GaussianKernelOperator(P, Q, h=0.1)
    for _ in range(args.warmup):   # (short warm-up builds: a full C5 build is minutes)
        rp.cur_build(op, "rplu-cur", min(rank, 4), rng=rp.RngState(seed))
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gemv = []
    launches0 = _ffi.kernel_launch_count()
    ev0.record()
    for _ in range(args.steps):
        fact, info = rp.cur_build(op, "rplu-cur", rank, rng=rp.RngState(seed), time_gemv=True)
        gemv += info.gemv_ms
    ev1.record()
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    launches = _ffi.kernel_launch_count() - launches0
    clk = clocks.stop()
    k = fact.rank
    value = args.steps * k / (total_ms / 1e3)
    evals = float(n) * n
    # every K7 launch of the run (row norms + one per step) over its launches
    avg_s = sum(gemv) / (len(gemv) + args.steps) / 1e3
    flops_per_eval = 13.0   # 3 sub, 3 mul/fma (d^2), 1 scale, 1 exp, 2 (accumulate)... see DESIGN.md
    achieved = evals * flops_per_eval / avg_s / 1e12
    peak = _ffi.fp64_peak_tflops(0)
    # e2e: host points in, host factorization out
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    oph = rp.GaussianKernelOperator(P, Q, h=0.1)
    facth, infoh = rp.cur_build(oph, "rplu-cur", rank, rng=rp.RngState(seed))
    Wh = facth.core_matrix()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    model, cores = _cpu_info()
    # CPU baseline: one full apply on a row sample, extrapolated to the
    # reference's 6 applies per step (labelled)
    rows = 200
    host = oracle.GaussianKernelHost(P[:rows], Q)
    t0 = time.perf_counter()
    host.apply(np.ones(n))
    dt = time.perf_counter() - t0
    per_apply = dt * n / rows
    cb_v = 1.0 / (6 * per_apply)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE construction)",
        "config": {"workload": cfg["desc"], "n": n, "m": n, "rank": rank, "seed": seed,
                   "step": f"one cur_build run of {rank} pivot steps",
                   "l2": "generated entries; points only in HBM (48 MB per side)"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "gauss_gemv_dot_kernel (K7 full generated GEMV g = A l, dot-product exponent form)",
                     "algorithmic_flops_per_launch": evals * flops_per_eval,
                     "avg_launch_ms": avg_s * 1e3, "evals_per_s": evals / avg_s,
                     "peak_source": "measured FP64 DFMA probe (rplu_diag_fp64_peak)",
                     "note": "13 flop/eval counts exp as one op; an entry costs 14 FP64-pipe instructions "
                             "(4 exponent + 3 reduction + 5 polynomial + scale + accumulate)"},
        "cpu_baseline": {"value": cb_v, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"one Gaussian-kernel apply on {rows} of {n} rows "
                                   f"({dt:.2f}s), extrapolated to the reference's 6 full "
                                   f"applies per step; CPU: {model}"},
        "e2e": {"value": k / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 48 * n,
                "d2h_bytes_per_step": Wh.nbytes + 8 * n},
        "gpu_launches": launches,
        "near_boundary_draws": info.near_boundary_draws,
        "rebuilds": info.rebuilds,
        "non_k7_fraction": 1.0 - (sum(gemv) / args.steps) / (total_ms / args.steps),
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def _supp_line(args, cfg, metric, unit, value, total_ms, roofline, cpu, e2e, launches, clk,
               extra=None):
    line = {"metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic (seeded)",
            "config": {"workload": cfg["desc"], "n": cfg["n"], "seed": cfg["seed"],
                       "l2": "inputs larger than L2"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk}
    line.update(extra or {})
    print(json.dumps(line), flush=True)


def run_gmres_arm(args, cfg):
    """One restart cycle of GMRES (20 MGS Arnoldi steps) at n = 2^24: the
    Krylov basis (21 x 256 MB) streams from HBM; the MGS kernel is timed
    per launch in a second pass against its algorithmic bytes
    (112 + 64 j) * 16 n / 16 ... see DESIGN.md §3."""
    import ctypes

    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _device, _ffi
    torch.cuda.set_device(0)
    n, steps_per = cfg["n"], cfg["rank"]
    g = torch.Generator(device="cuda").manual_seed(cfg["seed"])
    b = torch.complex(torch.randn(n, generator=g, device="cuda", dtype=torch.float64),
                      torch.randn(n, generator=g, device="cuda", dtype=torch.float64))

    @rp.device_callable
    def K(x):     # shifted 1-D Laplacian stencil (the user's operator)
        y = 4.0 * x
        y[1:] -= x[:-1]
        y[:-1] -= x[1:]
        return y

    def cycle(bb):
        return rp.gmres(K, bb, restart=steps_per, tol=1e-300, max_restarts=1)
    for _ in range(args.warmup):
        cycle(b)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _ffi.kernel_launch_count()
    e0.record()
    for _ in range(args.steps):
        res = cycle(b)
    e1.record()
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    launches = _ffi.kernel_launch_count() - launches0
    clk = clocks.stop()
    value = args.steps * res.iterations / (total_ms / 1e3)
    # second pass: the MGS kernel alone, per launch, on the same basis shape
    V = torch.zeros((steps_per + 1, n), dtype=torch.complex128, device="cuda")
    V[0] = b / torch.linalg.vector_norm(b)
    h = torch.zeros(steps_per + 2, dtype=torch.complex128, device="cuda")
    c = _device.ctx(torch.device("cuda", 0))
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ms, byts = [], []
    for j in range(steps_per):
        w = K(V[j]).contiguous()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        _ffi.check(c._lib.rplu_mgs_arnoldi(c.handle, V.data_ptr(), n, j, w.data_ptr(),
                                           V[j + 1].data_ptr(), h.data_ptr(), st))
        a1.record()
        torch.cuda.synchronize()
        ms.append(a0.elapsed_time(a1))
        byts.append((112 + 64 * j) * n)
    peak, peak_src = _peaks()
    achieved = sum(byts) / (sum(ms) / 1e3) / 1e9
    # e2e: host rhs in, host solution out (one cycle)
    bh = b.cpu().numpy()
    e0.record()
    resh = rp.gmres(K, bh, restart=steps_per, tol=1e-300, max_restarts=1)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # CPU baseline: the oracle's MGS GMRES cycle on a 2^20 sample, scaled to n
    ns = 1 << 20
    bs = bh[:ns]
    Kh = lambda x: 4.0 * x - np.concatenate([[0], x[:-1]]) - np.concatenate([x[1:], [0]])  # noqa
    t0 = time.perf_counter()
    oracle.consumers.gmres_mgs(Kh, bs, restart=steps_per, tol=1e-300, max_restarts=1)
    dt = (time.perf_counter() - t0) * n / ns
    model, _ = _cpu_info()
    _supp_line(args, cfg, "GMRES Arnoldi steps/s (MGS, restart 20)", "Arnoldi steps/s", value,
               total_ms,
               {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "mgs_arnoldi_kernel (one cooperative launch per Arnoldi step)",
                "algorithmic_bytes_per_cycle": float(sum(byts)),
                "avg_launch_ms": sum(ms) / len(ms), "peak_source": peak_src},
               {"value": steps_per / dt, "unit": "Arnoldi steps/s", "cores": 1, "kind": "port",
                "sample": f"oracle gmres_mgs cycle on {ns} of {n} unknowns "
                          f"({dt * ns / n:.2f}s), scaled linearly; CPU: {model}"},
               {"value": resh.iterations / (e2e_ms / 1e3), "unit": "Arnoldi steps/s",
                "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 16 * n},
               launches, clk)


def run_luerr_arm(args, cfg):
    """K11 at C3: the fused L.U reconstruction error of the C3 fp64 rank-512
    elimination (2 n m k flop on the FP64 tensor cores), against the measured
    DMMA issue rate; cuBLAS DGEMM L @ U (the unfused product alone) timed
    beside it for reference."""
    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _ffi, errors, gen
    torch.cuda.set_device(0)
    n, k, seed = cfg["n"], cfg["rank"], cfg["seed"]
    A = gen.c3_dense_device(seed, n=n)
    tr = rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(seed)), k)
    L, U = tr.L, tr.U
    del tr
    torch.cuda.empty_cache()
    for _ in range(args.warmup):
        errors.lu_error_sq(A, L, U)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _ffi.kernel_launch_count()
    kms = []
    e0.record()
    for _ in range(args.steps):
        e, a, ms = errors.lu_error_sq(A, L, U)
        kms.append(ms)
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    launches = _ffi.kernel_launch_count() - launches0
    flops = 2.0 * n * n * k
    value = args.steps / (total_ms / 1e3)
    peak = _ffi.dmma_peak_tflops(0)
    achieved = flops / (statistics.mean(kms) / 1e3) / 1e12
    # cuBLAS DGEMM L @ U alone (n x n output written, no subtraction / norm)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.matmul(L, U)
    torch.cuda.synchronize()
    t0.record()
    P = torch.matmul(L, U)
    t1.record()
    torch.cuda.synchronize()
    cublas_ms = t0.elapsed_time(t1)
    del P
    torch.cuda.empty_cache()
    # e2e: pinned host A, L, U in; the scalar error out
    Ah = torch.empty(A.shape, dtype=A.dtype, pin_memory=True)
    Ah.copy_(A)
    Lh, Uh = L.cpu().numpy(), U.cpu().numpy()
    del A
    torch.cuda.empty_cache()
    e0.record()
    err_h = errors.lu_error(Ah.numpy(), Lh, Uh)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # CPU baseline: the oracle's numpy A - L U and norm on a 1024-row sample
    rows = 1024
    t = time.perf_counter()
    oracle.lu_error(Ah.numpy()[:rows], Lh[:rows], Uh)
    cpu_s = (time.perf_counter() - t) * n / rows
    model, _ = _cpu_info()
    _supp_line(args, cfg, "L.U reconstruction error evaluations/s (K11, C3 rank 512)",
               "evaluations/s", value, total_ms,
               {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "lu_error_kernel<double,1> (DMMA m8n8k4, fused subtract + Frobenius)",
                "algorithmic_flops_per_launch": flops, "avg_launch_ms": statistics.mean(kms),
                "peak_source": "measured DMMA issue rate (rplu_diag_dmma_peak)",
                "cublas_dgemm_LU_ms": cublas_ms,
                "cublas_dgemm_tflops": flops / (cublas_ms / 1e3) / 1e12},
               {"value": 1.0 / cpu_s, "unit": "evaluations/s",
                "cores": len(os.sched_getaffinity(0)), "kind": "port",
                "sample": f"oracle.lu_error on {rows} of {n} rows ({cpu_s * rows / n:.2f}s, "
                          f"numpy/OpenBLAS), scaled linearly; CPU: {model}"},
               {"value": 1.0 / (e2e_ms / 1e3), "unit": "evaluations/s",
                "h2d_bytes_per_step": 8 * (n * n + 2 * n * k), "d2h_bytes_per_step": 8},
               launches, clk, extra={"dtype": "f64", "rel_error": float(np.sqrt(e / a)),
                                     "rel_error_e2e": err_h})


def run_bary_arm(args, cfg):
    """Barycentric evaluation kernel (generated Cauchy entries, FP64 pipe)
    at 2^24 points, degree 256; plus one cur_aaa fit as the e2e call."""
    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _ffi
    torch.cuda.set_device(0)
    n, k, seed = cfg["n"], cfg["rank"], cfg["seed"]
    g = np.random.default_rng(seed)
    t = np.exp(2j * np.pi * g.uniform(size=k)) * 1.2
    f = np.exp(t)
    w = g.standard_normal(k) + 1j * g.standard_normal(k)
    r = rp.BarycentricRational(t, f, w)
    zd = torch.complex(torch.rand(n, device="cuda", dtype=torch.float64) * 2 - 1,
                       torch.rand(n, device="cuda", dtype=torch.float64) * 2 - 1)
    for _ in range(args.warmup):
        r.eval_dev(zd)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        r.eval_dev(zd)
    e1.record()
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    per_ms = total_ms / args.steps
    flops = 22.0 * n * k     # 2 sub, |d|^2 (2), reciprocal (1), 2 mul, 2 complex MACs (8+8)... /pair
    achieved = flops / (per_ms / 1e3) / 1e12
    peak = _ffi.fp64_peak_tflops(0)
    # e2e: cur_aaa on 20000 spiral samples (host samples in, host rational out)
    m = 20000
    tt = g.uniform(size=m)
    zs = (0.1 + tt) * np.exp(1j * 4 * np.pi * tt) + 0.01 * (g.standard_normal(m)
                                                          + 1j * g.standard_normal(m))
    S = rp.SampleSet(zs, np.exp(zs) / (zs - 1.7))
    e0.record()
    ra, side = rp.cur_aaa(S, tol=1e-10, rng=rp.RngState(seed), leaf_size=16)
    sup = ra.support
    e1.record()
    torch.cuda.synchronize()
    fit_ms = e0.elapsed_time(e1)
    # CPU: oracle evaluation on a 2^14-point sample, scaled
    ns = 1 << 14
    zh = zd[:ns].cpu().numpy()
    t0 = time.perf_counter()
    oracle.consumers.bary_eval_flagged(t, f, w, zh)
    dt = (time.perf_counter() - t0) * n / ns
    model, _ = _cpu_info()
    _supp_line(args, cfg, "barycentric evaluations/s (degree 256, 2^24 points)", "evaluations/s",
               1e3 / per_ms, total_ms,
               {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": "bary_eval_kernel (generated Cauchy entries, two RHS)",
                "algorithmic_flops_per_launch": flops, "avg_launch_ms": per_ms,
                "peak_source": "measured FP64 DFMA probe (rplu_diag_fp64_peak)",
                "note": "22 flop per (z, t_j) pair, the reciprocal counted as one"},
               {"value": 1.0 / dt, "unit": "evaluations/s", "cores": 1, "kind": "port",
                "sample": f"oracle bary_eval_flagged on {ns} of {n} points, scaled; CPU: {model}"},
               {"value": 1e3 / fit_ms, "unit": "cur_aaa fits/s (20000 samples)",
                "h2d_bytes_per_step": 32 * m, "d2h_bytes_per_step": 16 * len(sup) * 3},
               args.steps, clk, {"cur_aaa": {"degree": int(ra.degree), "side": side,
                                             "ms": fit_ms}})


def run_cauchy_plan_arm(args, cfg):
    """C4 through the plan path: one bench step = one full rank-256
    structured_eliminate(plan=...) on the resident generators (the plan is
    built once, untimed, like the generators)."""
    import warnings

    import torch

    import oracle
    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import _ffi, gen
    torch.cuda.set_device(0)
    n, rank, seed, p = cfg["n"], cfg["rank"], cfg["seed"], cfg["p"]
    x, y, G, B = gen.c4_cauchy_like(seed, n=n, p=p)
    t0 = time.perf_counter()
    plan = rp.build_plan(x, y, nu=5.0)
    plan_s = time.perf_counter() - t0
    M = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    warnings.simplefilter("ignore")
    for _ in range(args.warmup):
        rp.structured_eliminate(M, "rplu", rank, plan=plan, rng=rp.RngState(seed),
                                host_steps=False)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _ffi.kernel_launch_count()
    e0.record()
    for _ in range(args.steps):
        tr = rp.structured_eliminate(M, "rplu", rank, plan=plan, rng=rp.RngState(seed),
                                     host_steps=False)
    e1.record()
    torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    launches = _ffi.kernel_launch_count() - l0
    clk = clocks.stop()
    k = tr.rank
    value = args.steps * k / (total_ms / 1e3)
    # second pass: the certified-bound kernels alone (the step's FP64 work)
    from paper_2601_22344_b200.cauchy import tree_bounds_device
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(10):
        tree_bounds_device(plan, M)
    a1.record()
    torch.cuda.synchronize()
    bounds_ms = a0.elapsed_time(a1) / 10
    tt, st = plan.target_tree, plan.source_tree
    n_agg = sum(len(plan.aggregated[l]) for l in tt.leaves)
    # algorithmic FP64 work of one bound evaluation: source Grams 8 p^2 flop
    # per source point, leaf folds 2 p^2 per aggregated entry, the quadratic
    # form 8 p^2 per target point
    flops = 8.0 * p * p * n + 2.0 * p * p * n_agg + 8.0 * p * p * n
    peak = _ffi.fp64_peak_tflops(0)
    # e2e: host generators in (public call incl. the host plan build), host
    # index lists out
    e0.record()
    Mh = rp.CauchyLikeMatrix(x, y, G, B, check_points=False)
    planh = rp.build_plan(x, y, nu=5.0)
    trh = rp.structured_eliminate(Mh, "rplu", rank, plan=planh, rng=rp.RngState(seed),
                                  host_steps=False)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # CPU: the oracle's restatement of the reference's certified bounds (the
    # reference's plan step is this per-leaf loop plus O(n + m) row work)
    t0 = time.perf_counter()
    oracle.plan.certified_upper_bounds(plan, G, B)
    cpu_s = time.perf_counter() - t0
    model, _ = _cpu_info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE construction)",
        "config": {"workload": cfg["desc"], "n": n, "m": n, "p": p, "rank": rank, "seed": seed,
                   "step": f"one structured_eliminate(plan=...) run of {rank} pivot steps",
                   "plan_build_s": plan_s, "l2": "generated entries; generators only in HBM"},
        "roofline": {"bound": "latency", "achieved": flops / (bounds_ms / 1e3) / 1e12,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / (bounds_ms / 1e3) / 1e12 / peak, "traffic": None,
                     "kernel": "tree Gram + bounds kernels (certified row-norm bounds per step)",
                     "algorithmic_flops_per_launch": flops, "avg_launch_ms": bounds_ms,
                     "peak_source": "measured FP64 DFMA probe (rplu_diag_fp64_peak)",
                     "note": "the plan step is latency bound (draws, host acceptance test); "
                             "bounds are %.0f%% of it" % (100 * bounds_ms * k * args.steps
                                                          / total_ms)},
        "cpu_baseline": {"value": 1.0 / cpu_s, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"one certified-bound evaluation at full size ({cpu_s:.1f}s, "
                                   f"the reference's per-step cost before its O(n+m) row work);"
                                   f" CPU: {model}"},
        "e2e": {"value": k / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 16 * (2 + 2 * p) * n,
                "d2h_bytes_per_step": 16 * k},
        "gpu_launches": launches,
        "near_boundary_draws": tr.near_boundary_draws,
        "proposals": tr.proposals, "acceptances": tr.acceptances,
        "near_tie_acceptances": tr.near_tie_acceptances,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def run_b200_arm(args, cfg, dist, rank_id, world):
    import torch
    if cfg.get("kind") == "cauchy":
        return run_cauchy_arm(args, cfg)
    if cfg.get("kind") == "cur":
        return run_cur_arm(args, cfg)
    if cfg.get("kind") == "cauchy_plan":
        return run_cauchy_plan_arm(args, cfg)
    if cfg.get("kind") == "gmres":
        return run_gmres_arm(args, cfg)
    if cfg.get("kind") == "bary":
        return run_bary_arm(args, cfg)
    if cfg.get("kind") == "luerr":
        return run_luerr_arm(args, cfg)

    import paper_2601_22344_b200 as rp
    from paper_2601_22344_b200 import gen

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, rank, seed = cfg["n"], cfg["rank"], cfg["seed"]
    tdtype = torch.float32 if cfg["dtype"] == "f32" else torch.float64
    esize = 4 if cfg["dtype"] == "f32" else 8

    if dist is not None:
        from paper_2601_22344_b200 import distributed as rdist
        return rdist.bench_sharded(args, cfg, dist, rank_id, world, dev, METRIC, UNIT,
                                   sampler_cls=ClockSampler if rank_id == 0 else None)

    if cfg["n"] <= 4096 and cfg.get("kind") == "c1":
        A = torch.from_numpy(gen.c1_dense(seed, n=n)).to(dev)
    else:
        A = gen.c3_dense_device(seed, n=n, dtype=tdtype, device=dev)
    torch.cuda.synchronize()

    def one_run(time_kernels=False):
        return rp.eliminate(A, rp.PivotRule("rplu", rp.RngState(seed)), rank,
                            compute_dtype=tdtype, time_kernels=time_kernels)

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stats = []
    # The timed region runs the public call as a user would (no per-launch
    # events: small residuals run as one CUDA graph per elimination, and the
    # event records between the ~5 launches of a pivot step would add ~4% at
    # C3).  The per-kernel durations behind `roofline` come from a second
    # pass of the same K runs with CUDA events around every launch on the
    # launching stream.
    graphable = n * n <= 64 * 1024 * 1024
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # a bench step of a small config is `reps` eliminations, so the timed
    # region is long enough (>= ~50 ms) not to be dominated by host noise
    reps = 20 if graphable else 1
    ev0.record()
    for _ in range(args.steps):
        for _ in range(reps):
            tr = one_run()
            stats.append(tr.kernel_stats)
    ev1.record()
    torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    timed_launches = sum(s["kernel_launches"] for s in stats)
    stats = [one_run(time_kernels=True).kernel_stats for _ in range(args.steps)]
    clk = clocks.stop()
    pivots_done = tr.steps
    value = args.steps * reps * pivots_done / (total_ms / 1e3)

    sweep_ms = sum(s["sweep_ms"] for s in stats)
    sweep_n = sum(s["sweep_launches"] for s in stats)
    select_ms = sum(s["select_ms"] for s in stats)
    launches = timed_launches
    # algorithmic bytes of the timed update launches: 2*n*m*s for an eager
    # update or a delayed-update flush, n*m*s for a delayed-update read pass
    sweep_bytes = sum(s.get("sweep_bytes", 0.0) for s in stats)
    lazy_block = stats[-1].get("lazy_block", 0)
    bytes_per_launch = sweep_bytes / sweep_n
    # share of flush launches (read + write R) among the timed update launches
    flush_share = (sweep_bytes / (float(n) * n * esize) - sweep_n) / sweep_n
    avg_s = (sweep_ms / sweep_n) / 1e3
    achieved = sweep_bytes / (sweep_ms / 1e3) / 1e9
    peak, peak_src = _peaks()

    # e2e: public drop-in call with host buffers (pinned numpy in, numpy out)
    host_t = torch.empty((n, n), dtype=tdtype, pin_memory=True)
    host_t.copy_(A)
    A_host = host_t.numpy()
    torch.cuda.synchronize()
    # small configs: `reps` eliminations per timed step as for `value`, so a
    # one-off host allocation (a fresh pinned block while the previous
    # trace is still held) does not dominate a ~10 ms region
    e2e_runs = max(1, min(args.steps, 3)) * reps
    # one untimed call first, as for `value` (host-buffer path: pinned staging
    # buffers and the graph of the new residual address are set up once)
    rp.eliminate(A_host, rp.PivotRule("rplu", rp.RngState(seed)), rank, compute_dtype=tdtype)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_runs):
        tr_h = rp.eliminate(A_host, rp.PivotRule("rplu", rp.RngState(seed)), rank,
                            compute_dtype=tdtype)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_pinned_value = e2e_runs * tr_h.steps / (e2e_ms / 1e3)
    e2e_pinned_ms = e2e_ms
    # the headline e2e: a plain pageable numpy array, as the reference's
    # callers pass (staged through the library's pinned ring, rplu_upload)
    A_page = np.array(A_host)                  # pageable, pages touched here
    rp.eliminate(A_page, rp.PivotRule("rplu", rp.RngState(seed)), rank, compute_dtype=tdtype)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(e2e_runs):
        tr_h = rp.eliminate(A_page, rp.PivotRule("rplu", rp.RngState(seed)), rank,
                            compute_dtype=tdtype)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_value = e2e_runs * tr_h.steps / (e2e_ms / 1e3)
    del A_page
    h2d = n * n * esize
    d2h = tr_h.L.nbytes + tr_h.U.nbytes + 16 * tr_h.steps + 8 * (tr_h.steps + 1)
    same = tr_h.pivots == tr.pivots

    # CPU baseline: oracle port on the same bytes, bounded sample (~10 s of CPU
    # work at C3 size: 24 pivot steps at ~2.2 steps/s on 16 threads)
    model, cores = _cpu_info()
    cpu_steps = min(24 if n > 8192 else 100, rank)
    A64 = A_host.astype(np.float64) if tdtype == torch.float32 else A_host.copy()
    del host_t
    cb_v, cb_dt = cpu_baseline(A64, rank, seed, cpu_steps, cores)
    del A64

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
        "data": "synthetic (seeded BASELINE construction, built on device with cuBLAS)",
        "config": {"workload": cfg["desc"], "n": n, "m": n, "rank": rank, "seed": seed,
                   "step": (f"{reps} full eliminations of {rank} pivot steps" if reps > 1
                            else f"one full elimination of {rank} pivot steps"),
                   "l2": f"inputs larger than L2 ({n * n * esize / 1e9:.1f} GB residual)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": _traffic(cfg, n, flush_share if lazy_block else None),
                     "kernel": ("lazy_pass4_kernel (TMA-fed delayed-update pass + row masses)"
                                if lazy_block else
                                "dense_sweep_kernel (K3 fused Schur update + row masses)"),
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "update": (f"delayed (read R per step, write every {lazy_block} steps)"
                                if lazy_block else "eager (read + write R per step)"),
                     "avg_launch_ms": avg_s * 1e3, "peak_source": peak_src,
                     "launch_timing": (f"CUDA events around every launch on the launching "
                                       f"stream, second pass of the same {args.steps} runs")},
        "step_breakdown_ms": {"sweep_per_pivot": sweep_ms / sweep_n,
                              "select_per_pivot": select_ms / (len(stats) * (pivots_done + 1)),
                              "total_per_pivot": total_ms / (args.steps * reps * pivots_done)},
        "cpu_baseline": {"value": cb_v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{cpu_steps} pivot steps of the oracle real-fp64 port on the "
                                   f"same {n}x{n} bytes ({cb_dt:.1f}s), row blocks over "
                                   f"{cores} threads; CPU: {model}"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "runs": e2e_runs, "ms_per_run": e2e_ms / e2e_runs,
                "input": "pageable numpy array (plain np.array, as a reference caller)",
                "pinned_input_value": e2e_pinned_value,
                "pinned_input_ms_per_run": e2e_pinned_ms / e2e_runs,
                "pivots_match_device_run": same},
        "gpu_launches": launches,
        "near_boundary_draws": tr.near_boundary_draws,
        "clocks": clk,
    }
    if cfg.get("kind") == "c1":
        # C1 is launch/latency bound (the residual lives in shared memory for
        # the whole run): no HBM roofline applies; report the resident
        # kernel's per-phase time instead (CTA 0 timestamps, separate run)
        line["roofline"] = {"bound": "latency", "achieved": None, "peak": None, "unit": "us/step",
                            "frac": None, "traffic": None,
                            "kernel": "dense_resident_kernel (one cooperative launch, R in SMEM)",
                            "us_per_pivot_step": 1e3 * total_ms / (args.steps * reps * pivots_done),
                            "phases_us_per_step": _resident_phases(n, rank, seed)}
    print(json.dumps(line), flush=True)


def _trace_phases(code, marker):
    """Per-phase microseconds printed by a resident loop under
    RPLU_PERSIST_TRACE=1 (CTA 0's globaltimer stamps), from a child process
    running `code` (the trace switch is read once per process)."""
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           timeout=300, env=dict(os.environ, RPLU_PERSIST_TRACE="1"))
        lines = [x for x in r.stderr.splitlines() if marker in x]
        toks = lines[-1].split("):", 1)[1].split()
        out, k = {}, 0
        while k + 1 < len(toks):       # "row cdf 1.40 row find 2.0 ..." -> names with spaces
            j = k
            while j < len(toks):
                try:
                    val = float(toks[j])
                    break
                except ValueError:
                    j += 1
            out[" ".join(toks[k:j])] = val
            k = j + 1
        return out
    except Exception as exc:  # diagnostics only
        return {"error": str(exc)[:200]}


def _resident_phases(n, rank, seed):
    """Per-phase microseconds of the C1 resident loop."""
    code = ("import sys; sys.path.insert(0, %r); import torch; import paper_2601_22344_b200 as rp;"
            "from paper_2601_22344_b200 import gen;"
            "A = torch.from_numpy(gen.c1_dense(%d, n=%d)).cuda();"
            "[rp.eliminate(A, rp.PivotRule('rplu', rp.RngState(%d)), %d) for _ in range(3)];"
            "torch.cuda.synchronize()") % (REPO, seed, n, seed, rank)
    return _trace_phases(code, "resident loop")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3f64", choices=sorted(CONFIGS))
    # (not --n / --rank: torchrun's parser would claim those prefixes)
    ap.add_argument("--size", type=int, default=None, help="override n (= m)")
    ap.add_argument("--pivots", type=int, default=None, help="override the rank k")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.size:
        cfg["n"] = args.size
        cfg["desc"] += f" [n overridden to {args.size}]"
    if args.pivots:
        cfg["rank"] = args.pivots
    dist, rank_id, world = _dist()
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank_id)
    else:
        run_b200_arm(args, cfg, dist, rank_id, world)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
