"""Summarise an ncu --set full report: duration, pipe utilisation, warp
stall reasons, and the SASS stall split (DMMA / LDS / barrier / epilogue)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(kind, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", kind, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
h, v = raw[0], raw[2] if len(raw) > 2 else raw[1]
want = ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active")
for name, val in zip(h, v):
    if name in want:
        print(f"{name:70s} {val}")
st = {name: float(val.replace(",", "")) for name, val in zip(h, v)
      if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued")
      and val not in ("", "n/a")}
tot = sum(st.values()) or 1
for name, val in sorted(st.items(), key=lambda x: -x[1])[:10]:
    print(f"  stall {name[33:]:30s} {val / tot:6.1%}")
src = page("source", ("--print-source", "sass"))
if len(src) > 2:
    hh = src[1]
    rows = [dict(zip(hh, r)) for r in src[2:]]
    def s(d):
        try:
            return float(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            return 0.0
    total = sum(s(d) for d in rows) or 1
    groups = {}
    for d in rows:
        op = d["Source"].split()[0] if d["Source"].split() else ""
        if op.startswith("@"):
            op = d["Source"].split()[1]
        key = op.split(".")[0]
        groups[key] = groups.get(key, 0) + s(d)
    print("  SASS opcode share of stall samples:",
          ", ".join(f"{k} {v / total:.1%}" for k, v in sorted(groups.items(), key=lambda x: -x[1])[:8]))
