"""Summarise an ncu report (--set full or a section list): per profiled launch
the duration, DRAM bytes, pipe utilisation and warp stall reasons, and (when
the report carries source counters, first launch) the SASS opcode split of the
stall samples."""
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
h = raw[0]
want = ("gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active")
units = dict(zip(h, raw[1])) if len(raw) > 1 else {}
for v in raw[2:]:
    d = dict(zip(h, v))
    print(f"== {d.get('Kernel Name', '?')}")
    for name in want:
        if name in d:
            print(f"{name:70s} {d[name]} {units.get(name, '')}")
    st = {name: float(val.replace(",", "")) for name, val in d.items()
          if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued")
          and val not in ("", "n/a")}
    tot = sum(st.values()) or 1
    for name, val in sorted(st.items(), key=lambda x: -x[1])[:8]:
        print(f"  stall {name[33:]:30s} {val / tot:6.1%}")
src = page("source", ("--print-source", "sass"))
if len(src) > 2 and "Warp Stall Sampling (All Samples)" in src[1]:
    hh = src[1]
    rows = [dict(zip(hh, r)) for r in src[2:]]

    def s(d):
        try:
            return float(d["Warp Stall Sampling (All Samples)"] or 0)
        except (ValueError, KeyError):
            return 0.0
    total = sum(s(d) for d in rows) or 1
    groups = {}
    for d in rows:
        parts = d.get("Source", "").split()
        op = parts[0] if parts else ""
        if op.startswith("@") and len(parts) > 1:
            op = parts[1]
        key = op.split(".")[0]
        groups[key] = groups.get(key, 0) + s(d)
    print("  SASS opcode share of stall samples (first launch):",
          ", ".join(f"{k} {v / total:.1%}" for k, v in sorted(groups.items(), key=lambda x: -x[1])[:8]))
