"""Stall breakdown and per-opcode instruction counts of one kernel in an
ncu --set full report (read with ncu -i, no GPU).  usage: ncu_stalls.py REP [cells]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else 16777216
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, r = rows[0], rows[2]
print("time_us", r[h.index("gpu__time_duration.sum")])
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        v = float(r[i] or 0)
        if v >= 0.05:
            print(f"  stall {k[34:-23]:24s} {v:6.2f}")
    if k in ("smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"):
        print(f"  {k} {r[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iS, iE = h.index("Source"), h.index("Instructions Executed")
tot = collections.Counter()
T = 0
for r in rows[2:]:
    ex = int(r[iE] or 0)
    T += ex
    op = r[iS].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    tot[o.split(".")[0]] += ex
print(f"instructions per cell {T * 32 / cells:.1f}")
print("  " + ", ".join(f"{o} {c * 32 / cells:.1f}" for o, c in tot.most_common(24)))
