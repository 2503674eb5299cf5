"""One-screen summary of an ncu --set full report (section metrics + DRAM bytes + stall reasons)."""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Dynamic Shared Memory Per Block", "Threads", "Grid Size", "Block Size")
out = [title]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(det.splitlines()))
if rows:
    h = rows[0]
    si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        if r[mi] in keep and r[mi] not in seen:
            seen.add(r[mi])
            out.append(f"{r[si][:28]:28s} | {r[mi]:45s} | {r[vi]:>14s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v, u = rows[0], rows[-1], rows[1]
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"):
    if k in h:
        out.append(f"{'raw':28s} | {k:45s} | {v[h.index(k)]:>14s} {u[h.index(k)]}")
st = [(k, float(v[i])) for i, k in enumerate(h)
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
out.append("stall reasons (warps per issue, top 8):")
for k, x in sorted(st, key=lambda t: -t[1])[:8]:
    out.append(f"   {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {x:.3f}")
# a capture of several launches (the split analysis: host pass, device pass, merge): one row each
if len(rows) > 3 and "Kernel Name" in h:
    out.append("per launch:")
    tot = 0
    for r in rows[2:]:
        b = sum(float(r[h.index(k)]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in h)
        tot += b
        d = r[h.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in h else "?"
        out.append(f"   {r[h.index('Kernel Name')][:70]:70s} {d:>12s} {u[h.index('gpu__time_duration.sum')] if 'gpu__time_duration.sum' in h else ''}"
                   f"  dram {b:.4g} {u[h.index('dram__bytes_read.sum')]}")
    out.append(f"   total dram bytes {tot:.6g} {u[h.index('dram__bytes_read.sum')]}")
print("\n".join(out))
