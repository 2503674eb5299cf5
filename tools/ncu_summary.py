"""One-screen summary of an ncu --set full report (section metrics + DRAM bytes + stall reasons),
one block per captured launch (a split analysis call is three), plus the DRAM total.

    python tools/ncu_summary.py rep.ncu-rep "title" """
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Dynamic Shared Memory Per Block", "Threads", "Grid Size", "Block Size")
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def as_bytes(value, unit):
    return float(value.replace(",", "")) * SCALE[unit]


out = [title]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
drows = list(csv.reader(det.splitlines()))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
dh = drows[0] if drows else []
total = 0.0
for idx, v in enumerate(rows[2:]):
    kid = v[h.index("ID")]
    out.append(f"== launch {kid}: {v[h.index('Kernel Name')][:90]}")
    seen = set()
    if dh:
        si, mi, ui, vi, ii = (dh.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
        for r in drows[1:]:
            if r[ii] == kid and r[mi] in keep and r[mi] not in seen:
                seen.add(r[mi])
                out.append(f"{r[si][:28]:28s} | {r[mi]:45s} | {r[vi]:>14s} {r[ui]}")
    dram = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in h:
            b = as_bytes(v[h.index(k)], u[h.index(k)])
            dram += b
            out.append(f"{'raw':28s} | {k:45s} | {b:>14.6g} byte")
    total += dram
    if "smsp__inst_executed.sum" in h:
        out.append(f"{'raw':28s} | {'smsp__inst_executed.sum':45s} | {v[h.index('smsp__inst_executed.sum')]:>14s} inst")
    st = [(k, float(v[i])) for i, k in enumerate(h)
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    out.append("stall reasons (warps per issue, top 8):")
    for k, x in sorted(st, key=lambda t: -t[1])[:8]:
        out.append(f"   {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {x:.3f}")
if len(rows) > 3:
    out.append(f"== total DRAM bytes over the {len(rows) - 2} launches: {total:.6g}")
print("\n".join(out))
