"""Per-source-line totals from an ncu report's source page (``--print-source cuda,sass``):
instructions executed and warp-stall samples, top lines first.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top]"""
import csv
import sys

rows = []
fname = None
with open(sys.argv[1]) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0] and r[0].isdigit():   # a source line with its aggregated metrics
            try:
                rows.append((fname, int(r[0]), r[1].strip()[:80], int(r[4]), int(r[7])))
            except (ValueError, IndexError):
                pass
tot_s = sum(x[3] for x in rows) or 1
tot_i = sum(x[4] for x in rows) or 1
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print(f"total stall samples {tot_s}, instructions {tot_i}")
print("-- by stall samples")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[3] / tot_s:6.1%} {x[4] / tot_i:6.1%}  {x[0]}:{x[1]:<5} {x[2]}")
print("-- by instructions")
for x in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{x[3] / tot_s:6.1%} {x[4] / tot_i:6.1%}  {x[0]}:{x[1]:<5} {x[2]}")
