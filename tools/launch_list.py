"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list: one line per launch."""
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        name = r["Kernel Name"].split("(")[0].replace("hb::", "")
        print(f"{name:54s} {us:10.1f} us")
