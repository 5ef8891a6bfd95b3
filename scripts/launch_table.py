"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
one line per launch (kernel, grid, us)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("sbw::<unnamed>::", "")
            print(f"{name[:48]:48s} {d['Grid Size']:>14s} {float(d['Metric Value']) / 1e3:8.2f}")
