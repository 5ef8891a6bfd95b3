"""Per-kernel totals from an `ncu --metrics gpu__time_duration.sum` launch list."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
agg = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0][-60:]
    t = float(r[14]) / (1000.0 if r[13] == "ns" else 1.0)
    c, s = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {c} | {s:.1f} | {s / c:.2f} | {100 * s / tot:.1f}% |")
