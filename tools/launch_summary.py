"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel totals."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0].strip('"') == "ID")
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[ix["Kernel Name"]]
    name = name.replace("xknn::", "").replace("(anonymous namespace)::", "").split("(")[0][:70]
    try:
        v = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    agg.setdefault(name, []).append(v)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = sum(sum(v) for v in agg.values())
print(f"{'total us':>10} {'n':>4} {'avg us':>9} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v)/1e3:10.1f} {len(v):4d} {sum(v)/len(v)/1e3:9.2f} {100*sum(v)/tot:5.1f}%  {k}")
