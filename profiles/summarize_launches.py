"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per kernel)."""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
agg = collections.OrderedDict()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    agg.setdefault(name, []).append(float(r["Metric Value"]) / 1e3)
total = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'sum_us':>9s} {'share':>6s}")
for k, v in agg.items():
    print(f"{k[:70]:70s} {len(v):4d} {sum(v)/len(v):9.1f} {sum(v):9.1f} {sum(v)/total:6.1%}")
