"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` output."""
import csv
import io
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
top = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
print("total samples", tot)
for r in top:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s:7d} {s/tot:6.1%}  {r['Address'][-5:]}  {r['Source'].strip()[:90]}")
