"""Average duration per kernel name over the last N launches of an ncu launch-list CSV.

    python scripts/launch_mix.py LAUNCHES.csv [N]
"""
import collections
import csv
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.defaultdict(list)
for r in rows[-n:]:
    agg[r["Kernel Name"][:70]].append(float(r["Metric Value"].replace(",", "")))
unit = rows[0]["Metric Unit"] if rows else "?"
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {k:70s} n={len(v):3d} avg={sum(v) / len(v):9.2f} {unit} share={sum(v) / tot:.2f}")
