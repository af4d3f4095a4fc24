"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.
usage: python tools/launch_summary.py launches.csv "command" > profiles/rNN_launches_summary.md"""
import collections
import csv
import sys

path = sys.argv[1]
cmd = sys.argv[2] if len(sys.argv) > 2 else ""
lines = open(path).read().splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
tot = collections.defaultdict(float)
cnt = collections.Counter()
units = set()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    units.add(u)
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(u, 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
grand = sum(tot.values())
print(f"# launch list (ncu --metrics gpu__time_duration.sum --clock-control none)")
print(f"command: `{cmd}`")
print("(cold-cache, serialised launches: compare shares, not absolutes; raw list next to this file)")
print(f"units seen: {sorted(units)}\n")
print("| kernel | launches | total ms | mean ms | share |")
print("|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"| {k} | {cnt[k]} | {v:.2f} | {v / cnt[k]:.3f} | {100 * v / grand:.2f}% |")
