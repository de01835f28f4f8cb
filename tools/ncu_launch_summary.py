"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
total and mean device time, share of the profiled total."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    val = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    tot[name] += val * scale
    cnt[name] += 1
grand = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]:10.1f} {tot[k] / cnt[k]:9.2f} {tot[k] / grand:6.3f}")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {grand:10.1f}")
