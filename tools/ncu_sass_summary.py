"""Summarise an ncu SASS source-page CSV: opcode mix, stall samples, hottest instructions.

usage: ncu -i X.ncu-rep --page source --csv --print-source=sass > s.csv
       python tools/ncu_sass_summary.py s.csv [kernel-name-substring]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
pick = [x for x in sections if len(sys.argv) < 3 or sys.argv[2] in x["name"]]
for sec in pick[:1]:
    hdr = sec["rows"][0]
    data = [dict(zip(hdr, r)) for r in sec["rows"][1:] if len(r) == len(hdr)]
    num = lambda v: int(v) if v not in ("", "-") else 0  # noqa: E731
    ti = sum(num(d["Instructions Executed"]) for d in data)
    ts = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
    print(sec["name"][:120])
    print(f"warp-instructions {ti}, stall samples {ts}, sass lines {len(data)}")
    ops, samp = Counter(), Counter()
    for d in data:
        toks = d["Source"].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        ops[op] += num(d["Instructions Executed"])
        samp[op] += num(d["Warp Stall Sampling (All Samples)"])
    for op, c in ops.most_common(25):
        print(f"  {op:10s} inst {c:10d} ({100 * c / max(ti, 1):5.1f}%)  stalls {samp[op]:7d} ({100 * samp[op] / max(ts, 1):5.1f}%)")
    print("hottest instructions by stall samples:")
    for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:25]:
        print(f"  {num(d['Warp Stall Sampling (All Samples)']):6d} {d['Address'][-5:]} {d['Source'].strip()[:90]}")
