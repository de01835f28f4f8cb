"""Top source lines / SASS of an ncu --page source --csv --print-source=sass,cuda export by
warp-stall samples.  usage: python tools/ncu_source_hot.py file.csv [N]"""
import csv, sys
from collections import defaultdict
path = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
cur_file = None; hdr = None; by_line = defaultdict(lambda: [0, 0, ""]); sass = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8 or not r[0].strip().isdigit():
        continue
    try:
        samp = int(r[4] or 0); inst = int(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    by_line[key][0] += samp; by_line[key][1] += inst
    by_line[key][2] = r[1][:90]
    if r[3]:
        sass.append((samp, r[3][:80], key))
tot = sum(v[0] for v in by_line.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (s, i, src) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100*s/tot:5.1f}%  inst {i:9d}  {f}:{ln:<5d} {src}")
