"""Write committed text summaries of ncu captures into profiles/.

usage: python tools/make_profile_summary.py <name> <rep-or-csv> [...]
  *.ncu-rep : key metrics, stall reasons, SASS opcode mix of every captured launch
  *.csv     : launch list (gpu__time_duration / dram bytes per kernel, solve average)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def rep_summary(path):
    out = []
    rows = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"kernel: {d['Kernel Name'][:140]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]} {u.get(k, '')}")
        stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        top = sorted(((float(d[k]) if d[k] not in ("", "n/a") else 0.0, k) for k in stall), reverse=True)[:8]
        out.append("  top stall reasons (warps per issue): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, k in top))
    sass = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "source", "--csv", "--print-source=sass"))))
    sec, cur = [], None
    for r in sass:
        if r and r[0] == "Kernel Name":
            cur = [r[1], []]
            sec.append(cur)
        elif cur is not None:
            cur[1].append(r)
    for name, rs in sec[:1]:
        h = rs[0]
        data = [dict(zip(h, x)) for x in rs[1:] if len(x) == len(h)]
        num = lambda v: int(v) if v not in ("", "-") else 0  # noqa: E731
        ti = sum(num(x["Instructions Executed"]) for x in data)
        ops = Counter()
        for x in data:
            t = x["Source"].split()
            if t:
                ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += num(x["Instructions Executed"])
        out.append(f"  SASS lines {len(data)}, warp-instructions {ti}; opcode mix: " +
                   ", ".join(f"{o} {100 * c / max(ti, 1):.1f}%" for o, c in ops.most_common(12)))
    return "\n".join(out)


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[i]
    per = defaultdict(lambda: defaultdict(list))
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(d.get("Metric Unit", ""), 1.0)
        per[d["Kernel Name"].split("(")[0]][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")) * scale)
    lines, stats = [], {}
    tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
    lines.append(f"{'kernel':64s} {'launches':>8s} {'mean_us':>9s} {'share':>6s} {'dram_rd_MB/launch':>18s} {'dram_wr_MB/launch':>18s}")
    for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
        t = m.get("gpu__time_duration.sum", [0])
        rd = m.get("dram__bytes_read.sum", [0])
        wr = m.get("dram__bytes_write.sum", [0])
        lines.append(f"{k[:64]:64s} {len(t):8d} {sum(t) / len(t):9.2f} {sum(t) / max(tot, 1e-9):6.3f} "
                     f"{sum(rd) / len(rd) / 1e6:18.3f} {sum(wr) / len(wr) / 1e6:18.3f}")
        stats[k] = {"launches": len(t), "mean_us": sum(t) / len(t), "dram_read_bytes_mean": sum(rd) / len(rd),
                    "dram_write_bytes_mean": sum(wr) / len(wr)}
    return "\n".join(lines), stats


if __name__ == "__main__":
    name = sys.argv[1]
    text, stats = [], {}
    for src in sys.argv[2:]:
        text.append(f"==== {os.path.basename(src)}")
        if src.endswith(".ncu-rep"):
            text.append(rep_summary(src))
        else:
            t, st = launches_summary(src)
            text.append(t)
            stats.update(st)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{name}.txt"), "w").write("\n".join(text) + "\n")
    if stats:
        json.dump(stats, open(os.path.join(ROOT, "profiles", f"{name}_launches.json"), "w"), indent=1)
    print("\n".join(text))
