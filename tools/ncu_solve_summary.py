"""Summarise an ncu launch list of ONE full solve (tools/one_solve.py CFG) and update
profiles/ncu_summary.json, which bench.py reads for the roofline's flops / traffic per launch.

The launch list must come from
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,\
sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum \
        --clock-control none --csv --log-file X.csv python tools/one_solve.py CFG
(cold-cache, serialised: per-launch SHARES and per-gpi counts are what carry over, not times).

usage: python tools/ncu_solve_summary.py CFG launches.csv out.txt "source note" [T]
Writes a per-kernel table to out.txt and, for the dominant rows kernel:
  rows_fp32_flops_per_gpi  (FADD + FMUL + 2 FFMA thread instructions) / (B L1 L2 T)
  rows_warp_inst_per_gpi   smsp__inst_executed / (B L1 L2 T)
  rows_dram_bytes_per_gpi  (dram read + write) / (B L1 L2 T)
  dense_phase              DRAM GB/s of the rows launches of the first 20 iterations
"""
import csv
import json
import os
import sys
from collections import OrderedDict, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
FLOP_KEYS = {"sm__sass_thread_inst_executed_op_fadd_pred_on.sum": 1,
             "sm__sass_thread_inst_executed_op_fmul_pred_on.sum": 1,
             "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": 2}


def read_launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    hdr = rows[i]
    launches = OrderedDict()
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        ent = launches.setdefault(key, {"kernel": d["Kernel Name"].split("(")[0], "m": {}})
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        ent["m"][d["Metric Name"]] = v * SCALE.get(d.get("Metric Unit", ""), 1.0)
    return list(launches.values())


def main():
    cfg, path, out_txt, note = int(sys.argv[1]), sys.argv[2], sys.argv[3], sys.argv[4]
    from paper_2509_13592_b200 import scenes
    w = scenes.workload(cfg)
    T = int(sys.argv[5]) if len(sys.argv) > 5 else w.iterations
    gpi = w.batch * w.l1 * w.l2 * T
    ls = read_launches(path)
    per = defaultdict(lambda: defaultdict(float))
    count = defaultdict(int)
    for e in ls:
        count[e["kernel"]] += 1
        for k, v in e["m"].items():
            per[e["kernel"]][k] += v
    tot_t = sum(p.get("gpu__time_duration.sum", 0.0) for p in per.values())
    lines = [f"{'kernel':64s} {'launches':>8s} {'mean_us':>9s} {'share':>6s} {'dram_MB/launch':>14s} "
             f"{'fp32_Gflop/launch':>17s} {'warp_inst_M/launch':>18s}"]
    for k in sorted(per, key=lambda k: -per[k].get("gpu__time_duration.sum", 0.0)):
        p, n = per[k], count[k]
        fl = sum(p.get(m, 0.0) * f for m, f in FLOP_KEYS.items())
        lines.append(f"{k[:64]:64s} {n:8d} {p.get('gpu__time_duration.sum', 0) / n:9.2f} "
                     f"{p.get('gpu__time_duration.sum', 0) / max(tot_t, 1e-9):6.3f} "
                     f"{(p.get('dram__bytes_read.sum', 0) + p.get('dram__bytes_write.sum', 0)) / n / 1e6:14.3f} "
                     f"{fl / n / 1e9:17.3f} {p.get('smsp__inst_executed.sum', 0) / n / 1e6:18.3f}")
    rows = [k for k in per if "rows_" in k and ("fista" in k or "admm" in k)]
    top = max(rows, key=lambda k: per[k].get("gpu__time_duration.sum", 0.0))
    p = per[top]
    flops = sum(p.get(m, 0.0) * f for m, f in FLOP_KEYS.items())
    dram = p.get("dram__bytes_read.sum", 0.0) + p.get("dram__bytes_write.sum", 0.0)
    # dense phase: the rows launches of the first 20 iterations (launches per iteration =
    # rows launches / (T + 1): the first forward-only launch per sub-batch is counted too)
    seq = [e for e in ls if e["kernel"] == top]
    per_it = max(1, round(len(seq) / (T + 1)))
    head = seq[: per_it * 21]
    hb = sum(e["m"].get("dram__bytes_read.sum", 0) + e["m"].get("dram__bytes_write.sum", 0) for e in head)
    ht = sum(e["m"].get("gpu__time_duration.sum", 0) for e in head) * 1e-6
    late = seq[-per_it * 100:]
    lt = sum(e["m"].get("gpu__time_duration.sum", 0) for e in late) * 1e-6
    lf = sum(sum(e["m"].get(m, 0.0) * f for m, f in FLOP_KEYS.items()) for e in late)
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    summary[f"cfg{cfg}"] = {
        "rows_kernel": top, "launches": count[top], "rows_mean_us_ncu": p.get("gpu__time_duration.sum", 0) / count[top],
        "rows_fp32_flops_per_gpi": flops / gpi,
        "rows_warp_inst_per_gpi": p.get("smsp__inst_executed.sum", 0.0) / gpi,
        "rows_dram_bytes_per_gpi": dram / gpi,
        "rows_share_serialised": p.get("gpu__time_duration.sum", 0) / max(tot_t, 1e-9),
        "dense_phase": {"iterations": "0-20", "launches": len(head), "gbs": hb / max(ht, 1e-12) / 1e9,
                        "dram_bytes": hb, "seconds_ncu": ht},
        "late_phase_fp32_tflops_ncu": lf / max(lt, 1e-12) / 1e12,
        "gpi_of_solve": gpi, "source": note,
    }
    json.dump(summary, open(summary_path, "w"), indent=1)
    lines.append("")
    lines.append(json.dumps(summary[f"cfg{cfg}"], indent=1))
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
