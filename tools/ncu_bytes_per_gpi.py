"""Update profiles/ncu_summary.json with the rows-pass DRAM bytes per grid-point-iteration of
one full solve, from a make_profile_summary launches json of tools/one_solve.py CFG under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`.
usage: python tools/ncu_bytes_per_gpi.py CFG launches.json source-note"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_13592_b200 import scenes

cfg, path, note = int(sys.argv[1]), sys.argv[2], sys.argv[3]
w = scenes.workload(cfg)
st = json.load(open(path))
rows = {k: v for k, v in st.items() if "rows_" in k and ("fista" in k or "admm" in k)}
k, v = max(rows.items(), key=lambda kv: kv[1]["launches"] * kv[1]["mean_us"])
total = (v["dram_read_bytes_mean"] + v["dram_write_bytes_mean"]) * v["launches"]
gpi = w.batch * w.l1 * w.l2 * w.iterations
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
summary = json.load(open(out_path)) if os.path.exists(out_path) else {}
summary[f"cfg{cfg}"] = {"rows_kernel": k, "rows_dram_bytes_per_gpi": total / gpi, "launches": v["launches"],
                        "rows_mean_us_ncu": v["mean_us"], "source": note}
json.dump(summary, open(out_path, "w"), indent=1)
print(cfg, k, total / gpi)
