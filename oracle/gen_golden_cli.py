"""Generate tests/golden/cli.npz by running the REAL reference CLI (bccblasso.cli.main) in
this container:

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden_cli.py

Stores the files `simulate` writes (byte-exact targets for the package's `simulate`), and
`solve`'s estimate.csv / support.csv for the fast backend of each solver on the reference
test scenario (pkg/tests/test_cli.py:24-38, 117-137), plus the `gram-dump` of its geometry.
"""

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
sys.path.insert(0, REF)

from bccblasso.cli import main  # noqa: E402

SIM = {"m1_count": 8, "m2_count": 6, "element_count": 20, "geometry_seed": 13,
       "targets": [{"f1": -0.25, "f2": 0.25, "re": 2.0, "im": 0.0},
                   {"f1": 0.3125, "f2": -0.375, "re": 0.0, "im": 1.5}],
       "snr_db": 40.0, "noise_seed": 4}
SIM_K = {"m1_count": 10, "m2_count": 6, "element_count": 24, "geometry_seed": 5, "k": 3, "target_seed": 9,
         "noise_variance": 0.01, "noise_seed": 2}
SOLVE = {"l1": 16, "l2": 8, "backend": "fast", "tau_fraction": 0.05, "threshold_fraction": 0.2}
RUNS = {"fista": 400, "ista": 300, "admm": 200}


def main_():
    out = {"sim_config": json.dumps(SIM), "simk_config": json.dumps(SIM_K), "solve_config": json.dumps(SOLVE)}
    with tempfile.TemporaryDirectory() as tmp:
        for tag, cfg in (("sim", SIM), ("simk", SIM_K)):
            path = os.path.join(tmp, f"{tag}.json")
            with open(path, "w") as fh:
                json.dump(cfg, fh)
            assert main(["simulate", "--config", path, "--output-dir", os.path.join(tmp, tag)]) == 0
            for name in ("geometry.json", "targets.csv", "snapshot.csv"):
                with open(os.path.join(tmp, tag, name)) as fh:
                    out[f"{tag}_{name}"] = fh.read()
        for solver, iters in RUNS.items():
            cfg = dict(SOLVE, solver=solver, iterations=iters,
                       geometry_path=os.path.join(tmp, "sim", "geometry.json"),
                       snapshot_path=os.path.join(tmp, "sim", "snapshot.csv"))
            path = os.path.join(tmp, f"solve_{solver}.json")
            with open(path, "w") as fh:
                json.dump(cfg, fh)
            d = os.path.join(tmp, f"out_{solver}")
            assert main(["solve", "--config", path, "--output-dir", d]) == 0
            for name in ("estimate.csv", "support.csv"):
                with open(os.path.join(d, name)) as fh:
                    out[f"{solver}_{name}"] = fh.read()
            out[f"{solver}_iterations"] = iters
        vpath = os.path.join(tmp, "verify.json")
        with open(vpath, "w") as fh:
            json.dump({"m1_count": 8, "m2_count": 6, "element_count": 20, "geometry_seed": 13, "l1": 16, "l2": 8}, fh)
        assert main(["gram-dump", "--config", vpath, "--output", os.path.join(tmp, "omega.csv")]) == 0
        with open(os.path.join(tmp, "omega.csv")) as fh:
            out["gram_dump"] = fh.read()
    np.savez_compressed(os.path.join(OUT, "cli.npz"), **{k: np.array(v) for k, v in out.items()})
    print("cli: done")


if __name__ == "__main__":
    main_()
