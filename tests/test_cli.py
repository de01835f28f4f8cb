"""CLI drop-in (python -m paper_2509_13592_b200): the reference CLI's behaviour and file
formats (pkg/tests/test_cli.py), checked against fixtures made by running the REAL reference
CLI (oracle/gen_golden_cli.py -> tests/golden/cli.npz).

CPU: config parsing, overrides, simulate (byte-identical files), text formats.
GPU: solve / verify / gram-dump through the CUDA path.
"""

import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import bccb_oracle as orc
from paper_2509_13592_b200 import arrays, textio
from paper_2509_13592_b200.cli import (
    apply_overrides,
    main,
    parse_config,
    read_eigenvalue_dump,
    serialize_config,
    write_eigenvalue_dump,
)
from paper_2509_13592_b200.errors import ConfigError


@pytest.fixture(scope="module")
def gold():
    g = load_golden("cli")
    return {k: (v.item() if v.shape == () else v) for k, v in g.items()}


def write_config(path, payload):
    path.write_text(json.dumps(payload, indent=2) + "\n")
    return str(path)


# ----------------------------------------------------------------------------- CPU
def test_config_round_trip_is_idempotent(tmp_path):
    path = tmp_path / "config.json"
    write_config(path, {"b": [1, 2], "a": {"x": 1.5}})
    once = serialize_config(parse_config(path))
    (tmp_path / "again.json").write_text(once)
    assert serialize_config(parse_config(tmp_path / "again.json")) == once


def test_parse_config_errors(tmp_path):
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(ConfigError):
        parse_config(tmp_path / "bad.json")
    (tmp_path / "array.json").write_text("[1, 2]\n")
    with pytest.raises(ConfigError):
        parse_config(tmp_path / "array.json")


def test_apply_overrides():
    assert apply_overrides({"a": 1}, ["a=2", "values=[1,2]", "name=fista"]) == {"a": 2, "values": [1, 2],
                                                                                 "name": "fista"}
    with pytest.raises(ConfigError):
        apply_overrides({}, ["novalue"])


@pytest.mark.parametrize("tag", ["sim", "simk"])
def test_simulate_files_identical_to_reference(tmp_path, gold, tag, capsys):
    config = write_config(tmp_path / "c.json", json.loads(gold[f"{tag}_config"]))
    assert main(["simulate", "--config", config, "--output-dir", str(tmp_path / "o")]) == 0
    for name in ("geometry.json", "targets.csv", "snapshot.csv"):
        assert (tmp_path / "o" / name).read_text() == gold[f"{tag}_{name}"], name
    capsys.readouterr()


def test_simulate_config_errors(tmp_path, gold, capsys):
    sim = json.loads(gold["sim_config"])
    assert main(["simulate", "--config", write_config(tmp_path / "c1.json", dict(sim, k=2, target_seed=1)),
                 "--output-dir", str(tmp_path)]) == 1
    assert "targets" in capsys.readouterr().err
    missing = {k: v for k, v in sim.items() if k != "m1_count"}
    assert main(["simulate", "--config", write_config(tmp_path / "c2.json", missing),
                 "--output-dir", str(tmp_path)]) == 1
    assert "m1_count" in capsys.readouterr().err
    assert main(["simulate", "--config", write_config(tmp_path / "c3.json", dict(sim, noise_variance=0.1)),
                 "--output-dir", str(tmp_path)]) == 1
    assert main(["simulate", "--config", str(tmp_path / "nope.json"), "--output-dir", str(tmp_path)]) == 1
    assert "error" in capsys.readouterr().err


def test_text_formats_round_trip_bitwise(tmp_path):
    rng = np.random.default_rng(3)
    v = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    textio.write_complex_vector(tmp_path / "v.csv", v)
    np.testing.assert_array_equal(textio.read_complex_vector(tmp_path / "v.csv"), v)
    geom = arrays.subsample_preserving_aperture(arrays.make_ura(8, 6), 20, seed=13)
    arrays.save_geometry(tmp_path / "g.json", geom)
    np.testing.assert_array_equal(arrays.load_geometry(tmp_path / "g.json").occupancy, geom.occupancy)


def test_eigenvalue_dump_helpers(tmp_path, gold):
    class Op:   # duck-typed operator (l1, l2, eigenvalues), no device needed
        l1, l2 = 16, 8
        eigenvalues = read_eigenvalue_dump_from_text(gold["gram_dump"])[2]
    write_eigenvalue_dump(tmp_path / "d.csv", Op)
    assert (tmp_path / "d.csv").read_text() == gold["gram_dump"]
    l1, l2, eig = read_eigenvalue_dump(tmp_path / "d.csv")
    assert (l1, l2) == (16, 8)
    np.testing.assert_array_equal(eig, Op.eigenvalues)


def read_eigenvalue_dump_from_text(text):
    lines = [ln for ln in text.splitlines() if ln.strip()]
    l1, l2 = (int(p) for p in lines[1].split(","))
    vals = np.array([complex(float(a), float(b)) for a, b in (ln.split(",") for ln in lines[3:])])
    return l1, l2, vals.reshape(l1, l2)


# ----------------------------------------------------------------------------- GPU
def _solve_setup(tmp_path, gold, **over):
    sim = write_config(tmp_path / "sim.json", json.loads(gold["sim_config"]))
    assert main(["simulate", "--config", sim, "--output-dir", str(tmp_path / "data")]) == 0
    cfg = dict(json.loads(gold["solve_config"]), geometry_path=str(tmp_path / "data" / "geometry.json"),
               snapshot_path=str(tmp_path / "data" / "snapshot.csv"))
    cfg.update(over)
    return write_config(tmp_path / "solve.json", cfg)


def _csv_vector(text):
    rows = [r.split(",") for r in text.splitlines()[1:] if r]
    return np.array([complex(float(a), float(b)) for a, b in rows])


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["fista", "ista", "admm"])
def test_solve_matches_reference_cli(tmp_path, gold, solver, capsys):
    config = _solve_setup(tmp_path, gold, solver=solver, iterations=int(gold[f"{solver}_iterations"]))
    out = tmp_path / "sol"
    assert main(["solve", "--config", config, "--output-dir", str(out)]) == 0
    stdout = capsys.readouterr().out
    assert f"{solver} (fast backend)" in stdout and "final objective" in stdout
    est = textio.read_complex_vector(out / "estimate.csv")
    ref = _csv_vector(gold[f"{solver}_estimate.csv"])
    assert est.shape == (16 * 8,)
    assert orc.rel_l2(est, ref) < 1e-4
    rows = (out / "support.csv").read_text().splitlines()
    ref_rows = gold[f"{solver}_support.csv"].splitlines()
    assert rows[0] == ref_rows[0] == "f1,f2,re,im,magnitude"
    assert [r.split(",")[:2] for r in rows[1:]] == [r.split(",")[:2] for r in ref_rows[1:]]
    if solver == "fista":
        found = {tuple(float(x) for x in r.split(",")[:2]) for r in rows[1:]}
        assert found == {(-0.25, 0.25), (0.3125, -0.375)}      # planted targets (test_cli.py:140-152)


@pytest.mark.gpu
def test_solve_zero_snapshot_and_errors(tmp_path, gold, capsys):
    config = _solve_setup(tmp_path, gold, solver="fista", iterations=50)
    (tmp_path / "data" / "snapshot.csv").write_text("\n".join(["re,im"] + ["0,0"] * 20) + "\n")
    assert main(["solve", "--config", config, "--output-dir", str(tmp_path / "z")]) == 0
    np.testing.assert_array_equal(textio.read_complex_vector(tmp_path / "z" / "estimate.csv"), np.zeros(128))
    assert (tmp_path / "z" / "support.csv").read_text() == "f1,f2,re,im,magnitude\n"
    for over, needle in (({"solver": "newton"}, "solver"), ({"backend": "regular"}, "backend"),
                         ({"geometry_path": str(tmp_path / "missing.json")}, "error")):
        cfg = _solve_setup(tmp_path, gold, **dict({"solver": "fista", "iterations": 5}, **over))
        assert main(["solve", "--config", cfg, "--output-dir", str(tmp_path)]) == 1
        assert needle in capsys.readouterr().err


VERIFY = {"m1_count": 8, "m2_count": 6, "element_count": 20, "geometry_seed": 13, "l1": 16, "l2": 8}


@pytest.mark.gpu
def test_verify_and_gram_dump(tmp_path, gold, capsys):
    import paper_2509_13592_b200 as bb
    config = write_config(tmp_path / "verify.json", VERIFY)
    dump = tmp_path / "eig.csv"
    assert main(["verify", "--config", config, "--dump-eigenvalues", str(dump)]) == 0
    stdout = capsys.readouterr().out
    assert stdout.count("PASS") == 4 and "FAIL" not in stdout
    op = bb.gram_operator(bb.subsample_preserving_aperture(bb.make_ura(8, 6), 20, seed=13), 16, 8)
    l1, l2, eig = read_eigenvalue_dump(dump)
    assert (l1, l2) == (16, 8)
    np.testing.assert_array_equal(eig, op.eigenvalues)          # 17 digits: lossless
    # the reference's dump is fft2 of the first column: equal to the exact L * 1_s to ~1e-14
    ref = read_eigenvalue_dump_from_text(gold["gram_dump"])[2]
    assert np.abs(eig - ref).max() <= 1e-12 * 128
    assert main(["gram-dump", "--config", config, "--output", str(tmp_path / "o.csv")]) == 0
    assert (tmp_path / "o.csv").read_text() == dump.read_text()
    assert main(["verify", "--config", config, "--set", "grid_perturbation=0.003"]) == 1
    assert "FAIL bccb structure" in capsys.readouterr().out
    assert main(["verify", "--config", write_config(tmp_path / "big.json", dict(VERIFY, l1=1024))]) == 1
    assert "cap" in capsys.readouterr().out
    assert main(["verify", "--config", write_config(tmp_path / "s.json", dict(VERIFY, l1=32)), "--set", "cap=256"]) == 0
    capsys.readouterr()


@pytest.mark.gpu
def test_bench_writes_records(tmp_path, capsys):
    """pkg/tests/test_cli.py:236-258 (figures aside: the CSVs they are drawn from)."""
    config = write_config(tmp_path / "bench.json", {"m1_count": 10, "m2_count": 6, "element_count": 24, "l2": 8,
                                                    "l1_values": [8, 16], "iteration_values": [10], "trials": 1,
                                                    "base_seed": 7, "solvers": ["ista", "admm"]})
    out = tmp_path / "bench"
    assert main(["bench", "--config", config, "--output-dir", str(out)]) == 0
    for name in ("records.csv", "summary.csv", "plot_data.csv"):
        assert (out / name).exists(), name
    assert len((out / "records.csv").read_text().splitlines()) == 1 + 2 * 2 * 1 * 1
    assert main(["bench", "--config", write_config(tmp_path / "bad.json", {"m1_counts": 10}),
                 "--output-dir", str(tmp_path)]) == 1
    assert "m1_counts" in capsys.readouterr().err
