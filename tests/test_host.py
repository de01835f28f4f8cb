"""CPU tests of the boundary: C-ABI exports, status-code mapping, host-side logic."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import _lib, scenes
from paper_2509_13592_b200.errors import (
    BccbLassoError,
    DivergenceError,
    InvalidArgumentError,
    SingularOperatorError,
)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bccb_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.findall(r"^\s*(?!typedef)[\w \t\*]+?\b(bccb_\w+)\s*\(", text, flags=re.M)


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 16
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/bccb_b200.h but not exported"
    assert set(names) == set(_lib.SIGNATURES), "ctypes signature table out of sync with the header"


def test_header_argument_counts_match_bindings():
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(rf"{name}\s*\(([^)]*)\)", text)
        assert m, name
        decl = m.group(1).strip()
        n = 0 if decl in ("", "void") else decl.count(",") + 1
        assert n == len(args), f"{name}: header has {n} args, binding {len(args)}"


def test_version_and_validation_without_gpu():
    assert b"sm_100a" in _lib.lib.bccb_version()
    plan = ctypes.c_void_p()
    box = np.ones(4, dtype=np.complex128)
    rc = _lib.lib.bccb_plan_create(0, 4, 1, 1, box.ctypes.data, 0.0, 0.0, 0, ctypes.byref(plan))
    assert rc == _lib.ERR_INVALID and "positive" in _lib.last_error()
    rc = _lib.lib.bccb_plan_create(4, 4, 5, 1, box.ctypes.data, 0.0, 0.0, 0, ctypes.byref(plan))
    assert rc == _lib.ERR_INVALID and "outside" in _lib.last_error()
    occ = np.zeros((3, 3), dtype=np.uint8)
    rc = _lib.lib.bccb_plan_create_gram(8, 8, 3, 3, occ.ctypes.data, 0, ctypes.byref(plan))
    assert rc == _lib.ERR_INVALID and "occupied" in _lib.last_error()
    assert _lib.lib.bccb_workspace_bytes(None, 4) == 0
    assert _lib.lib.bccb_topk(1, 10, None, 0, 0, None, None, None, None) == _lib.ERR_INVALID
    assert _lib.lib.bccb_topk(1, 10, None, 0, 65, None, None, None, None) == _lib.ERR_INVALID
    assert _lib.lib.bccb_matvec(None, 1, None, None, None, None) == _lib.ERR_INVALID


def test_status_mapping():
    _lib.check(_lib.OK)
    with pytest.raises(InvalidArgumentError):
        _lib.lib.bccb_matvec(None, 1, None, None, None, None)
        _lib.check(_lib.ERR_INVALID)
    with pytest.raises(DivergenceError) as e:
        _lib.check(_lib.ERR_DIVERGENCE, iteration=7)
    assert e.value.iteration == 7
    with pytest.raises(SingularOperatorError):
        _lib.check(_lib.ERR_SINGULAR)
    with pytest.raises(BccbLassoError):
        _lib.check(_lib.ERR_CUDA)
    assert issubclass(InvalidArgumentError, ValueError)


def test_solver_config_validation():
    for kwargs in ({"iterations": 0}, {"iterations": 1, "step_size_mu": 0.0},
                   {"iterations": 1, "rho": -1.0}, {"iterations": 1, "backend": "gpu"}):
        with pytest.raises(InvalidArgumentError):
            bb.SolverConfig(**kwargs)
    cfg = bb.SolverConfig(iterations=3)
    assert cfg.rho == 1.0 and cfg.backend is None and not cfg.record_objective


def test_fista_alpha_sequence_and_soft_threshold():
    a = bb.fista_alpha_sequence(60)
    assert a[0] == 1.0
    for i in range(59):
        assert a[i + 1] == 0.5 * (np.sqrt(1.0 + 4.0 * a[i] ** 2) + 1.0)
    assert np.all(a >= (np.arange(1, 61) + 1) / 2 - 1e-12)
    with pytest.raises(InvalidArgumentError):
        bb.fista_alpha_sequence(0)
    for value, kappa, expected in [(3.0, 1.0, 2.0), (0.5j, 1.0, 0.0), (-2.0, 0.5, -1.5), (3 + 4j, 2.0, 1.8 + 2.4j)]:
        np.testing.assert_allclose(bb.soft_threshold(np.array([value]), kappa)[0], expected, atol=1e-15)
    z = np.array([1 + 1j, 2.0])
    out = bb.soft_threshold(z, 0.0)
    assert out is not z and np.array_equal(out, z)
    with pytest.raises(InvalidArgumentError):
        bb.soft_threshold(z, -0.1)


def test_uniform_grid_convention():
    # f = -1/2 + l/L (dictionary.py:41-45), not BASELINE.json's "f = l/L" (SURVEY finding 5)
    g = bb.make_uniform_grid(4)
    np.testing.assert_array_equal(g.frequencies, [-0.5, -0.25, 0.0, 0.25])
    with pytest.raises(InvalidArgumentError):
        bb.make_uniform_grid(0)


def test_geometry_and_workloads():
    geom = bb.subsample_preserving_aperture(bb.make_ura(6, 4), 14, seed=3)
    assert geom.element_count == 14
    occ = geom.occupancy
    assert occ[0].any() and occ[-1].any() and occ[:, 0].any() and occ[:, -1].any()
    m1, m2 = geom.occupied_coordinates()
    assert np.all(np.diff(m1 + m2 * 6) > 0)        # scan order m2 outer, m1 inner
    with pytest.raises(InvalidArgumentError):
        bb.subsample_preserving_aperture(bb.make_ura(3, 3), 3, seed=0)
    w = scenes.workload(2)
    assert w.work_gpi == 64 * 256 * 256 * 1000
    assert scenes.workload(5).l1 == 4096
    with pytest.raises(InvalidArgumentError):
        scenes.workload(9)


def test_separated_targets_config5():
    w = scenes.workload(5)
    t = scenes.draw_scene_targets(w, np.random.default_rng(5))
    assert len(t) == 32
    for i in range(32):
        for j in range(i):
            d1 = abs(t[i].f1 - t[j].f1) % 1.0
            d2 = abs(t[i].f2 - t[j].f2) % 1.0
            assert min(d1, 1 - d1) >= 1 / w.l1 or min(d2, 1 - d2) >= 1 / w.l2


def test_host_modules_do_not_map_the_cuda_library():
    """The CPU reference arm of bench.py and the oracle workers import the package's host
    modules (scenes, arrays) but must not map libbccb_b200.so (the library loads lazily on
    the first GPU call)."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, sys.argv[1]);"
            "import paper_2509_13592_b200, paper_2509_13592_b200.scenes, oracle.bccb_oracle;"
            "from paper_2509_13592_b200 import _lib;"
            "maps = open('/proc/self/maps').read();"
            "assert 'libbccb_b200' not in maps and not _lib.is_loaded(), 'library mapped at import';"
            "_lib.lib;"
            "assert 'libbccb_b200' in open('/proc/self/maps').read() and _lib.is_loaded();"
            "print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code, root], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr
