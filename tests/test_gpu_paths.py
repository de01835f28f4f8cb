"""GPU cross-checks of the kernel paths and edge cases.

The solver picks, per shape, the small-grid persistent solver, the shape-specialised
(zero-skipping, fused-column) kernels or the generic runtime-shape kernels.  These tests
run the same problems through the automatic path and the generic path
(`bccb_set_path(1)`), and through the float64 oracle, on the shapes and batch sizes the
fast paths special-case.
"""

import numpy as np
import pytest
import torch

import paper_2509_13592_b200 as bb
from oracle import bccb_oracle as orc
from paper_2509_13592_b200 import _lib, scenes

pytestmark = pytest.mark.gpu


def assert_close(est, ref, tol):
    """rel-L2 <= tol, or both exactly zero (ADMM's z stays 0 when rho*tau is large, SURVEY finding 7)."""
    est, ref = np.asarray(est), np.asarray(ref)
    if not ref.any():
        assert not est.any()
    else:
        assert orc.rel_l2(est, ref) < tol


@pytest.fixture
def generic_path():
    def run(fn):
        _lib.check(_lib.lib.bccb_set_path(1))
        try:
            return fn()
        finally:
            _lib.check(_lib.lib.bccb_set_path(0))
    return run


def scene_problem(cfg, nsnap, iters=None):
    w = scenes.workload(cfg)
    geom, ys, _ = scenes.make_scene(w, range(nsnap))
    op = bb.gram_operator(geom, w.l1, w.l2)
    m1, m2 = geom.occupied_coordinates()
    bs = np.stack([orc.adjoint_fft(m1, m2, w.l1, w.l2, y) for y in ys])
    taus = np.array([w.tau_fraction * np.abs(b).max() for b in bs])
    return w, geom, op, bs, taus


@pytest.mark.parametrize("cfg,nsnap,iters", [(1, 3, 200), (2, 6, 150), (3, 2, 80), (4, 2, 60), (5, 1, 8)])
def test_fista_auto_vs_generic_vs_oracle(cfg, nsnap, iters, generic_path):
    w, geom, op, bs, taus = scene_problem(cfg, nsnap)
    mu = 1.0 / (w.l1 * w.l2)
    prob = bb.LassoProblem(op, bs, taus)
    conf = bb.SolverConfig(iterations=iters, step_size_mu=mu)
    auto = bb.fista_solve(prob, conf).estimate
    gen = generic_path(lambda: bb.fista_solve(bb.LassoProblem(op, bs, taus), conf).estimate)
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2).T)
    for i in range(nsnap):
        assert orc.rel_l2(auto[i], gen[i]) < 1e-6
        ref = orc.fista(eig_t, bs[i], taus[i], mu, iters) if cfg != 5 or i == 0 else None
        if ref is not None:
            assert orc.rel_l2(auto[i], ref) < 1e-4
            np.testing.assert_array_equal(np.sort(orc.topk(auto[i], w.targets)), np.sort(orc.topk(ref, w.targets)))


@pytest.mark.parametrize("cfg,nsnap", [(1, 2), (2, 4)])
def test_ista_auto_vs_generic(cfg, nsnap, generic_path):
    w, geom, op, bs, taus = scene_problem(cfg, nsnap)
    mu = 1.0 / (w.l1 * w.l2)
    conf = bb.SolverConfig(iterations=120, step_size_mu=mu)
    auto = bb.ista_solve(bb.LassoProblem(op, bs, taus), conf).estimate
    gen = generic_path(lambda: bb.ista_solve(bb.LassoProblem(op, bs, taus), conf).estimate)
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2).T)
    for i in range(nsnap):
        assert orc.rel_l2(auto[i], gen[i]) < 1e-6
        assert orc.rel_l2(auto[i], orc.ista(eig_t, bs[i], taus[i], mu, 120)) < 1e-4


def test_admm_auto_vs_generic_and_oracle(generic_path):
    """Small threshold: z leaves zero, exercising the z / r skipping of the split-dual kernels
    (the automatic path: complex64 band FFTs, dual growth on the float64 box) against the
    generic complex128 engine and the oracle.  This regime is ill-conditioned (points hover at
    the threshold: rounding b to complex64 moves the float64 answer by ~2e-3), so both sides
    get identical inputs: complex64 y, whose signed scatter (the GPU's fft2(b) on the box) is
    exact."""
    from paper_2509_13592_b200.solvers import admm_solve_with_c
    w = scenes.workload(3)
    geom, ys, _ = scenes.make_scene(w, range(2))
    op = bb.gram_operator(geom, w.l1, w.l2)
    y32 = ys.astype(np.complex64)
    m1, m2 = geom.occupied_coordinates()
    bs = np.stack([orc.adjoint_fft(m1, m2, w.l1, w.l2, y.astype(np.complex128)) for y in y32])
    taus = np.array([w.tau_fraction * np.abs(b).max() * 0.002 for b in bs])
    conf = bb.SolverConfig(iterations=40, rho=1.0)
    auto = bb.admm_solve(bb.LassoProblem.from_measurements(op, y32, tau=taus), conf).estimate
    gen = generic_path(lambda: bb.admm_solve(bb.LassoProblem.from_measurements(op, y32, tau=taus), conf).estimate)
    za, va, ca = (t.cpu().numpy() for t in admm_solve_with_c(bb.LassoProblem.from_measurements(op, y32, tau=taus), conf))
    eig = orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2)
    for i in range(2):
        z, c, v = orc.admm(eig, bs[i], taus[i], 1.0, 40)
        assert np.count_nonzero(z) > 0
        assert orc.rel_l2(auto[i], gen[i]) < 1e-6
        assert orc.rel_l2(auto[i], z) < 1e-6
        np.testing.assert_array_equal(za[i], auto[i])
        assert orc.rel_l2(ca[i], c) < 1e-6
        assert orc.rel_l2(va[i], v) < 1e-6


@pytest.mark.parametrize("m1,m2,l1,l2", [(6, 4, 9, 6), (5, 3, 12, 10), (4, 4, 20, 8), (3, 5, 7, 16)])
def test_non_power_of_two_grids(m1, m2, l1, l2):
    """Generic runtime-shape kernels: lengths with small power-of-two factors (KP = 1..4)."""
    geom = bb.subsample_preserving_aperture(bb.make_ura(m1, m2), max(4, m1 * m2 // 2), seed=11)
    op = bb.gram_operator(geom, l1, l2)
    rng = np.random.default_rng(l1 * l2)
    y = rng.standard_normal(geom.element_count) + 1j * rng.standard_normal(geom.element_count)
    m1i, m2i = geom.occupied_coordinates()
    b = orc.adjoint_fft(m1i, m2i, l1, l2, y)
    np.testing.assert_allclose(bb.apply_adjoint(op, y), b, rtol=1e-5, atol=1e-5 * np.abs(b).max())
    tau = 0.1 * np.abs(b).max()
    mu = 1.0 / (l1 * l2)
    eig = orc.gram_eigenvalues_exact(geom.occupancy, l1, l2)
    eig_t = np.ascontiguousarray(eig.T)
    r = bb.fista_solve(bb.LassoProblem(op, b, tau), bb.SolverConfig(iterations=50, step_size_mu=mu))
    assert orc.rel_l2(r.estimate, orc.fista(eig_t, b, tau, mu, 50)) < 1e-5
    r = bb.admm_solve(bb.LassoProblem(op, b, tau * 0.05), bb.SolverConfig(iterations=30, rho=2.0))
    assert_close(r.estimate, orc.admm(eig, b, tau * 0.05, 2.0, 30)[0], 1e-4)


def test_per_snapshot_divergence_in_a_batch():
    w, geom, op, bs, taus = scene_problem(2, 4)
    mu = 1.0 / (w.l1 * w.l2)
    bad = bs.copy()
    bad[2] *= 1e30                                    # overflows float64 after a few iterations
    conf = bb.SolverConfig(iterations=60, step_size_mu=mu * 1e6)
    with pytest.raises(bb.DivergenceError) as info:
        bb.fista_solve(bb.LassoProblem(op, bad, taus), conf)
    per = info.value.per_snapshot
    assert per is not None and per[2] >= 0 and info.value.iteration == per[per >= 0].min()


def test_admm_warm_start_and_torch_batch():
    w, geom, op, bs, taus = scene_problem(2, 3)
    eig = orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2)
    z0 = np.zeros_like(bs)
    z0[:, 5] = 0.01
    bt = torch.as_tensor(bs).cuda()
    r = bb.admm_solve(bb.LassoProblem(op, bt, torch.as_tensor(taus)), bb.SolverConfig(iterations=20, initial_c=z0))
    assert isinstance(r.estimate, torch.Tensor) and r.estimate.shape == bt.shape
    est = r.estimate.cpu().numpy()
    for i in range(3):
        assert_close(est[i], orc.admm(eig, bs[i], taus[i], 1.0, 20, z0=z0[i])[0], 1e-5)


def test_extract_support_device_tensor():
    c = torch.zeros(64, dtype=torch.complex128, device="cuda")
    c[[3, 17, 40, 41]] = torch.tensor([2.0 - 1j, -5j, 0.2, 1.0 + 1.0j], dtype=torch.complex128, device="cuda")
    g = bb.make_uniform_grid(8)
    got = bb.extract_support(c, g, g, 0.1)
    ref = orc.extract_support(c.cpu().numpy(), g.frequencies, g.frequencies, 0.1)
    assert got == ref


@pytest.fixture
def substreams():
    def run(n, fn):
        _lib.check(_lib.lib.bccb_set_substreams(n))
        try:
            return fn()
        finally:
            _lib.check(_lib.lib.bccb_set_substreams(0))
    return run


def test_substream_split_is_bitwise_neutral(substreams):
    """The sub-batch split runs independent snapshots on up to 8 streams (with programmatic
    dependent launch between the passes of each stream): FISTA (config 2 shape) and the split
    ADMM (config 3 shape, small threshold so z leaves zero) give identical bits for every split."""
    w, geom, op, bs, taus = scene_problem(2, 64)
    mu = 1.0 / (w.l1 * w.l2)
    conf = bb.SolverConfig(iterations=60, step_size_mu=mu)
    # 64 config-2 snapshots: 3, 4 and 8 parts keep >= 2048 lines each, so each split really runs
    from paper_2509_13592_b200 import _lib as lib_
    for n in (3, 4, 8):
        assert substreams(n, lambda: lib_.lib.bccb_substreams_for(op._plan, 64)) == n
    outs = [substreams(n, lambda: bb.fista_solve(bb.LassoProblem(op, bs, taus), conf).estimate)
            for n in (1, 3, 4, 8)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])
    w3 = scenes.workload(3)
    geom3, ys, _ = scenes.make_scene(w3, range(12))
    op3 = bb.gram_operator(geom3, w3.l1, w3.l2)
    y32 = ys.astype(np.complex64)
    m1, m2 = geom3.occupied_coordinates()
    taus3 = np.array([w3.tau_fraction * 0.002 * np.abs(orc.adjoint_fft(m1, m2, w3.l1, w3.l2, y.astype(np.complex128))).max()
                      for y in y32])
    conf3 = bb.SolverConfig(iterations=30, rho=1.0)
    outs = [substreams(n, lambda: bb.admm_solve(bb.LassoProblem.from_measurements(op3, y32, tau=taus3),
                                                conf3).estimate) for n in (1, 3)]
    assert np.count_nonzero(outs[0]) > 0
    np.testing.assert_array_equal(outs[0], outs[1])
    # (z, v, c) through the c-returning entry point agree with admm_solve's z
    from paper_2509_13592_b200.solvers import admm_solve_with_c
    z = substreams(3, lambda: admm_solve_with_c(bb.LassoProblem.from_measurements(op3, y32, tau=taus3), conf3)[0])
    np.testing.assert_array_equal(z.cpu().numpy(), outs[0])


_PDL_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2509_13592_b200 as bb
from paper_2509_13592_b200 import scenes
from oracle import bccb_oracle as orc
w = scenes.workload(int(sys.argv[3]))
geom, ys, _ = scenes.make_scene(w, range(9))
op = bb.gram_operator(geom, w.l1, w.l2)
m1, m2 = geom.occupied_coordinates()
bs = np.stack([orc.adjoint_fft(m1, m2, w.l1, w.l2, y) for y in ys])
taus = np.array([w.tau_fraction * np.abs(b).max() for b in bs])
solver = sys.argv[4] if len(sys.argv) > 4 else "fista"
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 120
conf = bb.SolverConfig(iterations=iters, step_size_mu=1.0 / (w.l1 * w.l2), rho=w.rho)
if solver == "admm":   # z stays zero at rho = 1 on this scene; compare the whole state (z, v, c)
    from paper_2509_13592_b200.solvers import admm_solve_with_c
    est = np.concatenate([np.asarray(t.cpu().numpy() if hasattr(t, "cpu") else t)
                          for t in admm_solve_with_c(bb.LassoProblem(op, bs, taus), conf)])
else:
    est = getattr(bb, solver + "_solve")(bb.LassoProblem(op, bs, taus), conf).estimate
np.save(sys.argv[2], est)
"""


@pytest.mark.parametrize("env,bitwise", [({"BCCB_PDL": "0"}, True), ({"BCCB_PDL": "1"}, True),
                                         ({"BCCB_PDL": "2"}, True),
                                         ({"BCCB_COLS_WARP": "0"}, False)])
def test_launch_modes_agree(tmp_path, env, bitwise):
    """Programmatic dependent launch (with early reads before the grid-dependency wait) must not
    change a bit: default (PDL, implicit release at grid completion) vs PDL off / early release, each in a fresh
    process (the modes are read once).  The warp-per-line column pass sums the band in a
    different order than the shared-memory pass: equal to rounding."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_PDL_SCRIPT)
    outs = []
    for extra in ({}, env):
        out = tmp_path / f"est{len(outs)}.npy"
        e = dict(os.environ, BCCB_SUB_MIN_LINES="256", **extra)
        subprocess.run([sys.executable, str(script), root, str(out), "2"], check=True, env=e, timeout=600)
        outs.append(np.load(out))
    if bitwise:
        np.testing.assert_array_equal(outs[0], outs[1])
    else:
        for a, b in zip(outs[0], outs[1]):
            assert orc.rel_l2(a, b) < 1e-6


@pytest.mark.parametrize("pdl", ["1", "2"])
def test_fused_column_pass_pdl(tmp_path, pdl):
    """The fused column pass (rows kernel whose last CTA per snapshot runs the column pass; taken
    at L1 = 64 when the cluster and small-grid solvers are off) has no separate column pass
    between two rows passes, so nothing may be read before the grid-dependency wait: with PDL on
    it must agree bitwise with PDL off and match the float64 oracle (config-1 geometry, 9
    snapshots, fresh processes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_PDL_SCRIPT)
    outs = []
    for extra in ({"BCCB_CLUSTER": "0", "BCCB_SMALL_GRID": "0", "BCCB_PDL": pdl},
                  {"BCCB_CLUSTER": "0", "BCCB_SMALL_GRID": "0", "BCCB_PDL": "0"}):
        out = tmp_path / f"est{len(outs)}.npy"
        e = dict(os.environ, **extra)
        subprocess.run([sys.executable, str(script), root, str(out), "1"], check=True, env=e, timeout=600)
        outs.append(np.load(out))
    assert np.isfinite(outs[0]).all() and np.count_nonzero(outs[0]) > 0
    np.testing.assert_array_equal(outs[0], outs[1])
    w = scenes.workload(1)
    geom, ys, _ = scenes.make_scene(w, range(9))
    m1, m2 = geom.occupied_coordinates()
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2).T)
    mu = 1.0 / (w.l1 * w.l2)
    for s_, y in enumerate(ys[:3]):
        b = orc.adjoint_fft(m1, m2, w.l1, w.l2, y)
        ref = orc.fista(eig_t, b, w.tau_fraction * np.abs(b).max(), mu, 120)
        assert orc.rel_l2(outs[0][s_], ref) < 1e-4


@pytest.mark.parametrize("cfg,solver,iters", [(3, "admm", 120), (2, "ista", 120), (4, "fista", 120), (1, "fista", 120)])
def test_pdl_bitwise_across_solvers(tmp_path, cfg, solver, iters):
    """PDL on (early release, mode 1; implicit release, the default) vs off must agree bitwise for every solver's default
    kernel path: a read placed before the grid-dependency wait that races the preceding pass
    shows up here as a difference (9 snapshots, fresh processes; ADMM compares z, v and c:
    z stays zero at rho = 1 on the config-3 scene)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_PDL_SCRIPT)
    outs = []
    for extra in ({"BCCB_PDL": "1"}, {}, {"BCCB_PDL": "0"}):
        out = tmp_path / f"est{len(outs)}.npy"
        e = dict(os.environ, BCCB_SUB_MIN_LINES="256", **extra)
        subprocess.run([sys.executable, str(script), root, str(out), str(cfg), solver, str(iters)], check=True, env=e,
                       timeout=600)
        outs.append(np.load(out))
    assert np.isfinite(outs[0]).all() and np.count_nonzero(outs[0]) > 0
    np.testing.assert_array_equal(outs[0], outs[2])
    np.testing.assert_array_equal(outs[1], outs[2])


@pytest.mark.parametrize("cfg,nsnap,iters", [(4, 3, 120), (5, 1, 40)])
def test_tensor_core_rows_engine_matches_cuda_core_engine(tmp_path, cfg, nsnap, iters):
    """The tensor-core rows engine (tcgen05 kind::tf32 level-2 stage of the band inverse,
    3-pass hi/lo split) against the CUDA-core engine (BCCB_ROWS_TC=0) and the float64 oracle:
    equal to fp32 rounding, identical top-K (fresh processes: the engine is chosen once)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_PDL_SCRIPT.replace("range(9)", f"range({nsnap})"))
    outs = []
    for env in ({"BCCB_ROWS_TC": "1"}, {"BCCB_ROWS_TC": "0"}):
        out = tmp_path / f"est{len(outs)}.npy"
        subprocess.run([sys.executable, str(script), root, str(out), str(cfg), "fista", str(iters)], check=True,
                       env=dict(os.environ, **env), timeout=900)
        outs.append(np.load(out))
    w = scenes.workload(cfg)
    geom, ys, _ = scenes.make_scene(w, range(nsnap))
    m1, m2 = geom.occupied_coordinates()
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(geom.occupancy, w.l1, w.l2).T)
    for s_, y in enumerate(ys):
        b = orc.adjoint_fft(m1, m2, w.l1, w.l2, y)
        ref = orc.fista(eig_t, b, w.tau_fraction * np.abs(b).max(), 1.0 / (w.l1 * w.l2), iters)
        e_tc, e_cc = orc.rel_l2(outs[0][s_], ref), orc.rel_l2(outs[1][s_], ref)
        assert e_tc < 1e-5 and e_cc < 1e-5, (e_tc, e_cc)
        assert orc.rel_l2(outs[0][s_], outs[1][s_]) < 1e-5
        np.testing.assert_array_equal(orc.topk(outs[0][s_], w.targets), orc.topk(ref, w.targets))


@pytest.mark.parametrize("cfg,solver,nsnap,iters", [(2, "fista", 9, 200), (3, "admm", 3, 120), (4, "fista", 3, 150),
                                                    (5, "fista", 1, 60), (5, "ista", 1, 40)])
def test_energy_screen_is_bitwise_neutral(tmp_path, cfg, solver, nsnap, iters):
    """The energy screen of the level-1 inverse register DFT (band_fft.cuh reg_idft_screened:
    residue classes whose Parseval bound lies below the soft threshold for the whole warp skip
    their sub-DFT and per-point tests; on tensor-core tiles the two-level screen straight from
    TMEM) only skips points that provably stay exactly zero: BCCB_SCREEN=0 (every class computed)
    must give the same bits as both screens on (fresh processes), and the iterate must have gone
    sparse so the screens really fire."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "run.py"
    script.write_text(_PDL_SCRIPT.replace("range(9)", f"range({nsnap})"))
    outs = []
    # config 5 runs the tensor-core engine: its TMEM screen is bit 2 (off by default)
    for env in ({"BCCB_SCREEN": "3"}, {"BCCB_SCREEN": "0"}):
        out = tmp_path / f"est{len(outs)}.npy"
        subprocess.run([sys.executable, str(script), root, str(out), str(cfg), solver, str(iters)], check=True,
                       env=dict(os.environ, **env), timeout=900)
        outs.append(np.load(out))
    assert np.isfinite(outs[0]).all() and np.count_nonzero(outs[0]) > 0
    if solver != "admm":
        assert np.count_nonzero(outs[0]) < 0.05 * outs[0].size
    np.testing.assert_array_equal(outs[0], outs[1])
