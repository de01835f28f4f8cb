"""GPU parity of the operator layer (bccb_matvec, construction, adjoint, spectrum, top-k).

Tolerances: the GPU computes in complex64 (BASELINE.json north_star), so matvecs
are checked at rel-L2 <= 1e-5 (measured ~1e-7..4e-7) against the reference's
float64 results held in tests/golden (made by oracle/gen_golden.py from the real
reference) and against the pinned oracle.  Integer/index results are bit-exact.
"""

import numpy as np
import pytest
import torch

import paper_2509_13592_b200 as bb
from conftest import load_golden
from oracle import bccb_oracle as orc
from paper_2509_13592_b200 import scenes

pytestmark = pytest.mark.gpu
MATVEC_TOL = 1e-5
MATVEC_TOL_Z = 1e-12   # complex128 engine (numpy callers): reference test tolerance 1e-11


@pytest.fixture(scope="module")
def small():
    return load_golden("small")


def test_generic_matvec_matches_reference(small):
    for l1, l2 in small["generic_shapes"]:
        l1, l2 = int(l1), int(l2)
        key = f"g{l1}x{l2}_"
        op = bb.BccbOperator(l1, l2, small[key + "eig"])
        got = bb.bccb_matvec(op, small[key + "c"])
        assert got.dtype == np.complex128 and got.shape == (l1 * l2,)
        # numpy (float64) callers get the complex128 engine: reference-grade agreement
        assert orc.rel_l2(got, small[key + "matvec"]) < MATVEC_TOL_Z, (l1, l2)
        got32 = bb.bccb_matvec(op, torch.as_tensor(small[key + "c"]).to(torch.complex64).cuda())
        assert got32.dtype == torch.complex64
        assert orc.rel_l2(got32.cpu().numpy(), small[key + "matvec"]) < MATVEC_TOL, (l1, l2)


def test_from_first_column_eigenvalues(small):
    for l1, l2 in small["generic_shapes"]:
        l1, l2 = int(l1), int(l2)
        key = f"g{l1}x{l2}_"
        op = bb.bccb_from_first_column(small[key + "col"], l1, l2)
        assert orc.rel_l2(op.eigenvalues, small[key + "eig"]) < MATVEC_TOL
        col = bb.bccb_first_column(op).values
        assert orc.rel_l2(col, small[key + "col"]) < MATVEC_TOL


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_gram_operator_eigenvalues_exact(small, seed):
    p = f"s{seed}_"
    geom = bb.ArrayGeometry(6, 4, small[p + "occupancy"])
    op = bb.gram_operator(geom, 8, 4)
    np.testing.assert_allclose(op.eigenvalues, small[p + "eig"], atol=1e-9)  # test_bccb.py:116-125
    assert (op.k1, op.k2) == (8, 4) or op.k1 * op.k2 < 32
    b = bb.apply_adjoint(op, small[p + "y"])
    assert orc.rel_l2(b, small[p + "b"]) < MATVEC_TOL


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_gram_matvec_and_adjoint_at_config_sizes(cfg):
    w = scenes.workload(cfg)
    g = load_golden(f"cfg{cfg}")
    geom = bb.ArrayGeometry(w.m1, w.m2, g["occupancy"])
    op = bb.gram_operator(geom, w.l1, w.l2)
    assert (op.k1, op.k2) == (w.m1, w.m2)          # band = occupied corner
    assert op.max_eigenvalue() == w.l1 * w.l2
    m1, m2 = geom.occupied_coordinates()
    eig_t = np.ascontiguousarray(orc.gram_eigenvalues_exact(g["occupancy"], w.l1, w.l2).T)
    rng = np.random.default_rng(cfg)
    c = rng.standard_normal(w.grid_points) + 1j * rng.standard_normal(w.grid_points)
    assert orc.rel_l2(bb.bccb_matvec(op, c), orc.matvec(eig_t, c)) < MATVEC_TOL_Z
    c32 = torch.as_tensor(c.astype(np.complex64)).cuda()
    assert orc.rel_l2(bb.bccb_matvec(op, c32).cpu().numpy(), orc.matvec(eig_t, c)) < MATVEC_TOL
    b = bb.apply_adjoint(op, g["y"][0])
    assert orc.rel_l2(b, orc.adjoint_fft(m1, m2, w.l1, w.l2, g["y"][0])) < MATVEC_TOL


def test_matvec_properties_full_size():
    """Linearity, Hermitian symmetry and projection idempotence at config-5 size."""
    w = scenes.workload(5)
    op = bb.gram_operator(scenes.geometry_for(w), w.l1, w.l2)
    gen = torch.Generator(device="cuda").manual_seed(0)
    shape = (2, w.grid_points)
    x = torch.randn(shape, dtype=torch.complex64, device="cuda", generator=gen)
    y = torch.randn(shape, dtype=torch.complex64, device="cuda", generator=gen)
    a, b = 0.7 - 0.2j, -1.3 + 0.4j
    lhs = bb.bccb_matvec(op, a * x + b * y)
    rhs = a * bb.bccb_matvec(op, x) + b * bb.bccb_matvec(op, y)
    assert float((lhs - rhs).norm() / rhs.norm()) < 1e-5
    gx, gy = bb.bccb_matvec(op, x), bb.bccb_matvec(op, y)
    s1 = (gx.conj() * y).sum(dim=1).to(torch.complex128)
    s2 = (x.conj() * gy).sum(dim=1).to(torch.complex128)
    assert float((s1 - s2).abs().max() / s1.abs().max()) < 1e-4
    # (G/L) is an orthogonal projection: (G/L)^2 = G/L
    L = float(w.grid_points)
    p1 = bb.bccb_matvec(op, x) / L
    p2 = bb.bccb_matvec(op, p1) / L
    assert float((p2 - p1).norm() / p1.norm()) < 1e-5


def test_batched_matvec_equals_single():
    w = scenes.workload(2)
    op = bb.gram_operator(scenes.geometry_for(w), w.l1, w.l2)
    x = torch.randn((5, w.l2, w.l1), dtype=torch.complex64, device="cuda")
    yb = bb.bccb_matvec(op, x)
    assert yb.shape == x.shape
    for i in range(5):
        assert torch.equal(yb[i], bb.bccb_matvec(op, x[i].reshape(-1)).reshape(w.l2, w.l1))


def test_scale_add_identity_and_inverse():
    rng = np.random.default_rng(23)
    spec = rng.uniform(0.5, 2.0, (5, 3)) + 0j
    op = bb.BccbOperator(5, 3, spec)
    inv = bb.bccb_inverse(op)
    c = rng.standard_normal(15) + 1j * rng.standard_normal(15)
    back = bb.bccb_matvec(inv, bb.bccb_matvec(op, c))
    assert orc.rel_l2(back, c) < 1e-5
    shifted = bb.bccb_scale_add_identity(op, 2.0, 3.5)
    assert orc.rel_l2(bb.bccb_matvec(shifted, c), 2.0 * bb.bccb_matvec(op, c) + 3.5 * c) < 1e-5
    # a partial-box Gram: shifting moves the outside value, inversion guards singularity
    geom = bb.subsample_preserving_aperture(bb.make_ura(4, 3), 8, seed=0)
    g = bb.gram_operator(geom, 16, 8)
    with pytest.raises(bb.SingularOperatorError) as info:
        bb.bccb_inverse(g)
    assert info.value.min_abs_eigenvalue < info.value.threshold
    gi = bb.bccb_inverse(bb.bccb_scale_add_identity(g, 1.0, 1.0))
    x = rng.standard_normal(128) + 1j * rng.standard_normal(128)
    eig_t = np.ascontiguousarray((1.0 / (orc.gram_eigenvalues_exact(geom.occupancy, 16, 8) + 1.0)).T)
    assert orc.rel_l2(bb.bccb_matvec(gi, x), orc.matvec(eig_t, x)) < 1e-5


def test_matvec_shape_check():
    op = bb.BccbOperator(3, 2, np.ones((3, 2)))
    with pytest.raises(bb.InvalidArgumentError):
        bb.bccb_matvec(op, np.zeros(5, dtype=complex))


def test_topk_bit_exact_with_ties():
    rng = np.random.default_rng(7)
    for length, k in [(10, 3), (4096, 8), (65536, 16), (300_001, 32), (1 << 20, 64)]:
        x = np.zeros((3, length), dtype=np.complex128)
        nz = rng.choice(length, size=min(length, 2000), replace=False)
        x[:, nz] = rng.standard_normal((3, nz.size)) + 1j * rng.standard_normal((3, nz.size))
        x[1, nz[:50]] = 1.0           # ties: equal magnitudes -> lower index first
        x[2, :] = 0.0                 # all zero -> index order
        idx, mag = bb.topk_peaks(x, k)
        idx = idx.cpu().numpy()
        for s in range(3):
            np.testing.assert_array_equal(idx[s], orc.topk(x[s], k))
        idx32, _ = bb.topk_peaks(x.astype(np.complex64), k)
        np.testing.assert_array_equal(idx32.cpu().numpy()[2], np.arange(k))


def test_extract_support_matches_reference(small):
    g8 = bb.make_uniform_grid(8)
    sup = bb.extract_support(small["support_c"], g8, g8, 0.1)
    got = np.array([[a, b, v.real, v.imag] for a, b, v in sup])
    np.testing.assert_array_equal(got, small["support_ref"])
    assert bb.extract_support(np.zeros(16, dtype=complex), bb.make_uniform_grid(4), bb.make_uniform_grid(4), 0.1) == []
    # more than 64 entries above threshold -> ordered fallback path
    c = np.ones(256, dtype=complex)
    c[10] = 2.0
    sup = bb.extract_support(c, bb.make_uniform_grid(16), bb.make_uniform_grid(16), 0.1)
    assert len(sup) == 256 and sup[0][2] == 2.0


def _dense_from_first_column(col, l1, l2):
    """Dense BCCB expansion by modular index arithmetic: entry (i, j) = col[(i1 - j1) mod L1 +
    ((i2 - j2) mod L2) L1] (the reference test's independent oracle, test_bccb.py:45-54)."""
    i = np.arange(l1 * l2)
    i1, i2 = i % l1, i // l1
    return col[((i1[:, None] - i1[None, :]) % l1) + ((i2[:, None] - i2[None, :]) % l2) * l1]


def test_first_column_operators_match_dense_at_reference_tolerance():
    """pkg/tests/test_bccb.py:99-107 through the drop-in: 20 random first columns (L1, L2 in
    1..8), bccb_from_first_column on the float64 band engine, numpy matvec vs the dense
    expansion at rtol 1e-11; bccb_first_column recovers the column at the same precision."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        l1, l2 = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        col = rng.standard_normal(l1 * l2) + 1j * rng.standard_normal(l1 * l2)
        op = bb.bccb_from_first_column(col, l1, l2)
        c = rng.standard_normal(l1 * l2) + 1j * rng.standard_normal(l1 * l2)
        np.testing.assert_allclose(bb.bccb_matvec(op, c), _dense_from_first_column(col, l1, l2) @ c,
                                   rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(bb.bccb_first_column(op).values, col, rtol=1e-11, atol=1e-12)
    # larger generic shapes of the golden fixture: eigenvalues at float64 accuracy
    small = load_golden("small")
    for l1, l2 in small["generic_shapes"]:
        l1, l2 = int(l1), int(l2)
        op = bb.bccb_from_first_column(small[f"g{l1}x{l2}_col"], l1, l2)
        assert orc.rel_l2(op.eigenvalues, small[f"g{l1}x{l2}_eig"]) < 1e-13


def test_concurrent_matvec_and_solves_on_one_operator():
    """an operator is shareable and matvec may run concurrently.  Two threads,
    each on its own CUDA stream, apply one config-2 operator and run FISTA solves on it at the
    same time; every result equals the single-threaded one bitwise (per-thread workspace and
    per-thread sub-batch streams)."""
    import threading
    w = scenes.workload(2)
    geom, ys, _ = scenes.make_scene(w, range(8))
    op = bb.gram_operator(geom, w.l1, w.l2)
    rng = np.random.default_rng(5)
    xs = [torch.as_tensor(rng.standard_normal((4, w.grid_points)) + 1j * rng.standard_normal((4, w.grid_points)),
                          dtype=torch.complex64).cuda() for _ in range(2)]
    conf = bb.SolverConfig(iterations=80, step_size_mu=1.0 / w.grid_points)
    probs = [bb.LassoProblem.from_measurements(op, ys[4 * i:4 * i + 4], tau_fraction=w.tau_fraction) for i in range(2)]

    def work(i):
        return bb.bccb_matvec(op, xs[i]).cpu().numpy(), bb.fista_solve(probs[i], conf).estimate

    ref = [work(i) for i in range(2)]
    out = [None, None]

    def run(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                mv, est = work(i)
                out[i] = (mv, est)
            s.synchronize()

    threads = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for i in range(2):
        np.testing.assert_array_equal(out[i][0], ref[i][0])
        np.testing.assert_array_equal(out[i][1], ref[i][1])
