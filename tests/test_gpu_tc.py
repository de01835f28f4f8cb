"""tcgen05 primitives (csrc/tcgen05.cuh) against numpy: descriptors, the canonical K-major
layout, kind::tf32 MMA into TMEM, tcgen05.commit -> mbarrier, tcgen05.ld read-back, and the
3-pass tf32 hi/lo split product that the band engine's tensor-core stage relies on."""

import ctypes
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PROBE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "paper_2509_13592_b200", "libbccb_tcprobe.so")


@pytest.fixture(scope="module")
def probe():
    assert os.path.exists(PROBE), "build the library first (__graft_entry__.build())"
    lib = ctypes.CDLL(PROBE)
    lib.bccb_tc_probe.restype = ctypes.c_int
    lib.bccb_tc_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("n", [32, 64, 128, 256])
@pytest.mark.parametrize("ksteps", [1, 2])
def test_tf32_mma_layout_and_split(probe, n, ksteps):
    rng = np.random.default_rng(n * 10 + ksteps)
    K = 8 * ksteps
    A = rng.standard_normal((128, K)).astype(np.float32)
    B = rng.standard_normal((n, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    out = {}
    for passes in (1, 3):
        a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        d = torch.full((128, n), float("nan"), dtype=torch.float32, device="cuda")
        rc = probe.bccb_tc_probe(a.data_ptr(), b.data_ptr(), d.data_ptr(), n, ksteps, passes,
                                 torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        out[passes] = d.cpu().numpy().astype(np.float64)
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    err1 = np.max(np.abs(out[1] - ref) / scale)
    err3 = np.max(np.abs(out[3] - ref) / scale)
    assert err1 < 2e-3, err1            # one tf32 pass: 10 explicit mantissa bits
    assert err3 < 2e-6, err3            # hi/lo split: fp32-grade
