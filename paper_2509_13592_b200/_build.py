"""Build the sm_100a shared library in-tree (no JIT cache: the .so travels with the repo).

`python paper_2509_13592_b200/_build.py` or `__graft_entry__.build()` (run as a file:
importing the package first would load the previous library).
"""

import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
LIB_NAME = "libbccb_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
SOURCES = ["bccb_capi.cu"]
HEADERS = ["band_fft.cuh", "bccb_kernels.cuh", "topk.cuh", "tcgen05.cuh"]
# self-test of the tcgen05 primitives (tests/test_gpu_tc.py only; not on any product path)
PROBE_NAME = "libbccb_tcprobe.so"
PROBE_PATH = os.path.join(PKG_DIR, PROBE_NAME)
PROBE_SOURCES = ["tc_probe.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "177",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _stale(path, sources) -> bool:
    if not os.path.exists(path):
        return True
    lib_mtime = os.path.getmtime(path)
    deps = [os.path.join(CSRC, f) for f in sources + HEADERS]
    deps.append(os.path.join(PKG_DIR, "..", "include", "bccb_b200.h"))
    return any(os.path.getmtime(d) > lib_mtime for d in deps if os.path.exists(d))


def _compile(path, sources, verbose):
    tmp = path + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", tmp] + [os.path.join(CSRC, s) for s in sources]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, path)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into LIB_PATH (and the tcgen05 self-test library) when sources are
    newer; return the library path."""
    if force or _stale(PROBE_PATH, PROBE_SOURCES):
        _compile(PROBE_PATH, PROBE_SOURCES, verbose)
    if force or _stale(LIB_PATH, SOURCES):
        _compile(LIB_PATH, SOURCES, verbose)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
