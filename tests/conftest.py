import glob
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def host_math():
    """ctypes handle of the host build of csrc/mf_math.cuh (tests only)."""
    import ctypes

    out_dir = os.path.join(ROOT, "tests", "native", "_build")
    so = os.path.join(out_dir, "libmf_host.so")
    src = os.path.join(ROOT, "tests", "native", "mf_host_shim.cpp")
    deps = [src] + sorted(glob.glob(os.path.join(ROOT, "paper_2603_00280_b200", "csrc", "*"))) + [
        os.path.join(ROOT, "include", "macrofacet_b200.h")]
    if not os.path.exists(so) or any(os.path.getmtime(d) > os.path.getmtime(so) for d in deps):
        os.makedirs(out_dir, exist_ok=True)
        subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
                        "-Wall", "-Wno-unknown-pragmas", "-Werror=return-type",
                        "-o", so, src], check=True)
    return ctypes.CDLL(so)


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_00280_b200 import build

    if not os.path.exists(build.OUT):
        build.build()
    torch.cuda.set_device(0)
    return torch
