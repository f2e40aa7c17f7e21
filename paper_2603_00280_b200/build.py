"""In-tree build of libmacrofacet_b200.so for sm_100a (nvcc cross-compiles
without a GPU).  `python -m paper_2603_00280_b200.build`"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "mf_kernels.cu")
OUT = os.path.join(HERE, "libmacrofacet_b200.so")
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [
    os.path.join(ROOT, "include", "macrofacet_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    # explicit intrinsics are used where accuracy allows; keep IEEE exp/log
    # (no --use_fast_math) but approximate division / sqrt and FTZ
    "-prec-div=false", "-prec-sqrt=false", "-ftz=true",
    # a value-returning function that can fall off its end is an error
    "-Xcudafe", "--diag_error=940", "-Xcompiler", "-Werror=return-type",
    "-Xptxas", "-v",
]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force=False, verbose=False):
    if not force and not needs_build():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, SRC, "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
