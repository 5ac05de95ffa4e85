"""Build libbsf.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("bsf_api.cu", "bsf_kernels.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(os.path.dirname(HERE), "include", "bsf.h"),
                                                             os.path.abspath(__file__)]
OUT = os.path.join(HERE, "libbsf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "--expt-relaxed-constexpr"]


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(OUT) or any(os.path.getmtime(d) > os.path.getmtime(OUT) for d in DEPS)
    if force or stale:
        extra = os.environ.get("BSF_NVCC_EXTRA", "").split()  # diagnostics builds only
        cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-o", OUT] + SRC
        subprocess.check_call(cmd)
    return OUT


def build_luts(orders=(1, 2)) -> None:
    from . import lut
    for r in orders:
        for b in (0, 1):
            lut.ensure(b, r)


if __name__ == "__main__":
    build(force="-f" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
