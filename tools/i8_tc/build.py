"""Build tools/i8_tc/libi8tc.so (the tcgen05 kind::i8 exact-contraction
prototype, sm_100a) in-tree; nvcc cross-compiles without a GPU."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "i8_contract.cu")
OUT = os.path.join(HERE, "libi8tc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False) -> str:
    if force or not os.path.exists(OUT) or os.path.getmtime(SRC) > os.path.getmtime(OUT):
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                               "-DI8TC_LIB", "-shared", "-Xcompiler", "-fPIC", "-o", OUT, SRC])
    return OUT


if __name__ == "__main__":
    print(build(force=True))
