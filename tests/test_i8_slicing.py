"""Host checks of the int8 tensor-core route (tools/i8_tc): the
byte-slice identity the tcgen05 kernel relies on, in exact integers, and that
the prototype library builds for sm_100a and exports its entry point.

With n = sum_{a<7} 2^{8a} A_a (A_0..A_5 unsigned bytes, A_6 the signed top
byte of a 56-bit two's complement value) and G = sum_{b<8} 2^{8b} B_b (B_7
signed), E = n G = sum_c 2^{8c} D_c with D_c = sum_{a+b=c} A_a B_b, and every
class sum over K <= 4096 slots stays inside int32 (the TMEM accumulators)."""
import ctypes
import os
import random
import subprocess


import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NA, NB = 7, 8


def slices(v, nbytes):
    """Byte slices of a two's complement value: unsigned low bytes, signed top byte."""
    u = v & ((1 << (8 * nbytes)) - 1)
    s = [(u >> (8 * i)) & 0xFF for i in range(nbytes)]
    if s[-1] >= 128:
        s[-1] -= 256
    return s


def test_slices_reassemble_two_complement_values():
    rng = random.Random(5)
    for nbits, nbytes in ((55, NA), (63, NB)):
        for v in [0, 1, -1, (1 << nbits) - 1, -(1 << nbits)] + [rng.randrange(-(1 << nbits), 1 << nbits) for _ in range(200)]:
            s = slices(v, nbytes)
            assert all(0 <= x <= 255 for x in s[:-1]) and -128 <= s[-1] <= 127
            assert sum(x << (8 * i) for i, x in enumerate(s)) == v


def test_class_sums_give_the_exact_contraction_and_fit_int32():
    rng = random.Random(11)
    K = 4096
    for trial in range(3):
        n = [rng.choice([(1 << 55) - 1, -(1 << 55), rng.randrange(-(1 << 55), 1 << 55)]) for _ in range(K)]
        G = [rng.choice([(1 << 63) - 1, -(1 << 63), rng.randrange(-(1 << 63), 1 << 63)]) for _ in range(K)]
        A = [slices(v, NA) for v in n]
        B = [slices(v, NB) for v in G]
        D = [0] * (NA + NB - 1)
        for s in range(K):
            for a in range(NA):
                for b in range(NB):
                    D[a + b] += A[s][a] * B[s][b]
        assert all(-(1 << 31) <= d < (1 << 31) for d in D)  # int32 accumulators
        assert sum(d << (8 * c) for c, d in enumerate(D)) == sum(x * y for x, y in zip(n, G))
    # the worst case bound used by the kernel: 7 pairs x 255 x 255 x 4096 < 2^31
    assert 7 * 255 * 255 * 4096 < (1 << 31)


def test_prototype_library_builds_and_exports():
    if subprocess.run(["which", "nvcc"], capture_output=True).returncode != 0 and \
            not os.path.exists("/usr/local/cuda/bin/nvcc"):
        pytest.skip("no nvcc")
    import importlib.util
    spec = importlib.util.spec_from_file_location("i8tc_build", os.path.join(ROOT, "tools", "i8_tc", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    path = B.build()
    L = ctypes.CDLL(path)  # loads without a GPU (the CUDA runtime binds lazily)
    assert hasattr(L, "i8tc_contract")
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "LDTM" in sass and "UTCCP" in sass
