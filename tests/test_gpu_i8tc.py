"""The int8 tensor-core route of the window contraction (DESIGN.md §10,
tools/i8_tc): the exact part E = sum_s n_s G_s of the order-3 interpolation
(Eq. (11); table numerators n as integers)
computed by tcgen05.mma kind::i8 byte-slice products with s32 accumulators in
TMEM must equal the exact integer result (Python integers) bit for bit,
including the extreme magnitudes (|n| up to 2^55, |G| up to 2^63)."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MREAL, N = 66, 32


def _lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location("i8tc_build", os.path.join(ROOT, "tools", "i8_tc", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    L = ctypes.CDLL(B.build())
    L.i8tc_contract.restype = ctypes.c_int
    L.i8tc_contract.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    return L


@pytest.mark.parametrize("K,ntab,ngroups,nbits,gbits", [(224, 3, 5, 48, 57), (64, 2, 3, 55, 63), (32, 1, 1, 8, 8)])
def test_tcgen05_i8_exact_contraction(K, ntab, ngroups, nbits, gbits):
    rng = np.random.default_rng(K + ngroups)
    n = rng.integers(-(1 << nbits), 1 << nbits, size=(ntab, K, MREAL), dtype=np.int64)
    G = rng.integers(-(1 << gbits), (1 << gbits) - 1, size=(ngroups, N, K), dtype=np.int64, endpoint=True)
    n.flat[0], n.flat[1] = (1 << nbits) - 1, -(1 << nbits)  # extremes
    G.flat[0], G.flat[1] = (1 << gbits) - 1, -(1 << gbits)
    E = np.zeros((ngroups, MREAL, N, 2), dtype=np.int64)
    ms = ctypes.c_float(0.0)
    rc = _lib().i8tc_contract(n.ctypes.data, ntab, G.ctypes.data, ngroups, K, E.ctypes.data, 1, ctypes.byref(ms))
    assert rc == 0
    got = [[[int(E[g, m, i, 1]) * (1 << 64) + (int(E[g, m, i, 0]) & ((1 << 64) - 1)) for i in range(N)]
            for m in range(MREAL)] for g in range(ngroups)]
    for g in range(ngroups):
        t = n[g % ntab].astype(object)  # exact Python integers
        ref = np.dot(t.T, G[g].astype(object).T)  # [MREAL][N]
        for m in range(MREAL):
            assert got[g][m] == list(ref[m]), (g, m)


def test_tcgen05_i8_rejects_bad_shapes():
    L = _lib()
    n = np.zeros((1, 48, MREAL), dtype=np.int64)
    G = np.zeros((1, N, 48), dtype=np.int64)
    E = np.zeros((1, MREAL, N, 2), dtype=np.int64)
    assert L.i8tc_contract(n.ctypes.data, 1, G.ctypes.data, 1, 48, E.ctypes.data, 0, None) == -1  # K % 32
