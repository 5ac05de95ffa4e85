"""Host-side tests (no GPU): the C-ABI library, the interpolation tables and
the input generators."""
import ctypes
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1109_5114_b200 import bsf, lut

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    """libbsf.so loads without a GPU and exports every function of include/bsf.h."""
    from paper_1109_5114_b200 import build
    build.build()
    L = ctypes.CDLL(bsf.LIB_PATH)
    names = bsf.exported_symbols()
    assert "bsf_plan_create" in names and "bsf_filter" in names and "bsf_preintegrate" in names
    for n in names:
        assert hasattr(L, n), n
    assert bsf.lib().bsf_version() >= 100
    assert bsf.lib().bsf_status_str(5).decode().startswith("kernel reach")


def test_product_does_not_import_oracle():
    """The product package never reaches the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1109_5114_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "bsf_oracle" not in src, f


@pytest.mark.parametrize("basis", [0, 1])
@pytest.mark.parametrize("r", [1, 2])
def test_tables_match_oracle_kernel(basis, r):
    """Exact-rational tables of the unit-lattice kernel (Eq. 11, r-fold) vs
    the oracle's independent evaluator, for the full kernel and the four
    zero-scale variants; and partition of unity."""
    tab = lut.load(basis, r)
    s = O.steps(basis).astype(float)
    h = np.linalg.norm(s, axis=1)
    rng = np.random.default_rng(basis * 10 + r)
    for vi, v in enumerate(tab["variants"]):
        drop = v["drop"]
        a = h.copy()
        keep = [k for k in range(4) if k != drop]
        if drop >= 0:
            a[drop] = 0.0
        centre = 0.5 * r * s[keep].sum(0)
        for _ in range(12 if r == 1 else 4):
            x, y = rng.uniform(0, 1, 2)
            offs, w = lut.eval_window(tab, vi, x, y)
            ref = O.beta(basis, r, a, x - offs[:, 0] - centre[0], y - offs[:, 1] - centre[1])
            np.testing.assert_allclose(w, ref, atol=1e-14)
            assert abs(w.sum() - 1) < 1e-13
        # on a lattice point (even-order central taps land there)
        offs, w = lut.eval_window(tab, vi, 0.0, 0.0)
        ref = O.beta(basis, r, a, -offs[:, 0] - centre[0], -offs[:, 1] - centre[1])
        np.testing.assert_allclose(w, ref, atol=1e-14)


def test_table_window_sizes():
    """24 taps for Theta' and 7 for Theta at r = 1 (PAPER.md:349-351 window)."""
    assert lut.load(1, 1)["variants"][0]["nmax"] == 24
    assert lut.load(0, 1)["variants"][0]["nmax"] == 7
    assert lut.load(1, 2)["variants"][0]["nmax"] == 96
    assert lut.load(0, 2)["variants"][0]["nmax"] == 28


def test_synth_is_deterministic_and_windowed():
    w = synth.workload(2)
    a = synth.make_image(w, window=(100, 140, 200, 260))
    b = synth.make_image(w)[100:140, 200:260]
    assert torch.equal(a, b)
    c1 = synth.make_cov(w, window=(10, 20, 30, 50))
    c2 = synth.make_cov(w)[:, 10:20, 30:50]
    assert torch.equal(c1, c2)
    assert float(c2[0].min()) >= 1.0 and float(c2[0].max()) <= 16.0
    u8 = synth.make_image(synth.workload(1))
    assert u8.dtype == torch.uint8 and int(u8.max()) > 250 and int(u8.min()) < 5
    w3 = synth.workload(3)
    cov = synth.make_cov(w3, window=(0, 64, 0, 64))
    assert float(cov[0].min()) >= 2.0 and float(cov[0].max()) <= 40.0
    assert float((cov[0] / cov[1]).max() ** 2) <= 6.0 + 1e-4


def test_plan_rejects_bad_descriptors():
    """Argument errors are synchronous and need no GPU."""
    with pytest.raises(bsf.BsfError) as e:
        bsf.Plan(0, 10)
    assert e.value.status == 1
    with pytest.raises(bsf.BsfError) as e:
        bsf.Plan(10, 10, order=5)
    assert e.value.status == 1
    with pytest.raises(bsf.BsfError) as e:
        bsf.Plan(10, 10, max_sigma=10.0, margin_x=5)
    assert e.value.status == 5


def test_binding_validates_tensors_before_the_c_abi():
    """The C ABI takes raw pointers and cannot check them: the binding does
    (dtype, contiguity, element count, device)."""
    import torch
    from paper_1109_5114_b200 import bsf
    t = torch.zeros(10, dtype=torch.float32)
    bsf._want(t, "x", ["float32"], 10, "cpu")
    for args in ((t, "x", ["float64"], 10, "cpu"), (t, "x", ["float32"], 11, "cpu"),
                 (t.view(2, 5).t(), "x", ["float32"], 10, "cpu"), (t, "x", ["float32"], 10, 0)):
        with pytest.raises(bsf.BsfError):
            bsf._want(*args)


def test_oracle_mutation_sites_exist():
    """tools/oracle_mutations.py (the mutation check of the pins): every
    mutation's original text occurs exactly once in oracle/bsf_oracle.c and
    differs from its replacement, so the tool keeps mutating what it names."""
    import importlib.util
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("oracle_mutations", os.path.join(root, "tools", "oracle_mutations.py"))
    m = importlib.util.module_from_spec(spec)
    argv, sys_mod = None, __import__("sys")
    argv, sys_mod.argv = sys_mod.argv, ["oracle_mutations.py"]
    try:
        spec.loader.exec_module(m)
    finally:
        sys_mod.argv = argv
    src = open(os.path.join(root, "oracle", "bsf_oracle.c")).read()
    assert len(m.MUTATIONS) >= 31
    for name, old, new in m.MUTATIONS:
        assert src.count(old) == 1, name
        assert old != new, name
