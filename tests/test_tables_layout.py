"""Host tests of the exact-split contraction's tables (no GPU).

* Version-2 tables hold integer numerators n and one common denominator L per
  variant; the double-double coefficients every kernel uses are derived from
  them and must be the correctly rounded pair of the exact rational n / L.
* The MMA column layout (bsf_internal.h: bsf_nt, bsf_part, bsf_mono_col) must
  map the monomials of every table degree injectively into the padded
  columns, give each lane of a quad whole polynomial rows, and keep every row
  within the lane's 2 * bsf_nt(deg) accumulator slots.
"""
import os
import subprocess
from fractions import Fraction as Fr

import numpy as np
import pytest

from paper_1109_5114_b200 import lut

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "paper_1109_5114_b200", "csrc", "bsf_internal.h")


@pytest.mark.parametrize("basis,r", [(0, 1), (1, 1), (0, 2), (1, 2)])
def test_v2_tables_integer_and_correctly_rounded(basis, r):
    tab = lut.load(basis, r)
    rng = np.random.default_rng(basis + 7 * r)
    for v in tab["variants"]:
        num, L = v["num"], v["L"]
        assert 1 <= L < 2**53
        assert np.all(num == np.round(num)) and np.abs(num).max() < 2**53
        nz = np.argwhere(num != 0)
        for idx in nz[rng.choice(len(nz), size=min(200, len(nz)), replace=False)]:
            idx = tuple(idx)
            exact = Fr(int(num[idx]), L)
            hi, lo = v["coef"][idx]
            assert hi == float(exact)                      # correctly rounded head
            assert lo == float(exact - Fr(hi))             # correctly rounded tail
        # the kernel weights sum to one on every region (partition of unity):
        # sum over slots of the constant-term numerators equals L
        mons = lut.monomials(v["deg"])
        c0 = mons.index((0, 0))
        for ri in range(num.shape[0]):
            assert int(num[ri, :, c0].sum()) == L


def _layout_program(tmp_path):
    src = open(HDR).read()
    a = src.index("__host__ __device__ constexpr int bsf_nt")
    b = src.index("// One interpolation table")
    prog = ("#define __host__\n#define __device__\n#include <cstdio>\n" + src[a:b] + r'''
int main() {
    const int degs[] = {1, 2, 4, 6, 7, 10, 14};
    for (int deg : degs) {
        const int nt = bsf_nt(deg);
        int used[256] = {0};
        int ok = nt > 0;
        for (int i = deg; i >= 0; --i) {
            const int lane = bsf_row_lane(deg, i), s0 = bsf_row_slot(deg, i);
            if (lane < 0 || s0 < 0 || s0 + (deg - i + 1) > 2 * nt) ok = 0;
            for (int j = deg - i; j >= 0; --j) {
                const int c = bsf_mono_col(deg, i, j);
                if (c < 0 || c >= 8 * nt || used[c]++) ok = 0;
                if ((c % 8) / 2 != lane) ok = 0;          // the row stays on its lane of the quad
            }
        }
        printf("%d %d %d\n", deg, nt, ok);
    }
    return 0;
}
''')
    c = tmp_path / "layout.cc"
    c.write_text(prog)
    exe = tmp_path / "layout"
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-o", str(exe), str(c)])
    return subprocess.check_output([str(exe)]).decode().split("\n")


def test_mma_column_layout(tmp_path):
    lines = [l.split() for l in _layout_program(tmp_path) if l.strip()]
    assert [int(l[0]) for l in lines] == [1, 2, 4, 6, 7, 10, 14]
    for deg, nt, ok in lines:
        assert ok == "1", (deg, nt)
    # every table degree in use has a layout (4r - 2 full, 3r - 2 zero-scale)
    degs = {int(l[0]) for l in lines}
    for r in (1, 2, 3, 4):
        assert 4 * r - 2 in degs and 3 * r - 2 in degs
