"""Mutation check of the oracle pins (test infrastructure, CPU only).

Applies plausible single-point mistakes to a copy of oracle/bsf_oracle.c in a
temporary directory, rebuilds it there and runs the `-m "not gpu"` oracle pins
against it; every mutation must make at least one pin fail.  Usage:
    python tools/oracle_mutations.py [first]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) -- each original must occur exactly once
MUTATIONS = [
    ("kurtosis off-diagonal weight 2 -> 0.5",
     "return K[0] * K[0] + 2 * K[1] * K[1] + K[2] * K[2];",
     "return K[0] * K[0] + 0.5 * K[1] * K[1] + K[2] * K[2];"),
    ("decode: sign of C12",
     "C[1] = (vx - vy) * s * c;",
     "C[1] = -(vx - vy) * s * c;"),
    ("Theta covariance: C12 = (u2 + u4)/24",
     "C[1] = (u2 - u4) / 24.0;",
     "C[1] = (u2 + u4) / 24.0;"),
    ("Theta' covariance: dropped 4 u4 in C11",
     "C[0] = (4 * u1 + u2 + u3 + 4 * u4) / 60.0;",
     "C[0] = (4 * u1 + u2 + u3) / 60.0;"),
    ("Theta' kurtosis: K22 weight of q2 4 -> 1",
     "K[2] = (q1 + 4 * q2 + 4 * q3 + q4) / 5.0;",
     "K[2] = (q1 + q2 + 4 * q3 + q4) / 5.0;"),
    ("Theta' bound: 3/5 -> 4/5",
     "double b1 = c2 > 0 ? 0.6 / c2 : INFINITY;",
     "double b1 = c2 > 0 ? 0.8 / c2 : INFINITY;"),
    ("clamp factor 0.95 -> 0.9",
     "double lim = 0.95 * rb;",
     "double lim = 0.9 * rb;"),
    ("B-spline: centring r/2 -> r",
     "double xx = s / a + 0.5 * r;",
     "double xx = s / a + 1.0 * r;"),
    ("order: C/r -> C",
     "double Cr[3] = {C[0] / r, C[1] / r, C[2] / r};",
     "double Cr[3] = {C[0], C[1], C[2]};"),
    ("support: transposed pixel offset",
     "or_beta(basis, r, a, (double)(px - qx), (double)(py - qy));",
     "or_beta(basis, r, a, (double)(py - qy), (double)(px - qx));"),
    ("pre-integration: step sign",
     "int py = y - sy, pxi = xi - sx;",
     "int py = y - sy, pxi = xi + sx;"),
    # second batch: the remaining terms of the covariance / kurtosis formulas,
    # the gradient, the decode diagonal, the bounds and the sector choice
    ("Theta covariance: C11 weight of u1 2 -> 1",
     "C[0] = (2 * u1 + u2 + u4) / 24.0;",
     "C[0] = (u1 + u2 + u4) / 24.0;"),
    ("Theta covariance: C22 takes u1 for u3",
     "C[2] = (2 * u3 + u2 + u4) / 24.0;",
     "C[2] = (2 * u1 + u2 + u4) / 24.0;"),
    ("Theta' covariance: C12 sign of u2",
     "C[1] = 2 * (u1 + u2 - u3 - u4) / 60.0;",
     "C[1] = 2 * (u1 - u2 - u3 - u4) / 60.0;"),
    ("Theta' covariance: C22 weight of u3 4 -> 1",
     "C[2] = (u1 + 4 * u2 + 4 * u3 + u4) / 60.0;",
     "C[2] = (u1 + 4 * u2 + u3 + u4) / 60.0;"),
    ("Theta' kurtosis: K12 sign of q3",
     "K[1] = 2 * (q1 + q2 - q3 - q4) / 5.0;",
     "K[1] = 2 * (q1 + q2 + q3 - q4) / 5.0;"),
    ("Theta kurtosis: K11 weight of q2 1/2 -> 1",
     "K[0] = q1 + q2 / 2 + q4 / 2;",
     "K[0] = q1 + q2 + q4 / 2;"),
    ("Theta kurtosis: K12 = (q2 + q4)/2",
     "K[1] = (q2 - q4) / 2;",
     "K[1] = (q2 + q4) / 2;"),
    ("gradient: off-diagonal weight 2 -> 1",
     "return 2 * (K[0] * dK[0] + 2 * K[1] * dK[1] + K[2] * dK[2]);",
     "return 2 * (K[0] * dK[0] + K[1] * dK[1] + K[2] * dK[2]);"),
    ("decode: C11 and C22 swapped trigonometry",
     "C[0] = vx * c * c + vy * s * s;",
     "C[0] = vx * s * s + vy * c * c;"),
    ("Theta' bound: 4/5 -> 3/5 on sin",
     "double b2 = s2 > 0 ? 0.8 / s2 : INFINITY;",
     "double b2 = s2 > 0 ? 0.6 / s2 : INFINITY;"),
    ("Theta bound: 1/(s2 + c2) -> 1/max",
     "if (basis == OR_THETA) return 1.0 / (s2 + c2);",
     "if (basis == OR_THETA) return 1.0 / (s2 > c2 ? s2 : c2);"),
    ("orientation: minor axis not rotated by pi/2",
     "p = th + M_PI / 2;",
     "p = th;"),
    ("select: sector comparison inverted",
     "return or_bound_e(OR_THETA_PRIME, phi) > or_bound_e(OR_THETA, phi) ? OR_THETA_PRIME : OR_THETA;",
     "return or_bound_e(OR_THETA_PRIME, phi) < or_bound_e(OR_THETA, phi) ? OR_THETA_PRIME : OR_THETA;"),
    # third batch: the clamp branch, the support window, the image edge
    ("clamp: rho bound (1 + e)/(1 - e) inverted",
     "double rb = (1 + eb) / (1 - eb);",
     "double rb = (1 - eb) / (1 + eb);"),
    ("clamp: trace not preserved (T = sx^2)",
     "double T = sx * sx + sy * sy;",
     "double T = sx * sx;"),
    ("clamp: eigenvalues swapped",
     "double l1 = T * (1 + e) / 2, l2 = T * (1 - e) / 2;",
     "double l1 = T * (1 - e) / 2, l2 = T * (1 + e) / 2;"),
    ("clamp: C12 sign",
     "C[1] = (l1 - l2) * c * s;",
     "C[1] = -(l1 - l2) * c * s;"),
    ("support: half extent r a/2 -> a/2",
     "sx += 0.5 * r * a[k] * fabs(u[k][0]);",
     "sx += 0.5 * a[k] * fabs(u[k][0]);"),
    ("edge: pixels outside the image replicate instead of zero",
     "if (x < 0 || y < 0 || x >= im->W || y >= im->H) return 0.0;",
     "if (x < 0 || y < 0 || x >= im->W || y >= im->H) return 1.0;"),
    ("direct sum: window clipped one column short",
     "if (x1 > im->W - 1) x1 = im->W - 1;",
     "if (x1 > im->W - 2) x1 = im->W - 2;"),
]


FIRST = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # skip the first FIRST mutations


def main() -> int:
    src = open(os.path.join(ROOT, "oracle", "bsf_oracle.c")).read()
    bad = 0
    with tempfile.TemporaryDirectory() as tmp:
        shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"))
        shutil.copytree(os.path.join(ROOT, "tests"), os.path.join(tmp, "tests"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        for name, old, new in MUTATIONS[FIRST:]:
            assert src.count(old) == 1, name
            with open(os.path.join(tmp, "oracle", "bsf_oracle.c"), "w") as fh:
                fh.write(src.replace(old, new))
            so = os.path.join(tmp, "oracle", "libbsf_oracle.so")
            if os.path.exists(so):
                os.remove(so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "tests/test_oracle_pins.py", "tests/test_accuracy.py"], cwd=tmp,
                               capture_output=True, text=True)
            caught = r.returncode != 0
            bad += not caught
            print("%-45s %s" % (name, "caught" if caught else "NOT CAUGHT"))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
