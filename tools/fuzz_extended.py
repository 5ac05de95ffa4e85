"""One-off extended fuzz (GPU): more seeds of tests/test_gpu_fuzz.py than the suite runs.
python tools/fuzz_extended.py [--shift N]: every seed range moved up by N (new seeds)."""
import argparse
import sys

sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import test_gpu_fuzz as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shift", type=int, default=0)
n = ap.parse_args().shift
bad = 0
for s in range(8 + n, 56 + n):
    try:
        T.test_fuzz_large_images_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL", s, e)
for s in range(32 + n, 160 + n):
    try:
        T.test_fuzz_fused_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL small", s, e)
for s in range(24 + n, 224 + n):
    try:
        T.test_fuzz_global_mode_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL global", s, e)
print("failures", bad)
