"""One-off extended fuzz (GPU): more seeds of tests/test_gpu_fuzz.py than the suite runs."""
import sys, traceback
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import test_gpu_fuzz as T
bad = 0
for s in range(8, 56):
    try:
        T.test_fuzz_large_images_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL", s, e)
for s in range(32, 160):
    try:
        T.test_fuzz_fused_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL small", s, e)
for s in range(24, 224):
    try:
        T.test_fuzz_global_mode_vs_oracle(s)
    except AssertionError as e:
        bad += 1; print("FAIL global", s, e)
print("failures", bad)
