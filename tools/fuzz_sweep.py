"""Longer run of the seeded random sweeps in tests/test_gpu_fuzz.py (tools;
the test suite runs 12 + 6 seeds): device entry vs the C oracle for seeds
[D0, D1), host entry vs device entry for seeds [H0, H1).
Usage: python tools/fuzz_sweep.py [D0 D1 H0 H1] (default 100 180 100 140)"""
import os
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import test_gpu_fuzz as T  # noqa: E402


class _Env:  # the monkeypatch subset the host test uses
    def setenv(self, k, v):
        os.environ[k] = v

    def delenv(self, k, raising=True):
        os.environ.pop(k, None)


d0, d1, h0, h1 = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (100, 180, 100, 140)
bad = 0
for seed in range(d0, d1):
    try:
        T.test_random_sweep_against_oracle(seed)
    except AssertionError as e:
        bad += 1
        print("device entry FAIL", seed, str(e)[:400], flush=True)
for seed in range(h0, h1):
    try:
        T.test_random_host_entry_equals_device_entry(seed, _Env())
    except AssertionError as e:
        bad += 1
        print("host entry FAIL", seed, str(e)[:400], flush=True)
print(f"device seeds {d0}..{d1 - 1} ({(d1 - d0) * 50} cases), host seeds {h0}..{h1 - 1} "
      f"({(h1 - h0) * 25} cases): {bad} failing seeds")
