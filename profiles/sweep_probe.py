"""Probe (not collected): the seeded st-HOSVD sweep of tests/test_gpu_sweep.py over more seeds.
Usage: python profiles/sweep_probe.py FIRST LAST [big]"""
import sys
import traceback
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as o  # noqa: E402
import test_gpu_sweep as t  # noqa: E402

o.load()
a, b = int(sys.argv[1]), int(sys.argv[2])
big = len(sys.argv) > 3
bad = 0
for s in range(a, b):
    try:
        t.test_sthosvd_sweep_vs_oracle(s, big, o)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("FAIL", s, t._case(s, big), repr(e)[:300], flush=True)
print(f"done {b - a} cases, {bad} failed", flush=True)
