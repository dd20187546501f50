"""Stress: many more randomised sessions than the test suite's (same checks,
new seeds): direct-mode sessions vs the host mirror, pack + delta + scatter
vs the oracle.  python tools/stress_random.py [n_direct] [n_pack]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_ctypes import oracle  # test-infrastructure checker only
import test_gpu_parity as t

orc = oracle()
nd = int(sys.argv[1]) if len(sys.argv) > 1 else 200
npk = int(sys.argv[2]) if len(sys.argv) > 2 else 200
t0 = time.time()
for k in range(100, 100 + nd):
    t.test_direct_checkpoint_random_sessions(orc, k)
print(f"direct sessions: {nd} passed ({time.time() - t0:.1f} s)", flush=True)
t0 = time.time()
for k in range(100, 100 + npk):
    t.test_pack_and_delta_random_vs_oracle(orc, k)
print(f"pack + delta + scatter sessions: {npk} passed ({time.time() - t0:.1f} s)", flush=True)
