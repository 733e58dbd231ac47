"""pm4g_sort_analyze with PM4G_DEBUG_POISON_FORMAT=1: the formatted activity column
is filled with 0xff before k_format and checked after it, so a row left unwritten
before the deferred exact fallback fails the call.  Logs with fallback cases: one
longer than the in-tile ranking takes (> 1024 rows), one running far past a tile
end across several tiles, and many just past the limit.  Run by
tests/test_gpu_parity.py in a subprocess (the hook is read once per process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PM4G_DEBUG_POISON_FORMAT"] = "1"

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from tests.parity import assert_parity, gpu_run  # noqa: E402

rng = np.random.default_rng(11)
for n_big, big_len, n in [(1, 3000, 40_000), (1, 20_000, 60_000), (6, 1100, 50_000), (2, 9000, 30_000)]:
    case = rng.integers(0, 5000, n)
    start = 0
    for b in range(n_big):
        case[start:start + big_len] = 7 + 997 * b
        start += big_len
    act = rng.integers(0, 13, n)
    ts = rng.integers(0, 10**7, n)
    ts[::9] = 5
    p = rng.permutation(n)
    case, act, ts = case[p], act[p], ts[p]
    assert_parity(gpu_run(case, act, ts, 13, n_case_codes=5000, sort_analyze=True), oracle.run(case, act, ts, 13))
print("poison_run ok")
