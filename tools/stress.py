"""Stress shapes vs the oracle (full parity; run by hand on a GPU box):
(a) one 20M-event case + 1M small cases, (b) 10M single-event cases,
(c) 5M events sharing one timestamp (ties only, ts_bits = 0)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from tests.parity import check_log  # noqa: E402


def run(name, case, act, ts, A):
    t0 = time.time()
    check_log(case, act, ts, A, n_case_codes=int(case.max()) + 1)
    print(f"{name}: {case.size:,} events parity ok ({time.time() - t0:.1f} s incl. oracle)", flush=True)


rng = np.random.default_rng(7)
big = 20_000_000
lens = rng.integers(1, 12, 1_000_000)
case = np.concatenate([np.full(big, 1_000_000), np.repeat(np.arange(1_000_000), lens)]).astype(np.int64)
act = rng.integers(0, 30, case.size)
ts = rng.integers(0, 10**11, case.size)
p = rng.permutation(case.size)
run("(a) giant case", case[p], act[p], ts[p], 30)

n = 10_000_000
run("(b) single-event cases", rng.permutation(n).astype(np.int64), rng.integers(0, 64, n), rng.integers(0, 10**12, n), 64)

n = 5_000_000
run("(c) all ties", rng.integers(0, 400_000, n), rng.integers(0, 8, n), np.full(n, 1_600_000_000_000), 8)
