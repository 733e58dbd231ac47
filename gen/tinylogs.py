"""Seeded random tiny logs for property tests (<= 50 cases, <= 20 events
per case, <= 8 activities).  Pure Python ``random``; holds none of the method's
arithmetic.  Varies the number of cases, events per case, activities, timestamp
ties, negative timestamps, sparse case codes and single-event cases.
"""
from __future__ import annotations

import random


def random_log(seed: int, max_cases: int = 50, max_len: int = 20, max_acts: int = 8):
    """Returns (case, act, ts, n_activities, n_case_codes) as Python lists."""
    rng = random.Random(seed)
    A = rng.randint(1, max_acts)
    C = rng.randint(0, max_cases)
    sparse = rng.random() < 0.3          # leave gaps in the case-code range
    n_codes = C * (3 if sparse else 1) + rng.randint(0, 3)
    codes = rng.sample(range(max(n_codes, 1)), C) if C else []
    tie_p = rng.choice([0.0, 0.1, 0.5, 1.0])
    base = rng.choice([0, -10**6, 10**12, -(10**15)])
    rows = []
    for c in codes:
        L = 1 if rng.random() < 0.2 else rng.randint(1, max_len)
        t = base + rng.randint(0, 10**6)
        for _ in range(L):
            rows.append((c, rng.randrange(A), t))
            if rng.random() >= tie_p:
                t += rng.randint(1, 10**5)
    rng.shuffle(rows)
    case = [r[0] for r in rows]
    act = [r[1] for r in rows]
    ts = [r[2] for r in rows]
    return case, act, ts, A, max(n_codes, 1)
