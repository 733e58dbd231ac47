"""Degenerate and maximum-shape logs at scale, element by element against O1:
(a) one 20M-event case among 1M small ones (the exact format fallback at its
largest), (b) 10M single-event cases (no directly-follows pair at all; one
variant per activity), (c) 5M events sharing one timestamp (ts_bits = 0: every
row of a case ties, so the in-case order is the ingest order)."""
import numpy as np
import pytest

from tests.parity import check_log

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_giant_case_among_small_ones():
    rng = np.random.default_rng(7)
    big = 20_000_000
    lens = rng.integers(1, 12, 1_000_000)
    case = np.concatenate([np.full(big, 1_000_000), np.repeat(np.arange(1_000_000), lens)]).astype(np.int64)
    act = rng.integers(0, 30, case.size)
    ts = rng.integers(0, 10**11, case.size)
    p = rng.permutation(case.size)
    check_log(case[p], act[p], ts[p], 30, n_case_codes=1_000_001)


def test_ten_million_single_event_cases():
    rng = np.random.default_rng(8)
    n = 10_000_000
    check_log(rng.permutation(n).astype(np.int64), rng.integers(0, 64, n), rng.integers(0, 10**12, n), 64,
              n_case_codes=n)


def test_all_rows_share_one_timestamp():
    rng = np.random.default_rng(9)
    n = 5_000_000
    check_log(rng.integers(0, 400_000, n), rng.integers(0, 8, n), np.full(n, 1_600_000_000_000), 8,
              n_case_codes=400_000)
