"""GPU filters vs the oracle (P:126 time filters, P:96-101/P:128 attribute filters)."""
import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from gen.tinylogs import random_log
from tests.parity import assert_parity, collect, to_device_cols
from paper_2204_04898_b200 import pm4g

pytestmark = pytest.mark.gpu


def _log(case, act, ts, A, ncodes, extra=None, sort_first=False):
    c, a, t = to_device_cols(case, act, ts, A)
    log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=ncodes, extra=extra)
    if sort_first:
        log.sort()
    return log


def _expect(case, act, ts, A, keep):
    keep = np.asarray(keep, dtype=bool)
    sub = lambda x: np.asarray(x, dtype=np.int64)[keep]  # noqa: E731
    return oracle.run(sub(case), sub(act), sub(ts), A)


def _check(out_log, r):
    out_log.sort()
    assert_parity(collect(out_log), r)


@pytest.mark.parametrize("sort_first", [False, True])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_time_filter_l1(l1, mode, sort_first):
    rows = l1["rows_ingest_order"]
    case, act, ts = rows["case"], rows["act"], rows["ts"]
    t1, t2 = {0: (0, 15), 1: (0, 20), 2: (90, 200)}[mode]
    log = _log(case, act, ts, 3, 3, sort_first=sort_first)
    out = log.filter_time(t1, t2, mode)
    keep = oracle.filter_time(case, ts, t1, t2, mode)
    _check(out, _expect(case, act, ts, 3, keep))
    ex = l1["expected"]
    if mode == 0:
        sc, sa, st = out.sorted_columns()
        got = [[int(x), int(y), int(z)] for x, y, z in zip(sc.cpu(), sa.cpu(), st.cpu())]
        assert got == ex["filter_events_0_15"]["value"]


@pytest.mark.parametrize("sort_first", [False, True])
@pytest.mark.parametrize("seed", range(0, 60, 3))
def test_time_filters_random(seed, sort_first):
    case, act, ts, A, ncodes = random_log(seed)
    if not case:
        return
    lo, hi = min(ts), max(ts)
    t1, t2 = lo + (hi - lo) // 5, lo + 4 * (hi - lo) // 5
    for mode in (0, 1, 2):
        log = _log(case, act, ts, A, ncodes, sort_first=sort_first)
        out = log.filter_time(t1, t2, mode)
        keep = oracle.filter_time(case, ts, t1, t2, mode)
        _check(out, _expect(case, act, ts, A, keep))


@pytest.mark.parametrize("lazy", [True, False])
@pytest.mark.parametrize("n", [2_500_003, 4_000_000])
def test_events_filter_ring_wraps_element_by_element(n, lazy, monkeypatch):
    """k_filter_cols streams each CTA's 2048-row tiles through a 3-stage TMA ring;
    with n >= 2.5M rows (> 3 x grid tiles) every CTA wraps its ring several times.
    The filtered log, formatted, equals O1 on exactly the kept rows element by
    element (sorted columns, ties broken by ingest order -- so a row dropped,
    duplicated or reordered by the compaction fails), plus every aggregate."""
    if not lazy:   # the materialised compaction (k_filter_cols) instead of the sort's fused pass 0
        monkeypatch.setenv("PM4G_NO_LAZY_FILTER", "1")
    rng = np.random.default_rng(n)
    case = rng.integers(0, n // 8, n)
    act = rng.integers(0, 40, n)
    ts = rng.integers(0, 2000, n)          # many timestamp ties inside a case
    t1, t2 = 300, 1700
    log = _log(case, act, ts, 40, n // 8)
    out = log.filter_time(t1, t2, 0)
    keep = oracle.filter_time(case, ts, t1, t2, 0)
    assert out.n == int(keep.sum())
    _check(out, _expect(case, act, ts, 40, keep))


def test_time_filter_rejects_bad_range():
    log = _log([0, 1], [0, 0], [1, 2], 1, 2)
    with pytest.raises(pm4g.Pm4gError) as e:
        log.filter_time(5, 1)
    assert e.value.status == pm4g.PM4G_EINVAL


def test_filter_removing_everything_and_keeping_everything():
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    log = _log(case, act, ts, L.n_activities, L.n_case_codes)
    none = log.filter_time(0, 1)
    assert none.n == 0
    none.sort()
    cnt, _, _ = none.dfg()
    assert int(cnt.sum()) == 0
    allr = log.filter_time(int(ts.min()), int(ts.max()))
    _check(allr, oracle.run(case, act, ts, L.n_activities))


@pytest.mark.parametrize("sort_first", [False, True])
@pytest.mark.parametrize("level", [0, 1])
@pytest.mark.parametrize("keep", [True, False])
def test_activity_filter(level, keep, sort_first):
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    log = _log(case, act, ts, L.n_activities, L.n_case_codes, sort_first=sort_first)
    out = log.filter_attr(pm4g.PM4G_COL_ACTIVITY, codes=[1, 4, 7], level=level, keep=keep)
    k = oracle.filter_attr(case, act, codes=[1, 4, 7], level=level, keep=keep)
    _check(out, _expect(case, act, ts, L.n_activities, k))


def test_activity_filter_l1_cases(l1):
    rows = l1["rows_ingest_order"]
    log = _log(rows["case"], rows["act"], rows["ts"], 3, 3)
    out = log.filter_attr(pm4g.PM4G_COL_ACTIVITY, codes=[1], level=pm4g.PM4G_LEVEL_CASES)
    out.sort()
    cc, _, _ = out.case_durations()
    assert cc.cpu().tolist() == l1["expected"]["filter_attr_act_B_cases"]["value"]


@pytest.mark.parametrize("sort_first", [False, True])
@pytest.mark.parametrize("level", [0, 1])
def test_extra_columns_with_nulls(level, sort_first):
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    n = case.size
    rng = np.random.default_rng(5)
    res = rng.integers(0, 50, n).astype(np.int64)         # resource codes
    cost = rng.integers(0, 2000, n).astype(np.int64)      # numeric i64
    amt = rng.random(n) * 100.0                           # numeric f64
    valid = (rng.random(n) > 0.1).astype(np.uint8)
    dev = "cuda"
    extra = [pm4g.Extra(pm4g.PM4G_KIND_CODES, torch.as_tensor(res).to(torch.int32).to(dev), None, 50),
             pm4g.Extra(pm4g.PM4G_KIND_I64, torch.as_tensor(cost).to(dev), torch.as_tensor(valid).to(dev)),
             pm4g.Extra(pm4g.PM4G_KIND_F64, torch.as_tensor(amt).to(dev), None)]
    log = _log(case, act, ts, L.n_activities, L.n_case_codes, extra=extra, sort_first=sort_first)
    # cost > 1000 (P:96 example) with nulls that never match
    out = log.filter_attr(1, lo=1001, hi=2**62, level=level)
    k = oracle.filter_attr(case, cost, lo=1001, hi=2**62, valid=valid, level=level)
    _check(out, _expect(case, act, ts, L.n_activities, k))
    out = log.filter_attr(0, codes=[3, 9, 11], level=level, keep=False)
    k = oracle.filter_attr(case, res, codes=[3, 9, 11], level=level, keep=False)
    _check(out, _expect(case, act, ts, L.n_activities, k))
    out = log.filter_attr(2, lo=10.0, hi=55.5, level=level)
    k = oracle.filter_attr(case, amt, lo=10.0, hi=55.5, level=level)
    _check(out, _expect(case, act, ts, L.n_activities, k))
    # chained: attribute filter on the filtered log (extra columns travel with rows)
    out2 = log.filter_attr(1, lo=0, hi=1500, level=0).filter_attr(0, codes=list(range(25)), level=level)
    k1 = oracle.filter_attr(case, cost, lo=0, hi=1500, valid=valid, level=0)
    sub = lambda x: np.asarray(x)[k1]  # noqa: E731
    k2 = oracle.filter_attr(sub(case), sub(res), codes=list(range(25)), level=level)
    r = oracle.run(sub(case)[k2], sub(act)[k2], sub(ts)[k2], L.n_activities)
    _check(out2, r)


def test_kind_mismatch_rejected():
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    extra = [pm4g.Extra(pm4g.PM4G_KIND_I64, torch.zeros(case.size, dtype=torch.int64, device="cuda"))]
    log = _log(case, act, ts, L.n_activities, L.n_case_codes, extra=extra)
    with pytest.raises(pm4g.Pm4gError) as e:
        log.filter_attr(0, codes=[1])
    assert e.value.status == pm4g.PM4G_EINVAL
    with pytest.raises(pm4g.Pm4gError):
        log.filter_attr(5, codes=[1])


def test_contained_subset_of_intersecting():
    """S:486 / S:619 law on the GPU outputs."""
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    log = _log(case, act, ts, L.n_activities, L.n_case_codes)
    lo, hi = int(ts.min()), int(ts.max())
    for j in range(4):
        t1 = lo + (hi - lo) * j // 8
        t2 = t1 + (hi - lo) // 2
        a = log.filter_time(t1, t2, 1).sort()
        b = log.filter_time(t1, t2, 2).sort()
        ca = set(a.case_durations()[0].cpu().tolist())
        cb = set(b.case_durations()[0].cpu().tolist())
        assert ca <= cb


# ---------------------------------------------------------------- the lazy events-mode filter
def _lazy_case(seed, n=300_000):
    rng = np.random.default_rng(seed)
    case = rng.integers(0, n // 7, n)
    act = rng.integers(0, 12, n)
    ts = rng.integers(-10**9, 10**9, n)
    ts[::5] = ts[1]                                    # ties
    return case, act, ts


def test_lazy_filter_chain_and_materialise():
    """pm4g_filter_time (events mode) on an ingested log is lazy: the kept rows
    are selected by the sort's first radix pass over the shared raw columns.
    Filtering it again intersects the ranges; an attribute filter, a case-level
    time filter or a partition materialises it first -- every path equals the
    oracle on exactly the kept rows."""
    case, act, ts = _lazy_case(1)
    A, nc = 12, int(case.max()) + 1
    t1, t2, u1, u2 = -6 * 10**8, 7 * 10**8, -9 * 10**8, 3 * 10**8
    k1 = oracle.filter_time(case, ts, t1, t2, 0)
    k12 = k1 & oracle.filter_time(case, ts, u1, u2, 0)
    # lazy -> lazy (intersected) -> sort
    f = _log(case, act, ts, A, nc).filter_time(t1, t2, 0).filter_time(u1, u2, 0)
    _check(f, _expect(case, act, ts, A, k12))
    # lazy -> attribute filter at case level (materialises)
    f = _log(case, act, ts, A, nc).filter_time(t1, t2, 0)
    g = f.filter_attr(codes=[3, 5], level=pm4g.PM4G_LEVEL_CASES)
    sub = lambda x: np.asarray(x)[k1]  # noqa: E731
    kk = oracle.filter_attr(sub(case), sub(act), codes=[3, 5], level=1)
    assert_parity((g.sort(), collect(g))[1], oracle.run(sub(case)[kk], sub(act)[kk], sub(ts)[kk], A))
    # lazy -> case-level time filter (materialises)
    h = f.filter_time(u1, u2, pm4g.PM4G_TIME_CASES_INTERSECTING)
    kh = oracle.filter_time(sub(case), sub(ts), u1, u2, 2)
    _check(h, oracle.run(sub(case)[kh], sub(act)[kh], sub(ts)[kh], A))
    # the lazy log itself still sorts after all that
    _check(f, _expect(case, act, ts, A, k1))


def test_lazy_filter_outlives_parent_and_edge_ranges():
    """The lazy child shares the parent's (copied, owned) columns: destroying
    the parent first leaves them alive until the child is sorted.  An empty
    range and a range keeping every row work too."""
    case, act, ts = _lazy_case(2)
    A, nc = 12, int(case.max()) + 1
    for t1, t2 in ((-5 * 10**8, 5 * 10**8), (10**9 + 1, 10**9 + 5), (-10**9, 10**9)):
        log = _log(case, act, ts, A, nc)
        f = log.filter_time(t1, t2, 0)
        log.close()
        torch.cuda.synchronize()
        _check(f, _expect(case, act, ts, A, oracle.filter_time(case, ts, t1, t2, 0)))


def test_lazy_filter_then_partition_and_sort_analyze():
    """A lazy log partitioned by case range (materialised) and a lazy log through
    pm4g_sort_analyze: both equal the oracle on the kept rows."""
    case, act, ts = _lazy_case(3)
    A, nc = 12, int(case.max()) + 1
    t1, t2 = -2 * 10**8, 9 * 10**8
    keep = oracle.filter_time(case, ts, t1, t2, 0)
    f = _log(case, act, ts, A, nc).filter_time(t1, t2, 0)
    assert_parity(collect(f, sort_analyze=True), _expect(case, act, ts, A, keep))
    f = _log(case, act, ts, A, nc).filter_time(t1, t2, 0)
    bounds = [0, nc // 3, nc]
    parts = f.partition_by_case(bounds)
    for r, p in enumerate(parts):
        m = keep & (case >= bounds[r]) & (case < bounds[r + 1])
        _check(p, oracle.run(case[m], act[m], ts[m], A))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_create_filtered_equals_create_then_filter(seed):
    """pm4g_log_create_filtered validates every row and builds the kept rows'
    metadata in one pass: the result equals the oracle on the kept rows (P:126,
    S:413), for ranges keeping some, none and all rows; invalid rows outside
    the range are still rejected."""
    case, act, ts = _lazy_case(10 + seed, n=200_000)
    A, nc = 12, int(case.max()) + 1
    for t1, t2 in ((-4 * 10**8, 6 * 10**8), (10**9 + 1, 10**9 + 9), (-10**9, 10**9)):
        c, a, t = to_device_cols(case, act, ts, A)
        f = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=nc, time_filter=(t1, t2))
        keep = oracle.filter_time(case, ts, t1, t2, 0)
        assert f.n == int(keep.sum())
        _check(f, _expect(case, act, ts, A, keep))
    bad = act.copy()
    bad[7] = A + 3
    ts2 = ts.copy()
    ts2[7] = 10**9   # outside the range, still validated
    c, a, t = to_device_cols(case, bad, ts2, A + 4)
    with pytest.raises(pm4g.Pm4gError) as e:
        pm4g.pm4g_log_create(c, a, t, A, n_case_codes=nc, time_filter=(-10**8, 10**8))
    assert e.value.status == pm4g.PM4G_EDATA
