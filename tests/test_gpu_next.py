"""GPU parity for SURVEY.md 8(f)'s NEXT rows against the oracle:
NEXT-2 per-edge min / max pair durations (pm4g_dfg_minmax, analyze(minmax=True))
and NEXT-1 whole-case filters (pm4g_filter_cases, pm4g_filter_variants)."""
import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from gen.tinylogs import random_log
from tests.parity import assert_parity, collect, to_device_cols
from paper_2204_04898_b200 import pm4g

pytestmark = pytest.mark.gpu


def _sorted_log(case, act, ts, A, ncodes=None):
    c, a, t = to_device_cols(case, act, ts, A)
    if ncodes is None:
        ncodes = (int(np.max(np.asarray(case, dtype=np.int64))) + 1) if len(case) else 1
    log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=ncodes)
    return log.sort()


def _u64(x):
    return x.contiguous().view(-1).cpu().numpy().view(np.uint64)


def _check_minmax(case, act, ts, A, ncodes=None):
    log = _sorted_log(case, act, ts, A, ncodes)
    mn, mx = log.dfg_minmax()
    rmn, rmx = oracle.dfg_minmax(case, act, ts, A)
    assert np.array_equal(_u64(mn), rmn.reshape(-1)), "min differs"
    assert np.array_equal(_u64(mx), rmx.reshape(-1)), "max differs"
    o = log.analyze(minmax=True)
    assert np.array_equal(_u64(o["dur_min"]), rmn.reshape(-1))
    assert np.array_equal(_u64(o["dur_max"]), rmx.reshape(-1))
    r = oracle.run(case, act, ts, A)
    assert np.array_equal(_u64(o["cnt"]), r.cnt.reshape(-1))
    assert np.array_equal(o["dur_sum"].cpu().numpy(), r.sum.reshape(-1))
    o["variants"].close()
    log.close()


# ------------------------------------------------------------------ NEXT-2
def test_minmax_l1(l1):
    r = l1["rows_ingest_order"]
    _check_minmax(r["case"], r["act"], r["ts"], 3, 3)


@pytest.mark.parametrize("seed", range(0, 40, 2))
def test_minmax_random(seed):
    case, act, ts, A, ncodes = random_log(seed)
    _check_minmax(case, act, ts, A, ncodes)


@pytest.mark.parametrize("name", ["tiny", "roadtraffic", "bpic2019"])
def test_minmax_configs(name):
    L = generate(CONFIGS[name])
    _check_minmax(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities, L.n_case_codes)


@pytest.mark.parametrize("A", [72, 200, 256, 300])
def test_minmax_hash_mode_and_wide_gaps(A):
    """A > 71 takes the shared-memory hash tables; gaps >= 2^32 take the global
    min / max path; one 50k-event case makes an oversized (unstaged) tile."""
    rng = np.random.default_rng(A)
    lens = rng.integers(1, 25, 4000)
    case = np.repeat(np.arange(4000, dtype=np.int64), lens)
    act = rng.integers(0, A, case.size)
    gaps = np.where(rng.random(case.size) < 0.05, rng.integers(2**32, 2**36, case.size),
                    rng.integers(0, 10**6, case.size))
    ts = np.cumsum(gaps).astype(np.int64)
    big = 50_000
    case = np.concatenate([case, np.full(big, 4000)])
    act = np.concatenate([act, rng.integers(0, 3, big)])
    ts = np.concatenate([ts, rng.integers(0, 10**9, big)])
    p = rng.permutation(case.size)
    _check_minmax(case[p], act[p], ts[p], A, 4001)


def test_minmax_sharded_merge_law():
    """Sharding by case range: the global min / max is the min / max over shards of
    the edges that occur there (what the ncclMin / ncclMax allreduce computes)."""
    L = generate(CONFIGS["bpic2019"])
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    bounds = [0, 60_000, 150_000, CONFIGS["bpic2019"].n_cases]
    mn = np.full(A * A, np.iinfo(np.uint64).max, np.uint64)
    mx = np.zeros(A * A, np.uint64)
    for lo, hi in zip(bounds, bounds[1:]):
        sel = (case >= lo) & (case < hi)
        log = _sorted_log(case[sel], act[sel], ts[sel], A, L.n_case_codes)
        a, b = log.dfg_minmax()
        cnt, _, _ = log.dfg(with_mean=False)
        occ = _u64(cnt) > 0
        mn[occ] = np.minimum(mn[occ], _u64(a)[occ])
        mx[occ] = np.maximum(mx[occ], _u64(b)[occ])
        log.close()
    mn[mn == np.iinfo(np.uint64).max] = 0
    rmn, rmx = oracle.dfg_minmax(case, act, ts, A)
    assert np.array_equal(mn, rmn.reshape(-1)) and np.array_equal(mx, rmx.reshape(-1))


# ------------------------------------------------------------------ NEXT-1
def _filter_check(case, act, ts, A, log, kind, codes=None, lo=0, hi=0, keep=True, ncodes=None):
    out = log.filter_cases(kind, codes=codes, lo=lo, hi=hi, keep=keep)
    m = oracle.filter_cases(case, act, ts, kind, codes=codes, lo=lo, hi=hi, keep=keep)
    sub = lambda x: np.asarray(x, dtype=np.int64)[m]  # noqa: E731
    r = oracle.run(sub(case), sub(act), sub(ts), A)
    assert_parity(collect(out), r)
    out.close()


def test_case_filters_l1(l1):
    rows, ex = l1["rows_ingest_order"], l1["expected"]
    case, act, ts = rows["case"], rows["act"], rows["ts"]
    log = _sorted_log(case, act, ts, 3, 3)

    def cases_of(out):
        C = out.info().n_cases
        cc, _, _ = out.case_durations()
        return sorted(int(x) for x in cc[:C].cpu())

    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_SIZE, lo=3, hi=3)) == ex["filter_case_size_3_3"]["value"]
    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_THROUGHPUT, lo=0, hi=10)) == ex["filter_throughput_0_10"]["value"]
    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_PATHS, codes=[0, 2])) == ex["filter_paths_keep_AC"]["value"]
    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_START_IN, codes=[0])) == ex["filter_start_in_A"]["value"]
    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_END_IN, codes=[1])) == ex["filter_end_in_B"]["value"]
    assert cases_of(log.filter_variants([[0, 2]])) == ex["filter_variants_keep_AC"]["value"]
    assert cases_of(log.filter_cases(pm4g.PM4G_CASE_PATHS, codes=[])) == []
    assert cases_of(log.filter_variants([], keep=False)) == [0, 1, 2]
    for bad in (dict(kind=pm4g.PM4G_CASE_SIZE, lo=4, hi=3), dict(kind=pm4g.PM4G_CASE_PATHS, codes=[0, 1, 2])):
        with pytest.raises(pm4g.Pm4gError) as e:
            log.filter_cases(**bad)
        assert e.value.status == pm4g.PM4G_EINVAL
    c, a, t = to_device_cols(case, act, ts, 3)
    unsorted = pm4g.pm4g_log_create(c, a, t, 3, n_case_codes=3)
    with pytest.raises(pm4g.Pm4gError):
        unsorted.filter_cases(pm4g.PM4G_CASE_SIZE, lo=0, hi=1)


@pytest.mark.parametrize("seed", range(0, 30, 3))
def test_case_filters_random(seed):
    case, act, ts, A, ncodes = random_log(seed)
    if not case:
        return
    rng = np.random.default_rng(seed)
    log = _sorted_log(case, act, ts, A, ncodes)
    codes = rng.integers(0, A + 1, 2).tolist()            # may include a code >= A (never matches)
    pairs = rng.integers(0, A, 4).tolist()
    dur = [t for t in ts]
    span = max(dur) - min(dur)
    for keep in (True, False):
        _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_START_IN, codes=codes, keep=keep)
        _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_END_IN, codes=codes, keep=keep)
        _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_SIZE, lo=2, hi=6, keep=keep)
        _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_THROUGHPUT, lo=0, hi=span // 3, keep=keep)
        _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_PATHS, codes=pairs, keep=keep)


@pytest.mark.parametrize("name", ["tiny", "bpic2019"])
def test_case_filters_configs(name):
    L = generate(CONFIGS[name])
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    log = _sorted_log(case, act, ts, A, L.n_case_codes)
    _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_SIZE, lo=3, hi=8)
    _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_THROUGHPUT, lo=3_600_000, hi=86_400_000 * 3)
    _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_PATHS, codes=[0, 1, 1, 2, 5, 5], keep=False)
    _filter_check(case, act, ts, A, log, pm4g.PM4G_CASE_START_IN, codes=[0, 3])


def _variant_check(case, act, ts, A, seqs, keep, ncodes=None):
    log = _sorted_log(case, act, ts, A, ncodes)
    out = log.filter_variants(seqs, keep=keep)
    m = oracle.filter_variants(case, act, ts, seqs, keep=keep)
    sub = lambda x: np.asarray(x, dtype=np.int64)[m]  # noqa: E731
    assert_parity(collect(out), oracle.run(sub(case), sub(act), sub(ts), A))


@pytest.mark.parametrize("weak", [False, True])
@pytest.mark.parametrize("name", ["tiny", "bpic2019"])
def test_variant_filter(name, weak, monkeypatch):
    """Query sequences are hashed on the host like A8 and verified exactly; with
    PM4G_DEBUG_WEAK_HASH=1 every key collides and only the verification decides."""
    if weak:
        monkeypatch.setenv("PM4G_DEBUG_WEAK_HASH", "1")
    L = generate(CONFIGS[name])
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    r = oracle.run(case, act, ts, A)
    vs = list(r.variants())
    seqs = vs[:3] + vs[-2:] + [[0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]] + [[A + 3]]   # unseen / invalid: ignored
    for keep in (True, False):
        _variant_check(case, act, ts, A, seqs, keep, L.n_case_codes)


@pytest.mark.parametrize("seed", range(0, 24, 4))
def test_variant_filter_random(seed):
    case, act, ts, A, ncodes = random_log(seed)
    if not case:
        return
    r = oracle.run(case, act, ts, A)
    seqs = list(r.variants())[::2]
    _variant_check(case, act, ts, A, seqs, True, ncodes)
    _variant_check(case, act, ts, A, seqs, False, ncodes)


# ------------------------------------------------------------------ NEXT-3: EFG + temporal profile
def _check_efg(case, act, ts, A, ncodes=None):
    log = _sorted_log(case, act, ts, A, ncodes)
    g = log.efg()
    r = oracle.efg(case, act, ts, A)
    for k_gpu, k_ref in (("cnt", "cnt"), ("sum", "sum"), ("sumsq_lo", "sq_lo"), ("sumsq_hi", "sq_hi")):
        assert np.array_equal(_u64(g[k_gpu]), r[k_ref].reshape(-1)), k_gpu
    # R22: same IEEE operations on both sides -> identical doubles
    assert np.array_equal(g["mean"].cpu().numpy().reshape(-1), r["mean"].reshape(-1))
    assert np.array_equal(g["stdev"].cpu().numpy().reshape(-1), r["stdev"].reshape(-1))
    log.close()


def test_efg_l1(l1):
    rows = l1["rows_ingest_order"]
    _check_efg(rows["case"], rows["act"], rows["ts"], 3, 3)


@pytest.mark.parametrize("seed", range(0, 40, 2))
def test_efg_random(seed):
    case, act, ts, A, ncodes = random_log(seed)
    _check_efg(case, act, ts, A, ncodes)


@pytest.mark.parametrize("name", ["tiny", "roadtraffic", "bpic2019"])
def test_efg_configs(name):
    L = generate(CONFIGS[name])
    _check_efg(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities, L.n_case_codes)


@pytest.mark.parametrize("A", [72, 256, 300])
def test_efg_hash_mode_long_cases_wide_gaps(A):
    """A > 71: hash tables; gaps >= 2^32: the global 128-bit path; a 3000-event
    case makes an unstaged tile walked case by case from global memory."""
    rng = np.random.default_rng(A + 1)
    lens = rng.integers(1, 20, 1500)
    case = np.repeat(np.arange(1500, dtype=np.int64), lens)
    act = rng.integers(0, A, case.size)
    gaps = np.where(rng.random(case.size) < 0.05, rng.integers(2**32, 2**34, case.size),
                    rng.integers(0, 10**6, case.size))
    ts = np.cumsum(gaps).astype(np.int64)
    big = 3000
    case = np.concatenate([case, np.full(big, 1500)])
    act = np.concatenate([act, rng.integers(0, 4, big)])
    ts = np.concatenate([ts, rng.integers(0, 2**40, big)])
    p = rng.permutation(case.size)
    _check_efg(case[p], act[p], ts[p], A, 1501)
