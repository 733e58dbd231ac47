"""GPU parity: the CUDA path (through the C-ABI) vs the oracle O1, element by element.

Integer outputs bit-exact; fp64 means within 1e-12 relative (north_star).
"""
import os

import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from gen.tinylogs import random_log
from tests.parity import assert_parity, check_log, gpu_run, to_device_cols
from paper_2204_04898_b200 import pm4g

pytestmark = pytest.mark.gpu


def _l1(l1):
    r = l1["rows_ingest_order"]
    return r["case"], r["act"], r["ts"], l1["n_activities"]


def test_l1_fixture(l1):
    g, r = check_log(*_l1(l1))
    ex = l1["expected"]
    assert g["dur"].tolist() == ex["throughput_ms"]["value"]
    assert g["cnt"][0, 1] == 2 and g["cnt"][1, 2] == 2 and g["cnt"][0, 2] == 1


def test_l1_separate_calls(l1):
    case, act, ts, A = _l1(l1)
    g = gpu_run(case, act, ts, A, fused=False)
    assert_parity(g, oracle.run(case, act, ts, A))


@pytest.mark.parametrize("seed", range(200))
def test_random_tiny_logs(seed):
    case, act, ts, A, ncodes = random_log(seed)
    check_log(case, act, ts, A, n_case_codes=ncodes)


@pytest.mark.parametrize("name", ["tiny", "roadtraffic", "bpic2019", "bpic2018"])
def test_configs_full_size(name):
    L = generate(CONFIGS[name])
    g, r = check_log(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities,
                     n_case_codes=L.n_case_codes)
    if name == "roadtraffic":
        assert len(r.v_count) == 231 and g["v_count"].size == 231
    if name == "bpic2019":
        assert g["v_count"].size == 11_973


# ---------------------------------------------------------------- edge cases
def test_empty_log():
    g = gpu_run([], [], [], 4, n_case_codes=1)
    assert g["cnt"].sum() == 0 and g["v_count"].size == 0 and g["case_code"].size == 0


def test_single_event():
    check_log([3], [1], [42], 2, n_case_codes=4)


def test_one_case_many_events():
    rng = np.random.default_rng(0)
    n = 20000
    check_log([7] * n, rng.integers(0, 5, n).tolist(), rng.integers(0, 1000, n).tolist(), 5)


def test_all_same_activity_and_timestamp():
    rng = np.random.default_rng(1)
    n = 9000
    case = rng.integers(0, 300, n)
    check_log(case.tolist(), [0] * n, [5] * n, 1)


@pytest.mark.parametrize("A", [1, 2, 255, 256, 257, 1000])
def test_activity_widths(A):
    rng = np.random.default_rng(A)
    n = 30000
    case = rng.integers(0, 2000, n)
    act = rng.integers(0, A, n)
    ts = rng.integers(-10**9, 10**9, n)
    check_log(case.tolist(), act.tolist(), ts.tolist(), A)


@pytest.mark.parametrize("n", [4095, 4096, 4097, 8191, 8193, 3 * 4096 + 1, 65537])
def test_ragged_tiles(n):
    rng = np.random.default_rng(n)
    case = rng.integers(0, max(1, n // 7), n)
    act = rng.integers(0, 9, n)
    ts = rng.integers(0, 10**6, n)
    check_log(case.tolist(), act.tolist(), ts.tolist(), 9)


def test_max_case_code_and_sparse_codes():
    codes = np.array([0, 5, 2**32 - 2, 2**31, 77], dtype=np.int64)
    rng = np.random.default_rng(3)
    case = rng.choice(codes, 5000)
    act = rng.integers(0, 4, 5000)
    ts = rng.integers(0, 10**9, 5000)
    check_log(case.tolist(), act.tolist(), ts.tolist(), 4, n_case_codes=2**32 - 1)


def test_extreme_timestamps_wide_span():
    """ts span near 2^63 with a single case code: key = 63-64 ts bits, 0 case bits."""
    ts = [-(2**62), 2**62, 0, 5, -5, 2**62 - 1]
    check_log([1] * 6, [0, 1, 0, 1, 0, 1], ts, 2)


def test_all_ones_key_ties():
    """key_bits = 64 with rows on the all-ones key (max case, max ts), tied: the
    format rank falls back to the two-compare form there (no key + 1)."""
    big, small = 2**63 - 1, -(2**63)
    check_log([1] * 7, [0, 1, 2, 1, 0, 2, 1], [big, small, big, 0, big, small, 5], 3)
    m = 2**62 - 1   # 1 case bit + 63 ts bits; case 3 at ts m is the all-ones key
    check_log([3, 2, 3, 3, 2, 3], [0, 1, 2, 1, 0, 2], [m, -(2**62), m, 0, m, m], 3)


def test_wide_key_small():
    """case_bits + ts_bits > 64 (here 32 + 64): the wide path
    keys on ts - ts_min alone and carries the case per row; results equal O1."""
    c, a, t = [0, 2**31, 5, 2**31, 0, 5, 5], [0, 1, 0, 2, 1, 1, 0], [-(2**62), 2**62, 0, -7, 3, 0, 0]
    g, r = check_log(c, a, t, 3, n_case_codes=2**32 - 1)
    c2, a2, t2 = to_device_cols(c, a, t, 3)
    log = pm4g.pm4g_log_create(c2, a2, t2, 3, n_case_codes=2**32 - 1)
    info = log.info()
    assert info.key_bits > 64 and info.case_bits == 32
    log.close()


def test_wide_key_with_extra_columns_and_filters():
    """A wide log with an extra column (ingest-row perm and case payload both
    travel) and the formatted-log filters / re-segmentation on a wide log."""
    from tests.parity import collect
    rng = np.random.default_rng(5)
    n = 30_000
    case = rng.integers(0, 40_000, n) * 97            # codes up to ~3.9e6: 22 case bits
    act = rng.integers(0, 6, n)
    ts = rng.integers(-(2**50), 2**50, n)             # 51 ts bits: 73-bit composite key
    ts[::7] = ts[3]                                   # ties
    c, a, t = to_device_cols(case, act, ts, 6)
    ex = [pm4g.Extra(pm4g.PM4G_KIND_I64, torch.as_tensor(rng.integers(0, 100, n)).cuda())]
    log = pm4g.pm4g_log_create(c, a, t, 6, n_case_codes=int(case.max()) + 1, extra=ex)
    assert log.info().key_bits > 64
    log.sort()
    assert_parity(collect(log), oracle.run(case, act, ts, 6))
    # formatted wide log -> events-mode time filter -> re-segmented wide log
    t1, t2 = -(2**49), 2**49
    f = log.filter_time(t1, t2, pm4g.PM4G_TIME_EVENTS)
    keep = oracle.filter_time(case, ts, t1, t2, oracle.EVENTS)
    assert_parity(collect(f), oracle.run(case[keep], act[keep], ts[keep], 6))
    # case-level attribute filter on the wide formatted log
    g = log.filter_attr(codes=[2], level=pm4g.PM4G_LEVEL_CASES)
    keep = oracle.filter_attr(case, act, codes=[2], level=1)
    assert_parity(collect(g), oracle.run(case[keep], act[keep], ts[keep], 6))


@pytest.mark.parametrize("long_case", [False, True])
def test_wide_key_fallback_and_sort_analyze(long_case):
    """Wide logs through pm4g_sort_analyze (non-deferred for wide) including cases
    longer than 1024 rows (the batched exact fallback with 64-bit keys)."""
    rng = np.random.default_rng(17)
    n = 50_000
    case = rng.integers(0, 2**24, n)
    if long_case:
        case[:5000] = 12345
        case[5000:7000] = 2**24 - 1
    ts = rng.integers(-(2**60), 2**60, n)
    ts[:5000:3] = 42                                   # ties inside the long case
    act = rng.integers(0, 9, n)
    p = rng.permutation(n)
    case, act, ts = case[p], act[p], ts[p]
    assert_parity(gpu_run(case, act, ts, 9, n_case_codes=2**24, sort_analyze=True),
                  oracle.run(case, act, ts, 9))


def test_validation_errors():
    c, a, t = to_device_cols([0, 1, 9], [0, 1, 0], [1, 2, 3], 2)
    with pytest.raises(pm4g.Pm4gError) as e:
        pm4g.pm4g_log_create(c, a, t, 2, n_case_codes=5)          # case 9 >= 5
    assert e.value.status == pm4g.PM4G_EDATA and "row 2" in str(e.value)
    c, a, t = to_device_cols([0, 1, 2], [0, 3, 0], [1, 2, 3], 4)
    with pytest.raises(pm4g.Pm4gError) as e:
        pm4g.pm4g_log_create(c, a, t, 3, n_case_codes=5)          # act 3 >= 3
    assert e.value.status == pm4g.PM4G_EDATA


def test_unsorted_log_rejected_by_aggregates():
    c, a, t = to_device_cols([0, 1], [0, 1], [1, 2], 2)
    log = pm4g.pm4g_log_create(c, a, t, 2)
    with pytest.raises(pm4g.Pm4gError) as e:
        log.dfg()
    assert e.value.status == pm4g.PM4G_EINVAL


def test_host_input_path(l1):
    """PM4G_HOST_INPUT: columns in host memory are copied inside the call."""
    case, act, ts, A = _l1(l1)
    c, a, t = to_device_cols(case, act, ts, A, device=None)
    log = pm4g.pm4g_log_create(c.pin_memory(), a.pin_memory(), t.pin_memory(), A, n_case_codes=3)
    log.sort()
    cnt, sm, mean = log.dfg()
    assert cnt.cpu().numpy()[0, 1] == 2 and sm.cpu().numpy()[1, 2] == 60


def test_sort_idempotent_and_deterministic():
    L = generate(CONFIGS["tiny"])
    c, a, t = to_device_cols(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities)
    outs = []
    for _ in range(3):
        log = pm4g.pm4g_log_create(c, a, t, L.n_activities, n_case_codes=L.n_case_codes)
        log.sort()
        log.sort()
        from tests.parity import collect
        outs.append(collect(log))
    for k in outs[0]:
        assert np.array_equal(outs[0][k], outs[1][k]) and np.array_equal(outs[0][k], outs[2][k]), k


def test_weak_hash_collisions_resolved_exactly(monkeypatch):
    """PM4G_DEBUG_WEAK_HASH=1 reduces the variant key to 4 bits: every bucket collides,
    the verify-and-rekey rounds must still give the exact variant multiset."""
    monkeypatch.setenv("PM4G_DEBUG_WEAK_HASH", "1")
    L = generate(CONFIGS["tiny"])
    check_log(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities, n_case_codes=L.n_case_codes)
    case, act, ts, A, ncodes = random_log(11)
    check_log(case, act, ts, A, n_case_codes=ncodes)


@pytest.mark.parametrize("cap", ["64", "1024"])
def test_variant_table_regrowth(monkeypatch, cap):
    """PM4G_DEBUG_VARIANT_CAP forces a first variant table far smaller than the number
    of distinct sequences: the load limit must trip, the follow-on kernels must skip
    the abandoned table, and the regrown table must give the exact variant multiset."""
    monkeypatch.setenv("PM4G_DEBUG_VARIANT_CAP", cap)
    for name in ("tiny", "roadtraffic", "bpic2019"):
        L = generate(CONFIGS[name])
        check_log(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities, n_case_codes=L.n_case_codes)
    monkeypatch.setenv("PM4G_DEBUG_WEAK_HASH", "1")
    case, act, ts, A, ncodes = random_log(12)
    check_log(case, act, ts, A, n_case_codes=ncodes)


@pytest.mark.parametrize("A", [92, 200, 256])
def test_hash_table_flush_exact(A):
    """A > 91 takes k_aggregate's TAB_HASH mode (a per-CTA shared-memory hash table
    of u32 counts and u32 lo / hi duration sums, flushed once per CTA with 64-bit
    atomics).  One case repeats a self-loop ~200k times (one oversized tile, read
    from global memory, and a 3.2e5-row exact-fallback case in the sort) and
    another alternates two activities, so single edges take ~1e5 increments inside
    one CTA and the u32 duration words carry into the high word; ordinary random
    cases fill the rest.  Counts and sums must match the oracle exactly."""
    rng = np.random.default_rng(A)
    lens = rng.integers(1, 30, 5000)
    case = np.repeat(np.arange(5000, dtype=np.int64), lens)
    act = rng.integers(0, A, case.size).astype(np.int64)
    ts = rng.integers(0, 10**9, case.size).astype(np.int64)
    big = 200_003
    c_big = np.full(big, 6000, np.int64)
    a_big = np.full(big, A - 1, np.int64)
    t_big = np.cumsum(rng.integers(0, 5, big)).astype(np.int64) + 1_000
    alt = 70_001
    c_alt = np.full(alt, 6001, np.int64)
    a_alt = np.where(np.arange(alt) % 2 == 0, 3, A - 2).astype(np.int64)
    t_alt = np.arange(alt, dtype=np.int64) * 7 + 5
    case = np.concatenate([case, c_big, c_alt])
    act = np.concatenate([act, a_big, a_alt])
    ts = np.concatenate([ts, t_big, t_alt])
    p = rng.permutation(case.size)
    check_log(case[p], act[p], ts[p], A, n_case_codes=6002)


@pytest.mark.parametrize("ts_bits,case_bits", [(0, 12), (1, 20), (24, 8), (31, 9), (32, 10), (33, 18),
                                               (40, 24), (56, 8), (62, 2), (63, 1), (64, 0), (20, 32),
                                               (45, 24), (64, 24), (40, 32), (64, 32), (57, 8), (33, 32)])
def test_digit_shift_boundaries(ts_bits, case_bits):
    """Onesweep digits sit at shift = ts_bits + 8p: the 64-bit path (shift < 32),
    the high-word path (32 <= shift < 64) and the single-case guard (shift 64);
    pass 0 takes its digit from the case column.  Spans are chosen so the
    composite key has exactly ts_bits + case_bits bits."""
    rng = np.random.default_rng(ts_bits * 100 + case_bits)
    n = 6000
    ncases = 1 << case_bits if case_bits < 32 else 2**32 - 1
    case = rng.integers(0, min(ncases, 3000), n).astype(np.int64)
    if case_bits == 32:
        case[:2] = [0, 2**32 - 2]            # the full 32-bit case range
    elif case_bits > 0:
        case[:2] = [0, ncases - 1]
    base = -(2**63) if ts_bits == 64 else -(2**(max(ts_bits, 1) - 1))
    span = (2**64 - 1) if ts_bits == 64 else ((1 << ts_bits) - 1 if ts_bits else 0)
    ts = (base + rng.integers(0, span + 1 if span < 2**63 else 2**63, n, dtype=np.int64)
          if span else np.full(n, 7, np.int64))
    if span:
        ts[2], ts[3] = base, base + span if span < 2**63 else 2**63 - 1
        if ts_bits == 64:
            ts[3] = 2**63 - 1
    act = rng.integers(0, 5, n)
    # case_bits + ts_bits > 64 takes the wide path (key = ts - ts_min, case per row)
    check_log(case.tolist(), act.tolist(), ts.tolist(), 5, n_case_codes=int(case.max()) + 1)


@pytest.mark.parametrize("act_bits", [8, 16])
def test_persistent_prefetch_key_passes(monkeypatch, act_bits):
    """Key passes above 2 x SMs tiles run the persistent, prefetching onesweep
    (k_onesweep_pf: next tile TMA-loaded into a second buffer; pass 0 with a u8
    activity: k_onesweep_pf0); below, or with PM4G_NO_OS_PF, the one-tile-per-CTA
    kernel.  Both must equal the oracle on a
    log with 3 case digits (2 key passes), several tiles per CTA and a ragged
    last tile."""
    rng = np.random.default_rng(act_bits)
    n = 1_500_007                       # 367 tiles of 4096 + a ragged tail
    ncases = 300_000                    # 19 case bits -> pass 0 + 2 key passes
    case = rng.integers(0, ncases, n)
    A = 200 if act_bits == 8 else 700   # u8 / u16 activities
    act = rng.integers(0, A, n)
    ts = rng.integers(0, 10**9, n)
    r = oracle.run(case, act, ts, A)
    assert_parity(gpu_run(case, act, ts, A, n_case_codes=ncases), r)
    monkeypatch.setenv("PM4G_NO_OS_PF", "1")
    assert_parity(gpu_run(case, act, ts, A, n_case_codes=ncases), r)


# ---------------------------------------------------------------- pm4g_sort_analyze
@pytest.mark.parametrize("seed", range(0, 200, 20))
def test_sort_analyze_random_tiny_logs(seed):
    case, act, ts, A, ncodes = random_log(seed)
    assert_parity(gpu_run(case, act, ts, A, n_case_codes=ncodes, sort_analyze=True),
                  oracle.run(case, act, ts, A))


@pytest.mark.parametrize("shape", ["one_long_case", "long_cases_across_tiles", "ragged", "many_long_with_ties"])
def test_sort_analyze_fallback_cases(shape):
    """Cases k_format leaves to the exact fallback (longer than 1024 rows, or running
    far past a tile): pm4g_sort_analyze finds them at the analysis' synchronisation,
    sorts them exactly and recomputes -- results equal the oracle's."""
    rng = np.random.default_rng(7)
    if shape == "one_long_case":
        n = 5000
        case = np.zeros(n, np.int64)
    elif shape == "long_cases_across_tiles":
        n = 40_000
        case = np.repeat(np.arange(20), n // 20)[rng.permutation(n)]   # 2000-row cases
    elif shape == "ragged":
        n = 3 * 4096 + 17
        case = rng.integers(0, n // 9, n)
        case[: 3000] = 5                                               # one 3000+-row case
        case = case[rng.permutation(n)]
    else:   # 60 fallback cases (1100-3000 rows) among short ones, timestamps with many ties:
        lens = np.concatenate([rng.integers(1100, 3000, 60), rng.integers(1, 20, 20_000)])
        case = np.repeat(rng.permutation(lens.size), lens)             # the batched exact sort
        n = case.size
        case = case[rng.permutation(n)]
    act = rng.integers(0, 7, n)
    ts = rng.integers(0, 10**7 if shape != "many_long_with_ties" else 50, n)
    assert_parity(gpu_run(case, act, ts, 7, n_case_codes=int(case.max()) + 1, sort_analyze=True),
                  oracle.run(case, act, ts, 7))


@pytest.mark.parametrize("name", ["bpic2019", "bpic2018"])
def test_sort_analyze_config(name):
    L = generate(CONFIGS[name])
    c, a, t = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    assert_parity(gpu_run(c, a, t, L.n_activities, n_case_codes=L.n_case_codes, sort_analyze=True),
                  oracle.run(c, a, t, L.n_activities))


@pytest.mark.parametrize("long_case", [False, True])
def test_sort_analyze_with_extra_columns(long_case):
    """Logs with extra columns take pm4g_sort_analyze's non-deferred path (the extra
    columns are gathered by the final order): results equal the oracle's."""
    from tests.parity import collect
    rng = np.random.default_rng(11)
    n = 20_000
    case = rng.integers(0, 2_000, n)
    if long_case:
        case[:3000] = 7                                  # a 3000+-row case: the exact fallback
        case = case[rng.permutation(n)]
    act = rng.integers(0, 9, n)
    ts = rng.integers(0, 10**8, n)
    c, a, t = to_device_cols(case, act, ts, 9)
    ex = [pm4g.Extra(pm4g.PM4G_KIND_I64, torch.as_tensor(rng.integers(0, 100, n)).cuda())]
    log = pm4g.pm4g_log_create(c, a, t, 9, n_case_codes=2_000, extra=ex)
    g = collect(log, sort_analyze=True)
    log.close()
    assert_parity(g, oracle.run(case, act, ts, 9))


def test_sort_analyze_fallback_over_stale_allocator_blocks():
    """pm4g_sort_analyze analyses the provisional order before the exact fallback
    runs; the rows of fallback cases must hold valid activity codes then, not the
    previous contents of a recycled allocator block.  A first log of the same size
    with every activity = 255 (A = 256) is sorted and destroyed, so its blocks (act
    bytes 0xFF) return to the library's cache; the second log (A = 7, fallback
    cases) reuses them.  Results equal the oracle's and no CUDA error is raised."""
    rng = np.random.default_rng(3)
    n = 40_000
    case = np.repeat(np.arange(20), n // 20)[rng.permutation(n)]        # 2000-row cases
    for _ in range(2):
        c, a, t = to_device_cols(case, np.full(n, 255), rng.integers(0, 10**7, n), 256)
        log = pm4g.pm4g_log_create(c, a, t, 256, n_case_codes=20)
        log.sort()
        torch.cuda.synchronize()
        log.close()
    act = rng.integers(0, 7, n)
    ts = rng.integers(0, 10**7, n)
    assert_parity(gpu_run(case, act, ts, 7, n_case_codes=20, sort_analyze=True), oracle.run(case, act, ts, 7))
    torch.cuda.synchronize()


@pytest.mark.parametrize("ts_range", [1, 3, 40, 10**4])
@pytest.mark.parametrize("extras", [False, True])
def test_format_tie_groups(ts_range, extras):
    """k_format ranks rows of narrow cases by #(smaller keys) only: rows with
    equal keys claim one slot and are laid out in ingest order afterwards (a
    per-tile list of tie groups, or in place once the list is full).  Cases of
    1-300 rows with timestamps from a small range give from a few tie groups per
    tile (listed) to thousands (list overflow); results equal the oracle's
    (ties keep the absolute index order)."""
    rng = np.random.default_rng(ts_range)
    lens = np.concatenate([rng.integers(1, 30, 15_000), rng.integers(100, 300, 300)])
    case = np.repeat(rng.permutation(lens.size), lens)
    n = case.size
    case = case[rng.permutation(n)]
    act = rng.integers(0, 9, n)
    ts = rng.integers(0, ts_range, n) * 1000 - 7
    if extras:   # the ingest-row payload orders an extra column: an event-level range
        # filter on it after the sort must keep exactly the oracle's rows
        from tests.parity import collect
        c, a, t = to_device_cols(case, act, ts, 9)
        x = rng.integers(0, 100, n)
        log = pm4g.pm4g_log_create(c, a, t, 9, n_case_codes=int(case.max()) + 1,
                                   extra=[pm4g.Extra(pm4g.PM4G_KIND_I64, torch.as_tensor(x).cuda())])
        log.sort()
        assert_parity(collect(log), oracle.run(case, act, ts, 9))
        f = log.filter_attr(column=0, lo=20, hi=60)
        keep = oracle.filter_attr(case, x, lo=20, hi=60)
        assert_parity(collect(f), oracle.run(case[keep], act[keep], ts[keep], 9))
    else:
        assert_parity(gpu_run(case, act, ts, 9, n_case_codes=int(case.max()) + 1),
                      oracle.run(case, act, ts, 9))


def test_long_cases_up_to_the_rank_limit():
    """Cases of 300-1024 rows (the in-shared-memory ranking's O(m) per row at its
    largest; 1024 = FMT_WARP_MAX) mixed with short ones and cases just past the
    limit (the exact fallback), shuffled, with timestamp ties: the formatted log
    and every aggregate equal the oracle's."""
    rng = np.random.default_rng(41)
    lens = np.concatenate([rng.integers(300, 1025, 300), rng.integers(1, 40, 20_000), [1025, 1030, 2000]])
    case = np.repeat(rng.permutation(lens.size), lens)
    n = case.size
    case = case[rng.permutation(n)]
    act = rng.integers(0, 30, n)
    ts = rng.integers(0, 5_000, n) * 7
    for sa in (False, True):
        assert_parity(gpu_run(case, act, ts, 30, n_case_codes=int(case.max()) + 1, sort_analyze=sa),
                      oracle.run(case, act, ts, 30))


@pytest.mark.parametrize("name", ["bpic2019", "bpic2018"])
def test_variant_ordering_radix_fallback(monkeypatch, name):
    """A table of 2k-1.2M groups is ordered by one cooperative kernel; when the
    grid cannot be launched (PM4G_DEBUG_NO_COOP forces it) the library radix
    passes order it instead -- same results (R11: count desc, rep asc)."""
    monkeypatch.setenv("PM4G_DEBUG_NO_COOP", "1")
    L = generate(CONFIGS[name])
    c, a, t = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    assert_parity(gpu_run(c, a, t, L.n_activities, n_case_codes=L.n_case_codes, sort_analyze=True),
                  oracle.run(c, a, t, L.n_activities))


def test_variant_table_past_cooperative_capacity():
    """A table with more groups than the cooperative ordering's co-resident
    chunks hold (one CTA per SM x 4096 groups) takes the radix ordering instead
    of failing: 800k cases of 4-6 random activities out of 64, nearly all
    distinct variants (R11 order, every output vs the oracle)."""
    rng = np.random.default_rng(7)
    C = 800_000
    m = rng.integers(4, 7, size=C)
    case = np.repeat(np.arange(C, dtype=np.int64), m)
    n = case.size
    act = rng.integers(0, 64, size=n)
    ts = rng.integers(0, 1 << 40, size=n)
    perm = rng.permutation(n)
    case, act, ts = case[perm], act[perm], ts[perm]
    r = oracle.run(case, act, ts, 64)
    assert len(r.v_count) > 148 * 4096   # past a one-CTA-per-SM cooperative grid
    assert_parity(gpu_run(case, act, ts, 64, n_case_codes=C, sort_analyze=True), r)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_format_mixed_narrow_and_wide_cases(seed):
    """k_format ranks every case narrow first (32-bit key differences) and
    re-ranks a case found wide (a key > 2^30 units from its first) exactly:
    tiles mixing narrow and wide cases, ties inside both, cases crossing tile
    ends -- every output vs the oracle."""
    rng = np.random.default_rng(100 + seed)
    C = 6000
    m = rng.integers(1, 40, size=C)
    case = np.repeat(np.arange(C, dtype=np.int64), m)
    n = case.size
    wide = rng.random(C) < 0.1                        # ~10% of the cases span > 2^30
    span = np.where(wide[case], 1 << 34, 1 << 20)
    ts = (rng.random(n) * span).astype(np.int64)
    tie = rng.random(n) < 0.2                         # equal timestamps inside a case
    ts[tie] = (case[tie] * 7) % 1000
    act = rng.integers(0, 12, size=n)
    p = rng.permutation(n)
    case, act, ts = case[p], act[p], ts[p]
    assert_parity(gpu_run(case, act, ts, 12, n_case_codes=C, sort_analyze=True), oracle.run(case, act, ts, 12))


@pytest.mark.parametrize("dtype", [torch.int16, torch.int32])
@pytest.mark.parametrize("A", [7, 60, 91])
def test_wide_activity_codes_with_dense_table(dtype, A):
    """2- and 4-byte activity codes with a small alphabet (the caller's choice of
    width): the dense shared-memory DFG table next to the wider stages, with and
    without the min / max tables -- every output vs the oracle."""
    from tests.parity import collect
    rng = np.random.default_rng(A)
    n = 60_000
    case = rng.integers(0, 5_000, n)
    act = rng.integers(0, A, n)
    ts = rng.integers(0, 10**9, n)
    c = torch.as_tensor(case).to(torch.uint32).cuda()
    a = torch.as_tensor(act).to(dtype).cuda()
    t = torch.as_tensor(ts).cuda()
    log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=5_000)
    log.sort()
    assert_parity(collect(log), oracle.run(case, act, ts, A))
    o = log.analyze(minmax=True)
    rmn, rmx = oracle.dfg_minmax(case, act, ts, A)
    assert np.array_equal(o["dur_min"].cpu().numpy().view(np.uint64), rmn.reshape(-1).astype(np.uint64))
    assert np.array_equal(o["dur_max"].cpu().numpy().view(np.uint64), rmx.reshape(-1).astype(np.uint64))
    o["variants"].close()
    log.close()


def test_fallback_rows_written_before_the_deferred_fallback():
    """Every formatted row holds a valid activity code before the deferred exact
    fallback runs (the analysis reads the provisional order first): the formatted
    column is poisoned before k_format and checked after it (PM4G_DEBUG_POISON_FORMAT)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "poison_run.py")],
                       capture_output=True, text=True, timeout=900, cwd=root)
    assert "poison_run ok" in r.stdout, (r.stdout + r.stderr)[-4000:]
