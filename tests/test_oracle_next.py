"""Pins for the oracle's NEXT rows: NEXT-1 whole-case filters
(start / end activity, case size, throughput, paths, variants) and NEXT-2
per-edge min / max durations.  No GPU.

Each is tied to something other than O1 itself: SPEC's L1 examples
(tests/golden/l1.json: S:374, hand-derived
min / max), O2 brute force (per-trace enumeration) on random logs, and the
keep / remove partition law.
"""
import numpy as np
import pytest

import oracle
from oracle import brute
from gen.synth import CONFIGS, generate
from gen.tinylogs import random_log


def _l1(l1):
    r = l1["rows_ingest_order"]
    return r["case"], r["act"], r["ts"], l1["n_activities"]


def _cases(case, keep):
    return sorted({int(c) for c, k in zip(case, keep) if k})


def test_l1_case_filters(l1):
    case, act, ts, A = _l1(l1)
    ex = l1["expected"]
    assert _cases(case, oracle.filter_cases(case, act, ts, oracle.CASE_SIZE, lo=3, hi=3)) == \
        ex["filter_case_size_3_3"]["value"]
    assert _cases(case, oracle.filter_cases(case, act, ts, oracle.CASE_THROUGHPUT, lo=0, hi=10)) == \
        ex["filter_throughput_0_10"]["value"]
    assert _cases(case, oracle.filter_cases(case, act, ts, oracle.CASE_PATHS, codes=[0, 2])) == \
        ex["filter_paths_keep_AC"]["value"]
    assert _cases(case, oracle.filter_cases(case, act, ts, oracle.CASE_START_IN, codes=[0])) == \
        ex["filter_start_in_A"]["value"]
    assert _cases(case, oracle.filter_cases(case, act, ts, oracle.CASE_END_IN, codes=[1])) == \
        ex["filter_end_in_B"]["value"]
    assert _cases(case, oracle.filter_variants(case, act, ts, [[0, 2]])) == \
        ex["filter_variants_keep_AC"]["value"]
    # keep {} -> empty, remove {} -> identity
    assert not oracle.filter_cases(case, act, ts, oracle.CASE_PATHS, codes=[]).any()
    assert oracle.filter_cases(case, act, ts, oracle.CASE_PATHS, codes=[], keep=False).all()
    assert oracle.filter_variants(case, act, ts, [], keep=False).all()
    with pytest.raises(ValueError):
        oracle.filter_cases(case, act, ts, oracle.CASE_SIZE, lo=4, hi=3)
    with pytest.raises(ValueError):
        oracle.filter_cases(case, act, ts, oracle.CASE_PATHS, codes=[0, 1, 2])


def test_l1_dfg_min_max(l1):
    case, act, ts, A = _l1(l1)
    mn, mx = oracle.dfg_minmax(case, act, ts, A)
    want_mn = np.zeros((A, A), np.uint64)
    want_mx = np.zeros((A, A), np.uint64)
    for a, b, lo, hi in l1["expected"]["dfg_min_max_hand"]["value"]:
        want_mn[a, b], want_mx[a, b] = lo, hi
    assert (mn == want_mn).all() and (mx == want_mx).all()
    b = brute.analyse(case, act, ts, A)
    assert b["min"] == {(x, y): lo for x, y, lo, _ in l1["expected"]["dfg_min_max_hand"]["value"]}


@pytest.mark.parametrize("seed", range(40))
def test_o1_equals_o2_random(seed):
    case, act, ts, A, _ = random_log(1000 + seed)
    rng = np.random.default_rng(seed)
    mn, mx = oracle.dfg_minmax(case, act, ts, A)
    b = brute.analyse(case, act, ts, A)
    for (x, y), v in b["min"].items():
        assert mn[x, y] == v and mx[x, y] == b["max"][(x, y)]
    assert int((mn > 0).sum() + (mx > 0).sum()) <= 2 * len(b["min"])
    codes = rng.integers(0, A, rng.integers(0, 3)).tolist()
    pairs = rng.integers(0, A, 2 * int(rng.integers(0, 3))).tolist()
    lo = int(rng.integers(0, 5))
    hi = lo + int(rng.integers(0, 5))
    tl = int(rng.integers(0, 10**6))
    for kind, kw in [(0, dict(codes=codes)), (1, dict(codes=codes)), (2, dict(lo=lo, hi=hi)),
                     (3, dict(lo=tl, hi=tl + 10**6)), (4, dict(codes=pairs))]:
        for keep in (True, False):
            got = oracle.filter_cases(case, act, ts, kind, keep=keep, **kw)
            want = brute.filter_cases(case, act, ts, kind, keep=keep, **kw)
            assert [i for i, k in enumerate(got) if k] == want
    seqs = list(brute.analyse(case, act, ts, A)["variants"])[: int(rng.integers(0, 3))]
    seqs.append([A - 1] * 3)                     # possibly unobserved: ignored
    for keep in (True, False):
        got = oracle.filter_variants(case, act, ts, seqs, keep=keep)
        assert [i for i, k in enumerate(got) if k] == brute.filter_variants(case, act, ts, seqs, keep=keep)


def test_case_filter_partition_and_variant_subset():
    """keep(S) and remove(S) partition the cases; variants after keep(S) are in S."""
    L = generate(CONFIGS["tiny"])
    case, act, ts = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    r = oracle.run(case, act, ts, L.n_activities)
    seqs = list(r.variants())[:5]
    k = oracle.filter_variants(case, act, ts, seqs)
    assert (k ^ oracle.filter_variants(case, act, ts, seqs, keep=False)).all()
    sub = oracle.run(case[k], act[k], ts[k], L.n_activities)
    assert set(sub.variants()) <= set(seqs) and sum(sub.variants().values()) == sum(r.variants()[s] for s in seqs)
    for kind, kw in [(0, dict(codes=[0, 1])), (2, dict(lo=3, hi=9)), (4, dict(codes=[0, 1, 2, 3]))]:
        a = oracle.filter_cases(case, act, ts, kind, keep=True, **kw)
        b = oracle.filter_cases(case, act, ts, kind, keep=False, **kw)
        assert (a ^ b).all()


# ------------------------------------------------------------------ NEXT-3: EFG + temporal profile
def test_l1_efg(l1):
    case, act, ts, A = _l1(l1)
    ex = l1["expected"]
    e = oracle.efg(case, act, ts, A)
    want = np.zeros((A, A), np.uint64)
    for a, b, k in ex["efg_count"]["value"]:
        want[a, b] = k
    assert (e["cnt"] == want).all()
    assert int(e["sum"][0, 2]) == ex["efg_sum_AC"]["value"]
    mu, sd = ex["temporal_profile_AC"]["value"]
    assert round(float(e["mean"][0, 2]), 2) == mu and round(float(e["stdev"][0, 2]), 2) == sd
    assert int(e["sq_lo"][0, 2]) == 20**2 + 10**2 + 100**2 and int(e["sq_hi"][0, 2]) == 0


@pytest.mark.parametrize("seed", range(30))
def test_efg_o1_equals_o2_random(seed):
    """Exact count / sum / sumsq against per-trace enumeration; the R22 stdev
    against statistics.pstdev of the enumerated durations; S:328 invariant."""
    import statistics
    case, act, ts, A, _ = random_log(2000 + seed)
    e = oracle.efg(case, act, ts, A)
    b = brute.efg(case, act, ts)
    for (x, y), ds in b.items():
        assert int(e["cnt"][x, y]) == len(ds)
        assert int(e["sum"][x, y]) == sum(ds) % (1 << 64)
        assert int(e["sq_lo"][x, y]) + (int(e["sq_hi"][x, y]) << 64) == sum(d * d for d in ds) % (1 << 128)
        sd = statistics.pstdev(ds)
        mu = statistics.fmean(ds)
        assert e["mean"][x, y] == pytest.approx(mu, rel=1e-12)
        if sd > 1e-6 * max(mu, 1.0):            # well-conditioned: the formula is accurate
            assert e["stdev"][x, y] == pytest.approx(sd, rel=1e-6)
    assert int(e["cnt"].sum()) == sum(len(ds) for ds in b.values())
    per = {}
    for c in case:
        per[c] = per.get(c, 0) + 1
    assert int(e["cnt"].sum()) == sum(m * (m - 1) // 2 for m in per.values())


def test_efg_huge_durations_exact_128():
    """d up to ~2^62: d^2 needs the high word; sums wrap modulo 2^64 (R8)."""
    case = [0, 0, 0, 1, 1]
    act = [0, 1, 1, 0, 1]
    ts = [-(2**61), 0, 2**61, 5, 7]
    e = oracle.efg(case, act, ts, 2)
    ds = [2**61, 2**62, 2**61, 2]                    # (0,1) pairs: 0->1 (x2 in case 0) and case 1
    q = sum(d * d for d in ds[:2] + [2])
    assert int(e["cnt"][0, 1]) == 3
    assert int(e["sq_lo"][0, 1]) + (int(e["sq_hi"][0, 1]) << 64) == q
    assert int(e["sum"][0, 1]) == (2**61 + 2**62 + 2) % (1 << 64)
    assert int(e["cnt"][1, 1]) == 1 and int(e["sq_hi"][1, 1]) == (2**61) ** 2 >> 64
