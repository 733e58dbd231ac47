"""Pins for the CPU oracle (O1 = oracle.cpp, O2 = oracle/brute.py).

No GPU.  Each test ties the oracle to something other than itself: the paper's
/ SPEC's worked example L1 (tests/golden/l1.json), brute force on tiny random
logs, closed forms from planted generator structure, invariants
 and the replication law.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import brute
from gen.synth import CONFIGS, generate, replicate
from gen.tinylogs import random_log


def _l1_cols(l1):
    r = l1["rows_ingest_order"]
    return r["case"], r["act"], r["ts"], l1["n_activities"]


# ------------------------------------------------------------------ L1 worked example
def test_l1_o1_matches_spec(l1):
    case, act, ts, A = _l1_cols(l1)
    ex = l1["expected"]
    r = oracle.run(case, act, ts, A)
    assert r.n_events.tolist() == ex["n_events_per_case"]["value"]
    assert r.dur.tolist() == ex["throughput_ms"]["value"]
    exp_cnt = np.zeros((A, A), np.uint64)
    for a, b, k in ex["dfg_count"]["value"]:
        exp_cnt[a, b] = k
    assert (r.cnt == exp_cnt).all()                      # also catches a transposed (a, b)
    for a, b, m in ex["dfg_mean"]["value"]:
        assert r.mean[a, b] == m
    exp_sum = np.zeros((A, A), np.int64)
    for a, b, s in ex["dfg_sum_hand"]["value"]:
        exp_sum[a, b] = s
    assert (r.sum == exp_sum).all()
    assert {i: int(v) for i, v in enumerate(r.start) if v} == {a: k for a, k in ex["start"]["value"]}
    assert {i: int(v) for i, v in enumerate(r.end) if v} == {a: k for a, k in ex["end"]["value"]}
    assert r.variants() == {tuple(s): k for s, k in ex["variants"]["value"]}
    # prev_activity of c1: formatted rows of case 0 are A, B, C
    c1 = r.sorted_act[r.sorted_case == 0].tolist()
    assert [None] + c1[:-1] == ex["prev_activity_c1"]["value"]
    rep = ex["report"]["value"]
    assert (r.n_cases, len(case), len(r.variants())) == (rep["cases"], rep["events"], rep["variants"])


def test_l1_variant_order_and_case_index():
    """S:369 L1 -> {<A,B,C>: 2, <A,C>: 1}; reading R11 orders them count descending,
    so <A,B,C> (count 2) is variant 0 and <A,C> variant 1; "c1 and c3 share
    variant_id, c2 differs" -> case_variant = [0, 1, 0] (cases in code order)."""
    case, act, ts = [0, 1, 2, 0, 1, 2, 0, 2], [0, 0, 0, 1, 2, 1, 2, 2], [0, 5, 0, 10, 15, 50, 20, 100]
    r = oracle.run(case, act, ts, 3)
    seqs = [r.v_act[r.v_off[i]:r.v_off[i + 1]].tolist() for i in range(r.v_count.size)]
    assert seqs == [[0, 1, 2], [0, 2]]
    assert r.v_count.tolist() == [2, 1] and r.v_len.tolist() == [3, 2]
    assert r.v_rep.tolist() == [0, 1]                 # smallest case holding each variant
    assert r.case_variant.tolist() == [0, 1, 0]


def test_variant_order_ties_by_smallest_case():
    """R11 tie-break: equal counts ordered by the smallest case code ascending (not by
    sequence, not by first appearance in ingest order).  Case 5 holds <1> and is
    ingested first; case 2 holds <0, 0>, case 3 holds <2>, case 9 holds <1>, case 7
    holds <0, 0>: counts {<1>: 2, <0,0>: 2, <2>: 1}, reps {<1>: 5, <0,0>: 2, <2>: 3}."""
    case = [5, 9, 7, 2, 3, 7, 2]
    act = [1, 1, 0, 0, 2, 0, 0]
    ts = [0, 0, 0, 0, 0, 1, 1]
    r = oracle.run(case, act, ts, 3)
    seqs = [tuple(r.v_act[r.v_off[i]:r.v_off[i + 1]].tolist()) for i in range(r.v_count.size)]
    assert seqs == [(0, 0), (1,), (2,)]
    assert r.v_rep.tolist() == [2, 5, 3]
    # cases in code order 2, 3, 5, 7, 9
    assert r.case_variant.tolist() == [0, 2, 1, 0, 1]


def test_l1_o2_matches_spec(l1):
    case, act, ts, A = _l1_cols(l1)
    ex = l1["expected"]
    b = brute.analyse(case, act, ts, A)
    assert b["cnt"] == {(a, bb): k for a, bb, k in ex["dfg_count"]["value"]}
    assert b["sum"] == {(a, bb): s for a, bb, s in ex["dfg_sum_hand"]["value"]}
    assert [c[1] for c in b["cases"]] == ex["n_events_per_case"]["value"]
    assert [c[2] for c in b["cases"]] == ex["throughput_ms"]["value"]
    assert b["variants"] == {tuple(s): k for s, k in ex["variants"]["value"]}


def test_l1_filters(l1):
    case, act, ts, A = _l1_cols(l1)
    ex = l1["expected"]
    keep = oracle.filter_time(case, ts, 0, 15, oracle.EVENTS)
    sub = [(c, a, t) for c, a, t, k in zip(case, act, ts, keep) if k]
    r = oracle.run(*zip(*sub), A)
    got = list(zip(r.sorted_case.tolist(), r.sorted_act.tolist(), r.sorted_ts.tolist()))
    assert [list(x) for x in got] == ex["filter_events_0_15"]["value"]
    for (t1, t2, mode, key) in [(0, 20, 1, "filter_contained_0_20"),
                                (90, 200, 2, "filter_intersecting_90_200")]:
        keep = oracle.filter_time(case, ts, t1, t2, mode)
        assert sorted({c for c, k in zip(case, keep) if k}) == ex[key]["value"]
        assert [i for i, k in enumerate(keep) if k] == brute.filter_time(case, ts, t1, t2, mode)
    keep = oracle.filter_attr(case, act, codes=[1], level=1)
    assert sorted({c for c, k in zip(case, keep) if k}) == ex["filter_attr_act_B_cases"]["value"]
    with pytest.raises(ValueError):
        oracle.filter_time(case, ts, 20, 0, oracle.EVENTS)


def test_l1_after_time_filter_dfg():
    """SURVEY Appendix A / S:499: adjacency re-derived after an events-mode filter."""
    case, act, ts = [0, 1, 2, 0, 1, 2, 0, 2], [0, 0, 0, 1, 2, 1, 2, 2], [0, 5, 0, 10, 15, 50, 20, 100]
    keep = oracle.filter_time(case, ts, 0, 15, oracle.EVENTS)
    sub = [(c, a, t) for c, a, t, k in zip(case, act, ts, keep) if k]
    r = oracle.run(*zip(*sub), 3)
    assert r.cnt[0, 1] == 1 and r.sum[0, 1] == 10     # c1: A@0 -> B@10
    assert r.cnt[0, 2] == 1 and r.sum[0, 2] == 10     # c2: A@5 -> C@15
    assert int(r.cnt.sum()) == 2


def test_tie_broken_by_ingest_index():
    """equal timestamps, ingest order X then Y -> X precedes Y."""
    r = oracle.run([7, 7, 7], [1, 0, 2], [5, 5, 5], 3)
    assert r.sorted_act.tolist() == [1, 0, 2]
    assert r.cnt[1, 0] == 1 and r.cnt[0, 2] == 1 and int(r.cnt.sum()) == 2
    r2 = oracle.run([7, 7, 7], [0, 1, 2], [5, 5, 5], 3)
    assert r2.sorted_act.tolist() == [0, 1, 2]


# ------------------------------------------------------------------ O1 == O2
def _o1_vs_o2(case, act, ts, A):
    r = oracle.run(case, act, ts, A)
    b = brute.analyse(case, act, ts, A)
    cnt = {(a, bb): int(r.cnt[a, bb]) for a in range(A) for bb in range(A) if r.cnt[a, bb]}
    assert cnt == b["cnt"]
    sm = {k: int(r.sum[k]) for k in b["cnt"]}
    assert sm == b["sum"]
    for k, m in b["mean"].items():
        assert r.mean[k] == pytest.approx(m, rel=1e-15, abs=0)
    assert {i: int(v) for i, v in enumerate(r.start) if v} == b["start"]
    assert {i: int(v) for i, v in enumerate(r.end) if v} == b["end"]
    assert list(zip(r.case_code.tolist(), r.n_events.tolist(), r.dur.tolist())) == b["cases"]
    assert r.variants() == b["variants"]
    for i in range(r.v_count.size):
        seq = tuple(r.v_act[r.v_off[i]:r.v_off[i + 1]].tolist())
        assert r.v_rep[i] == b["rep"][seq]
    # R11 output order and the per-case variant index, by enumeration
    ordered, cv = brute.variant_order(case, act, ts)
    got = [(tuple(r.v_act[r.v_off[i]:r.v_off[i + 1]].tolist()), int(r.v_count[i]), int(r.v_rep[i]))
           for i in range(r.v_count.size)]
    assert got == ordered
    assert r.v_len.tolist() == [len(s) for s, _, _ in ordered]
    assert r.case_variant.tolist() == cv
    assert [(c, t, i, a) for c, t, i, a in zip(r.sorted_case.tolist(), r.sorted_ts.tolist(),
                                               r.perm.tolist(), r.sorted_act.tolist())] == b["sorted"]
    return r


@pytest.mark.parametrize("seed", range(200))
def test_o1_equals_o2_random(seed):
    case, act, ts, A, _ = random_log(seed)
    r = _o1_vs_o2(case, act, ts, A)
    # filters: O1 vs O2 on the same log
    if case:
        lo, hi = min(ts), max(ts)
        t1 = lo + (hi - lo) // 4
        t2 = lo + 3 * (hi - lo) // 4
        for mode in (0, 1, 2):
            keep = oracle.filter_time(case, ts, t1, t2, mode)
            assert [i for i, k in enumerate(keep) if k] == brute.filter_time(case, ts, t1, t2, mode)
        for level in (0, 1):
            for kp in (True, False):
                keep = oracle.filter_attr(case, act, codes=[0], level=level, keep=kp)
                assert [i for i, k in enumerate(keep) if k] == brute.filter_codes(case, act, [0], level, kp)


# ------------------------------------------------------------------ invariants
def _invariants(r, n):
    C = r.n_cases
    assert int(r.cnt.sum()) == n - C
    assert int(r.start.sum()) == C and int(r.end.sum()) == C
    assert int(r.v_count.sum()) == C
    assert int(r.n_events.astype(np.int64).sum()) == n
    # telescoping: sum over edges of the duration sums == sum of case durations
    assert int(r.sum.astype(np.int64).sum()) == int(r.dur.sum())
    assert (r.dur >= 0).all()
    # formatted log: grouped by case ascending, ts ascending within a case
    sc, st = r.sorted_case.astype(np.int64), r.sorted_ts
    assert (np.diff(sc) >= 0).all()
    same = np.diff(sc) == 0
    assert (np.diff(st)[same] >= 0).all()
    assert sorted(r.perm.tolist()) == list(range(n))        # S:204 permutation
    assert (r.case_code == np.unique(sc)).all()
    assert (np.diff(r.first_row) > 0).all() if C > 1 else True


@pytest.mark.parametrize("seed", range(0, 200, 7))
def test_invariants_random(seed):
    case, act, ts, A, _ = random_log(seed)
    _invariants(oracle.run(case, act, ts, A), len(case))


@pytest.mark.parametrize("name", ["tiny", "roadtraffic"])
def test_invariants_generator(name):
    L = generate(CONFIGS[name])
    r = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities)
    _invariants(r, L.n)
    assert r.n_cases == CONFIGS[name].n_cases
    if name == "roadtraffic":   # PAPER.md Table 1 shape (x1 base of roadtraffic_2)
        assert L.n == 561_470 and len(r.variants()) == 231 and L.n_activities == 11


# ------------------------------------------------------------------ closed forms
def test_closed_form_planted_pool():
    """No-tie twin of roadtraffic: DFG counts = sum_v m_v * pairs(v), start/end and
    the variant multiset follow from the planted pool assignment alone."""
    spec = CONFIGS["roadtraffic"]
    L = generate(spec, no_ties=True)
    r = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities)
    m = np.bincount(L.case_variant.numpy(), minlength=len(L.pool_seqs))
    A = L.n_activities
    cnt = np.zeros((A, A), np.int64)
    start = np.zeros(A, np.int64)
    end = np.zeros(A, np.int64)
    want = {}
    for v, seq in enumerate(L.pool_seqs):
        if m[v] == 0:
            continue
        for a, b in zip(seq, seq[1:]):
            cnt[a, b] += m[v]
        start[seq[0]] += m[v]
        end[seq[-1]] += m[v]
        want[tuple(seq)] = int(m[v])
    assert (r.cnt.astype(np.int64) == cnt).all()
    assert (r.start.astype(np.int64) == start).all() and (r.end.astype(np.int64) == end).all()
    assert r.variants() == want
    assert (r.n_events.astype(np.int64) == L.case_len.numpy()).all()


def test_closed_form_planted_order_tiny():
    """Tiny config, no ties: the formatted sequences equal the generator's unshuffled
    (case, position) rows, so every aggregate is an enumeration over those rows."""
    spec = CONFIGS["tiny"]
    L = generate(spec, no_ties=True)
    P = generate(spec, no_ties=True, shuffle=False)
    r = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities)
    assert (r.sorted_act == P.act.numpy()).all()
    assert (r.sorted_ts == P.ts.numpy()).all()
    b = brute.analyse(P.case.tolist(), P.act.tolist(), P.ts.tolist(), L.n_activities)
    assert {k: int(r.cnt[k]) for k in b["cnt"]} == b["cnt"] and int(r.cnt.sum()) == sum(b["cnt"].values())


# ------------------------------------------------------------------ replication law
@pytest.mark.parametrize("k", [2, 5, 10, 20])
def test_replication_law(k):
    """P:176 ("variants and activities are unchanged"): x k cases under fresh
    ids multiply counts and sums by k, leave means and the variant set unchanged."""
    L = generate(CONFIGS["tiny"])
    r1 = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities)
    R = replicate(L, k)
    rk = oracle.run(R.case.numpy(), R.act.numpy(), R.ts.numpy(), R.n_activities)
    assert (rk.cnt == r1.cnt * k).all()
    assert (rk.sum == r1.sum * k).all()
    assert (rk.mean == r1.mean).all()
    assert (rk.start == r1.start * k).all() and (rk.end == r1.end * k).all()
    v1, vk = r1.variants(), rk.variants()
    assert set(v1) == set(vk) and all(vk[s] == k * c for s, c in v1.items())
    assert rk.n_cases == k * r1.n_cases


# ------------------------------------------------------------------ special cases
def test_empty_log():
    r = oracle.run([], [], [], 4)
    assert r.n_cases == 0 and int(r.cnt.sum()) == 0 and r.v_count.size == 0 and (r.start == 0).all()


def test_single_event_cases():
    """k single-event cases of activity X -> one variant <X> with count k."""
    r = oracle.run(list(range(6)), [2] * 6, [10, 9, 8, 7, 6, 5], 3)
    assert r.variants() == {(2,): 6}
    assert (r.dur == 0).all() and int(r.cnt.sum()) == 0
    assert r.start[2] == 6 and r.end[2] == 6


def test_self_loops_and_equal_timestamps():
    """R5: self-loops count; equal consecutive timestamps give a 0 ms edge."""
    r = oracle.run([0, 0, 0, 0], [1, 1, 1, 1], [3, 3, 3, 3], 2)
    assert r.cnt[1, 1] == 3 and r.sum[1, 1] == 0 and r.mean[1, 1] == 0.0


def test_negative_timestamps():
    r = oracle.run([0, 0], [0, 1], [-5, -2], 2)
    assert r.sum[0, 1] == 3 and r.dur.tolist() == [3]


def test_validate():
    """code out of range is reported with the first bad row."""
    assert oracle.validate([0, 1], [0, 1], 2, 2) == (0, -1)
    assert oracle.validate([0, 2], [0, 1], 2, 2) == (2, 1)
    assert oracle.validate([0, 1], [0, 3], 2, 3) == (2, 1)


def test_wraparound_is_modulo_2_64_and_flagged():
    """R8: duration sums are int64 modulo 2^64; O1 flags a wrap."""
    big = (1 << 62)
    case = [0, 0, 1, 1, 2, 2]
    ts = [0, big, 0, big, 0, big]
    r = oracle.run(case, [0, 1] * 3, ts, 2)
    want = (3 * big) & ((1 << 64) - 1)
    want = want - (1 << 64) if want >> 63 else want
    assert int(r.sum[0, 1]) == want and r.overflow
    assert not oracle.run([0, 0], [0, 1], [0, 5], 2).overflow


def test_time_filter_laws():
    """contained subset of intersecting; events-mode rows in range."""
    L = generate(CONFIGS["tiny"])
    case, ts = L.case.numpy(), L.ts.numpy()
    lo, hi = int(ts.min()), int(ts.max())
    for j in range(10):
        t1 = lo + (hi - lo) * j // 20
        t2 = t1 + (hi - lo) // 3
        con = oracle.filter_time(case, ts, t1, t2, 1)
        inter = oracle.filter_time(case, ts, t1, t2, 2)
        assert not (con & ~inter).any()
        ev = oracle.filter_time(case, ts, t1, t2, 0)
        assert ((ts[ev] >= t1) & (ts[ev] <= t2)).all() and not ((ts[~ev] >= t1) & (ts[~ev] <= t2)).any()


def test_attr_filter_keep_remove_partition():
    """S:383 analogue: keep(S) and remove(S) partition the rows/cases."""
    L = generate(CONFIGS["tiny"])
    case, act = L.case.numpy(), L.act.numpy()
    for level in (0, 1):
        k = oracle.filter_attr(case, act, codes=[1, 3], level=level, keep=True)
        rm = oracle.filter_attr(case, act, codes=[1, 3], level=level, keep=False)
        assert (k ^ rm).all()
    # numeric range predicate with nulls: nulls never match
    val = np.arange(case.size, dtype=np.int64)
    valid = (val % 3 != 0)
    k = oracle.filter_attr(case, val, lo=10, hi=50, valid=valid, level=0)
    assert k.tolist() == [(10 <= v <= 50) and (v % 3 != 0) for v in val.tolist()]


@pytest.mark.parametrize("seed", range(40))
def test_attr_range_f64_and_i64_vs_brute(seed):
    """S:447-448 numeric-in-[lo, hi] (inclusive) with nulls, both levels, keep and
    remove: O1's f64 and i64 range kinds against enumeration (O2)."""
    case, act, ts, A, _ = random_log(seed)
    if not case:
        return
    rng = np.random.default_rng(1000 + seed)
    n = len(case)
    f = rng.normal(0.0, 10.0, n)
    f[rng.random(n) < 0.1] = 2.5          # exact hits on the bounds
    f[rng.random(n) < 0.05] = -2.5
    valid = rng.random(n) >= 0.15
    iv = rng.integers(-20, 20, n)
    for level in (0, 1):
        for kp in (True, False):
            k = oracle.filter_attr(case, f, lo=-2.5, hi=2.5, valid=valid, level=level, keep=kp)
            assert [i for i, x in enumerate(k) if x] == brute.filter_range(
                case, f.tolist(), -2.5, 2.5, valid.tolist(), level, kp)
            k = oracle.filter_attr(case, iv, lo=-3, hi=4, valid=valid, level=level, keep=kp)
            assert [i for i, x in enumerate(k) if x] == brute.filter_range(
                case, iv.tolist(), -3, 4, valid.tolist(), level, kp)
    with pytest.raises(ValueError):
        oracle.filter_attr(case, f, lo=1.0, hi=0.0)   # S:458 min > max
