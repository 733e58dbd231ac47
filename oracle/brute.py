"""O2 -- per-trace brute force in pure Python (TEST INFRASTRUCTURE ONLY).

Independent of O1 (oracle.cpp): no sort of the whole table, no single loop.
Each case is gathered into its own list of (ts, ingest index, activity) and
sorted on its own (case, then timestamp, then absolute index), then
every output is enumerated per trace ("enumerate consecutive pairs per
case by brute force", S:369 hand enumeration of variants).  For tiny logs only.
"""
from __future__ import annotations

from collections import defaultdict


def traces(case, act, ts):
    """{case code: [(ts, ingest index, act), ...] sorted by (ts, index)}."""
    per = defaultdict(list)
    for i, (c, a, t) in enumerate(zip(case, act, ts)):
        per[int(c)].append((int(t), i, int(a)))
    return {c: sorted(v) for c, v in per.items()}


def analyse(case, act, ts, A: int) -> dict:
    """All hot-path outputs as plain Python dicts/lists."""
    tr = traces(case, act, ts)
    cnt = defaultdict(int)
    dsum = defaultdict(int)
    dmin, dmax = {}, {}
    start = defaultdict(int)
    end = defaultdict(int)
    cases = []
    variants = defaultdict(int)
    rep = {}
    for c in sorted(tr):
        evs = tr[c]
        seq = tuple(a for _, _, a in evs)
        for (t0, _, a0), (t1, _, a1) in zip(evs, evs[1:]):
            cnt[(a0, a1)] += 1
            dsum[(a0, a1)] += t1 - t0
            dmin[(a0, a1)] = min(dmin.get((a0, a1), t1 - t0), t1 - t0)
            dmax[(a0, a1)] = max(dmax.get((a0, a1), t1 - t0), t1 - t0)
        start[seq[0]] += 1
        end[seq[-1]] += 1
        cases.append((c, len(evs), evs[-1][0] - evs[0][0]))
        variants[seq] += 1
        rep.setdefault(seq, c)
    mean = {k: dsum[k] / cnt[k] for k in cnt}
    return {"cnt": dict(cnt), "sum": dict(dsum), "mean": mean, "min": dmin, "max": dmax,
            "start": dict(start),
            "end": dict(end), "cases": cases, "variants": dict(variants), "rep": rep,
            "sorted": [(c, t, i, a) for c in sorted(tr) for (t, i, a) in tr[c]]}


def filter_time(case, ts, t1, t2, mode):
    """S:413 by enumeration; returns kept row indices in input order."""
    if t1 > t2:
        raise ValueError("t1 > t2")
    if mode == 0:
        return [i for i, t in enumerate(ts) if t1 <= t <= t2]
    span = {}
    for c, t in zip(case, ts):
        lo, hi = span.get(int(c), (t, t))
        span[int(c)] = (min(lo, t), max(hi, t))
    ok = {c: (lo >= t1 and hi <= t2) if mode == 1 else (lo <= t2 and hi >= t1)
          for c, (lo, hi) in span.items()}
    return [i for i, c in enumerate(case) if ok[int(c)]]


def filter_codes(case, col, codes, level, keep=True):
    """S:448 by enumeration (u32 in-set predicate); kept row indices."""
    codes = set(int(x) for x in codes)
    m = [int(v) in codes for v in col]
    if level == 0:
        return [i for i in range(len(m)) if m[i] == keep]
    anym = defaultdict(bool)
    for c, x in zip(case, m):
        anym[int(c)] |= x
    return [i for i, c in enumerate(case) if anym[int(c)] == keep]


def filter_cases(case, act, ts, kind, codes=(), lo=0, hi=0, keep=True):
    """S:428-435, S:454-471 by enumeration over traces; kept row indices.
    kind 0 start in codes, 1 end in codes, 2 size in [lo, hi], 3 throughput in
    [lo, hi], 4 some directly-follows pair in the pairs (codes[0::2], codes[1::2])."""
    tr = traces(case, act, ts)
    codes = [int(x) for x in codes]
    pairs = set(zip(codes[0::2], codes[1::2]))
    ok = {}
    for c, evs in tr.items():
        seq = [a for _, _, a in evs]
        if kind == 0:
            m = seq[0] in codes
        elif kind == 1:
            m = seq[-1] in codes
        elif kind == 2:
            m = lo <= len(seq) <= hi
        elif kind == 3:
            m = lo <= evs[-1][0] - evs[0][0] <= hi
        else:
            m = any((x, y) in pairs for x, y in zip(seq, seq[1:]))
        ok[c] = m == keep
    return [i for i, c in enumerate(case) if ok[int(c)]]


def filter_variants(case, act, ts, seqs, keep=True):
    """S:372-380 by enumeration: cases whose exact sequence is in seqs."""
    tr = traces(case, act, ts)
    want = set(tuple(int(x) for x in q) for q in seqs)
    ok = {c: (tuple(a for _, _, a in evs) in want) == keep for c, evs in tr.items()}
    return [i for i, c in enumerate(case) if ok[int(c)]]


def efg(case, act, ts):
    """S:318-329 by enumeration: {(a, b): [durations of every in-case pair i < j]}."""
    out = defaultdict(list)
    for c, evs in traces(case, act, ts).items():
        for x in range(len(evs)):
            for y in range(x + 1, len(evs)):
                out[(evs[x][2], evs[y][2])].append(evs[y][0] - evs[x][0])
    return dict(out)


def variant_order(case, act, ts):
    """Variants in the ABI order by enumeration (reading R11: count descending,
    then the smallest case code holding the variant ascending), and each case's
    index into that list (S:358 case_to_variant, cases in ascending code).
    Returns (ordered [(seq, count, rep)], [variant index per case])."""
    tr = traces(case, act, ts)
    groups = {}
    for c in tr:
        seq = tuple(a for _, _, a in tr[c])
        g = groups.setdefault(seq, [0, c])
        g[0] += 1
        g[1] = min(g[1], c)
    ordered = sorted(((s, k, r) for s, (k, r) in groups.items()), key=lambda x: (-x[1], x[2]))
    pos = {s: i for i, (s, _, _) in enumerate(ordered)}
    return ordered, [pos[tuple(a for _, _, a in tr[c])] for c in sorted(tr)]


def filter_range(case, col, lo, hi, valid=None, level=0, keep=True):
    """S:447-448 numeric-in-[lo, hi] by enumeration (i64 or f64 values; nulls,
    valid[i] == 0, never match); kept row indices in input order."""
    m = [(valid is None or bool(valid[i])) and (lo <= col[i] <= hi) for i in range(len(col))]
    if level == 0:
        return [i for i in range(len(m)) if m[i] == keep]
    anym = defaultdict(bool)
    for c, x in zip(case, m):
        anym[int(c)] |= x
    return [i for i, c in enumerate(case) if anym[int(c)] == keep]
