"""CPU oracle for the PM4Py-GPU hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_2204_04898_b200``) never imports it.

* O1 (``oracle.cpp`` -> ``liboracle.so``): single-threaded C++17, the plain
  definition of every output (stable sort, then one loop), see its header.
* O2 (``brute.py``): per-trace brute force in pure Python for tiny logs.

Every function cites the passage it follows; readings R1..R19 are listed in
DESIGN.md.  Pins (tests/test_oracle_*.py) tie O1/O2 to the paper's worked
example, closed forms, invariants and brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")
_lib = None

EVENTS, CASES_CONTAINED, CASES_INTERSECTING = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile O1 with g++ (-O2, no threads, no SIMD intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _SO, _SRC])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P, I64, U64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.orc_validate.argtypes = [I64, P, P, U64, ctypes.c_uint32, P]
        L.orc_validate.restype = I32
        L.orc_run.argtypes = [I64, P, P, P, ctypes.c_uint32]
        L.orc_run.restype = P
        L.orc_free.argtypes = [P]
        for f in ("orc_n_cases", "orc_n_variants", "orc_variants_total_len"):
            getattr(L, f).argtypes = [P]
            getattr(L, f).restype = I64
        L.orc_overflow.argtypes = [P]
        L.orc_overflow.restype = I32
        L.orc_timing.argtypes = [P, P, P]
        L.orc_get_sorted.argtypes = [P, P, P, P, P]
        L.orc_get_dfg.argtypes = [P, P, P, P]
        L.orc_get_start_end.argtypes = [P, P, P]
        L.orc_get_cases.argtypes = [P, P, P, P, P, P]
        L.orc_get_variants.argtypes = [P, P, P, P, P, P]
        L.orc_filter_time.argtypes = [I64, P, P, I64, I64, I32, P]
        L.orc_filter_time.restype = I32
        L.orc_filter_attr.argtypes = [I64, P, I32, P, P, P, I64, I64, I64,
                                      ctypes.c_double, ctypes.c_double, I32, I32, P]
        L.orc_filter_attr.restype = I32
        L.orc_get_dfg_minmax.argtypes = [P, P, P]
        L.orc_filter_cases.argtypes = [I64, P, P, P, I32, P, I64, I64, I64, I32, P]
        L.orc_filter_cases.restype = I32
        L.orc_filter_variants.argtypes = [I64, P, P, P, P, P, I64, I32, P]
        L.orc_filter_variants.restype = I32
        L.orc_efg.argtypes = [I64, P, P, P, ctypes.c_uint32, P, P, P, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x).astype(np.int64).astype(np.uint32))


def _i64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x).astype(np.int64))


@dataclass
class OracleResult:
    """Everything O1 computes for one log (numpy arrays)."""
    n_activities: int
    sorted_case: np.ndarray
    sorted_act: np.ndarray
    sorted_ts: np.ndarray
    perm: np.ndarray
    cnt: np.ndarray          # u64[A, A]   (a -> b)
    sum: np.ndarray          # i64[A, A]   modulo 2^64
    mean: np.ndarray         # f64[A, A]   sum / cnt where cnt > 0, else 0
    start: np.ndarray        # u64[A]
    end: np.ndarray          # u64[A]
    case_code: np.ndarray    # u32[C]  ascending
    n_events: np.ndarray     # u32[C]
    dur: np.ndarray          # i64[C]
    first_row: np.ndarray    # i64[C]  (CSR offsets without the final n)
    case_variant: np.ndarray # u32[C]  index into the variant list
    v_count: np.ndarray      # u64[V]  count desc, rep asc
    v_len: np.ndarray        # u32[V]
    v_rep: np.ndarray        # u32[V]
    v_off: np.ndarray        # u64[V+1]
    v_act: np.ndarray        # u32[sum len]
    overflow: bool
    t_sort: float = 0.0      # wall seconds of step 1 (stable sort) in O1
    t_loop: float = 0.0      # wall seconds of steps 2 + 3 (the loop) in O1

    @property
    def n_cases(self) -> int:
        return int(self.case_code.size)

    def variants(self) -> dict:
        """{activity-sequence tuple: count}."""
        return {tuple(self.v_act[self.v_off[i]:self.v_off[i + 1]].tolist()): int(self.v_count[i])
                for i in range(self.v_count.size)}


def validate(case, act, n_case_codes: int, n_activities: int):
    """(status, first bad row)."""
    L = _load()
    c, a = _u32(case), _u32(act)
    bad = ctypes.c_int64(-1)
    st = L.orc_validate(c.size, _ptr(c), _ptr(a), n_case_codes, n_activities, ctypes.byref(bad))
    return st, bad.value


def run(case, act, ts, n_activities: int) -> OracleResult:
    """O1 on one log given in ingest order."""
    L = _load()
    c, a, t = _u32(case), _u32(act), _i64(ts)
    n, A = c.size, int(n_activities)
    h = L.orc_run(n, _ptr(c), _ptr(a), _ptr(t), A)
    try:
        C = L.orc_n_cases(h)
        V = L.orc_n_variants(h)
        T = L.orc_variants_total_len(h)
        sc, sa, st, pm = (np.empty(n, np.uint32), np.empty(n, np.uint32),
                          np.empty(n, np.int64), np.empty(n, np.int64))
        L.orc_get_sorted(h, _ptr(sc), _ptr(sa), _ptr(st), _ptr(pm))
        cnt, sm, mn = np.empty(A * A, np.uint64), np.empty(A * A, np.int64), np.empty(A * A, np.float64)
        L.orc_get_dfg(h, _ptr(cnt), _ptr(sm), _ptr(mn))
        s0, e0 = np.empty(A, np.uint64), np.empty(A, np.uint64)
        L.orc_get_start_end(h, _ptr(s0), _ptr(e0))
        cc, ne, du, fr, cv = (np.empty(C, np.uint32), np.empty(C, np.uint32), np.empty(C, np.int64),
                              np.empty(C, np.int64), np.empty(C, np.uint32))
        L.orc_get_cases(h, _ptr(cc), _ptr(ne), _ptr(du), _ptr(fr), _ptr(cv))
        vc, vl, vr, vo, va = (np.empty(V, np.uint64), np.empty(V, np.uint32), np.empty(V, np.uint32),
                              np.empty(V + 1, np.uint64), np.empty(T, np.uint32))
        L.orc_get_variants(h, _ptr(vc), _ptr(vl), _ptr(vr), _ptr(vo), _ptr(va))
        ov = bool(L.orc_overflow(h))
        tsort, tloop = ctypes.c_double(0), ctypes.c_double(0)
        L.orc_timing(h, ctypes.byref(tsort), ctypes.byref(tloop))
    finally:
        L.orc_free(h)
    return OracleResult(A, sc, sa, st, pm, cnt.reshape(A, A), sm.reshape(A, A), mn.reshape(A, A),
                        s0, e0, cc, ne, du, fr, cv, vc, vl, vr, vo, va, ov, tsort.value, tloop.value)


def filter_time(case, ts, t1: int, t2: int, mode: int) -> np.ndarray:
    """P:126 / S:410-418: keep mask (bool, input order).  Raises on t1 > t2."""
    L = _load()
    c, t = _u32(case), _i64(ts)
    keep = np.zeros(c.size, np.uint8)
    st = L.orc_filter_time(c.size, _ptr(c), _ptr(t), int(t1), int(t2), int(mode), _ptr(keep))
    if st != 0:
        raise ValueError("EINVAL: t1 > t2 or bad mode (S:414)")
    return keep.astype(bool)


def filter_attr(case, col, *, codes=None, lo=None, hi=None, valid=None, level: int = 0,
                keep: bool = True) -> np.ndarray:
    """P:101, P:128 / S:445-453: keep mask (bool, input order).

    ``codes`` -> u32 in-set predicate; ``lo``/``hi`` ints -> i64 range; floats -> f64 range.
    """
    L = _load()
    c = _u32(case)
    out = np.zeros(c.size, np.uint8)
    v = None if valid is None else np.ascontiguousarray(np.asarray(valid, dtype=np.uint8))
    if codes is not None:
        kind, colv = 0, _u32(col)
        s = _u32(codes)
        args = (_ptr(s), s.size, 0, 0, 0.0, 0.0)
    elif isinstance(lo, float) or np.asarray(col).dtype.kind == "f":
        kind, colv = 2, np.ascontiguousarray(np.asarray(col, dtype=np.float64))
        args = (None, 0, 0, 0, float(lo), float(hi))
    else:
        kind, colv = 1, _i64(col)
        args = (None, 0, int(lo), int(hi), 0.0, 0.0)
    st = L.orc_filter_attr(c.size, _ptr(c), kind, _ptr(colv), _ptr(v), *args, int(level),
                           1 if keep else 0, _ptr(out))
    if st != 0:
        raise ValueError("EINVAL (S:449, S:458)")
    return out.astype(bool)


def dfg_minmax(case, act, ts, n_activities: int):
    """NEXT-2: per-edge min / max pair duration (u64, R20),
    0 where the edge never occurs.  Returns (min[A, A], max[A, A])."""
    L = _load()
    c, a, t = _u32(case), _u32(act), _i64(ts)
    A = int(n_activities)
    h = L.orc_run(c.size, _ptr(c), _ptr(a), _ptr(t), A)
    try:
        mn = np.zeros(A * A, np.uint64)
        mx = np.zeros(A * A, np.uint64)
        L.orc_get_dfg_minmax(h, _ptr(mn), _ptr(mx))
    finally:
        L.orc_free(h)
    return mn.reshape(A, A), mx.reshape(A, A)


CASE_START_IN, CASE_END_IN, CASE_SIZE, CASE_THROUGHPUT, CASE_PATHS = 0, 1, 2, 3, 4


def filter_cases(case, act, ts, kind: int, *, codes=None, lo: int = 0, hi: int = 0,
                 keep: bool = True) -> np.ndarray:
    """NEXT-1 whole-case filters: keep mask (bool, input
    order).  ``codes``: activity codes (START_IN / END_IN) or flattened pairs
    a0, b0, a1, b1, ... (PATHS).  Raises on lo > hi or an odd pair list."""
    L = _load()
    c, a, t = _u32(case), _u32(act), _i64(ts)
    cs = _u32([] if codes is None else codes)
    out = np.zeros(c.size, np.uint8)
    st = L.orc_filter_cases(c.size, _ptr(c), _ptr(a), _ptr(t), int(kind), _ptr(cs), cs.size,
                            int(lo), int(hi), 1 if keep else 0, _ptr(out))
    if st != 0:
        raise ValueError("EINVAL (S:459)")
    return out.astype(bool)


def filter_variants(case, act, ts, seqs, keep: bool = True) -> np.ndarray:
    """filter_by_variants: keep mask (bool, input order);
    ``seqs``: iterable of activity-code sequences."""
    L = _load()
    c, a, t = _u32(case), _u32(act), _i64(ts)
    seqs = [list(x) for x in seqs]
    off = np.zeros(len(seqs) + 1, np.uint64)
    for i, q in enumerate(seqs):
        off[i + 1] = off[i] + len(q)
    flat = _u32([x for q in seqs for x in q])
    out = np.zeros(c.size, np.uint8)
    L.orc_filter_variants(c.size, _ptr(c), _ptr(a), _ptr(t), _ptr(off), _ptr(flat), len(seqs),
                          1 if keep else 0, _ptr(out))
    return out.astype(bool)


def efg(case, act, ts, n_activities: int) -> dict:
    """NEXT-3: eventually-follows graph over all
    in-case ordered pairs i < j and the temporal profile (reading R22).
    Returns {"cnt", "sum" (u64), "sumsq" (Python int matrix as lo / hi u64),
    "sq_lo", "sq_hi", "mean", "stdev"}, each [A, A]."""
    L = _load()
    c, a, t = _u32(case), _u32(act), _i64(ts)
    A = int(n_activities)
    out = {k: np.zeros(A * A, np.uint64) for k in ("cnt", "sum", "sq_lo", "sq_hi")}
    out["mean"] = np.zeros(A * A, np.float64)
    out["stdev"] = np.zeros(A * A, np.float64)
    L.orc_efg(c.size, _ptr(c), _ptr(a), _ptr(t), A, _ptr(out["cnt"]), _ptr(out["sum"]),
              _ptr(out["sq_lo"]), _ptr(out["sq_hi"]), _ptr(out["mean"]), _ptr(out["stdev"]))
    return {k: v.reshape(A, A) for k, v in out.items()}
