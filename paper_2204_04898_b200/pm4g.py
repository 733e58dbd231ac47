"""Thin ctypes binding of libpm4g (include/pm4g.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels.  This module
only converts torch tensors to pointers/sizes, passes the current CUDA stream,
allocates output tensors and turns non-zero status codes into exceptions.
There is no CPU fallback: if libpm4g.so is missing, loading raises.

Functions keep the C names (pm4g_log_create, pm4g_sort, pm4g_dfg, ...); the
``Log`` / ``VariantTable`` classes are small conveniences over them.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpm4g.so")

PM4G_OK, PM4G_EINVAL, PM4G_EDATA, PM4G_ENOMEM, PM4G_ECUDA, PM4G_ENCCL, PM4G_EKEYWIDTH, PM4G_ECOLLISION = range(8)
PM4G_BORROW, PM4G_HOST_INPUT = 1, 2
PM4G_KIND_CODES, PM4G_KIND_I64, PM4G_KIND_F64 = 0, 1, 2
PM4G_TIME_EVENTS, PM4G_TIME_CASES_CONTAINED, PM4G_TIME_CASES_INTERSECTING = 0, 1, 2
PM4G_COL_ACTIVITY = -1
PM4G_PRED_IN_SET, PM4G_PRED_RANGE_I64, PM4G_PRED_RANGE_F64 = 0, 1, 2
PM4G_LEVEL_EVENTS, PM4G_LEVEL_CASES = 0, 1
PM4G_CASE_START_IN, PM4G_CASE_END_IN, PM4G_CASE_SIZE, PM4G_CASE_THROUGHPUT, PM4G_CASE_PATHS = range(5)

_STATUS = {1: "EINVAL", 2: "EDATA", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "EKEYWIDTH", 7: "ECOLLISION"}


class Pm4gError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"PM4G_{_STATUS.get(status, status)}: {msg}")
        self.status = status


P = ctypes.c_void_p
I32, I64, U32, U64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64


class pm4g_column(ctypes.Structure):
    _fields_ = [("kind", I32), ("data", P), ("valid", P), ("dict_size", U64)]


class pm4g_log_desc(ctypes.Structure):
    _fields_ = [("n_events", I64), ("case_code", P), ("act", P), ("act_bytes", I32), ("ts", P),
                ("n_case_codes", U64), ("case_lo", U32), ("case_hi", U32), ("n_activities", U32),
                ("n_extra", I32), ("extra", ctypes.POINTER(pm4g_column)), ("flags", U32)]


class pm4g_log_info(ctypes.Structure):
    _fields_ = [("n_events", I64), ("n_cases", I64), ("sorted", I32), ("act_bytes", I32),
                ("n_activities", U32), ("case_lo", U32), ("case_hi", U32), ("ts_min", I64),
                ("ts_max", I64), ("case_bits", I32), ("ts_bits", I32), ("key_bits", I32),
                ("radix_passes", I32)]


class pm4g_pred(ctypes.Structure):
    _fields_ = [("kind", I32), ("codes", P), ("n_codes", I64), ("lo_i", I64), ("hi_i", I64),
                ("lo_f", ctypes.c_double), ("hi_f", ctypes.c_double)]


class pm4g_case_pred(ctypes.Structure):
    _fields_ = [("kind", I32), ("codes", P), ("n_codes", I64), ("lo", I64), ("hi", I64)]


class pm4g_outputs(ctypes.Structure):
    _fields_ = [("cnt", P), ("dur_sum", P), ("mean", P), ("start", P), ("end", P),
                ("case_code", P), ("n_events", P), ("dur", P), ("capacity", U64),
                ("variants", ctypes.POINTER(P)), ("dur_min", P), ("dur_max", P)]


_SIGS = {
    "pm4g_log_create": ([ctypes.POINTER(pm4g_log_desc), P, ctypes.POINTER(P)], I32),
    "pm4g_log_create_filtered": ([ctypes.POINTER(pm4g_log_desc), I64, I64, P, ctypes.POINTER(P)], I32),
    "pm4g_log_destroy": ([P], I32),
    "pm4g_log_info_get": ([P, ctypes.POINTER(pm4g_log_info)], I32),
    "pm4g_sort": ([P, P], I32),
    "pm4g_sorted_columns": ([P, P, P, P, P], I32),
    "pm4g_dfg": ([P, P, P, P, P, P], I32),
    "pm4g_start_end": ([P, P, P, P, P], I32),
    "pm4g_dfg_minmax": ([P, P, P, P, P], I32),
    "pm4g_efg": ([P, P, P, P, P, P, P, P], I32),
    "pm4g_case_capacity": ([P, ctypes.POINTER(U64)], I32),
    "pm4g_repartition": ([P, P, P, P, ctypes.POINTER(P)], I32),
    "pm4g_partition_by_case": ([P, P, I32, P, ctypes.POINTER(P)], I32),
    "pm4g_log_concat": ([ctypes.POINTER(P), I32, U32, U32, P, ctypes.POINTER(P)], I32),
    "pm4g_case_durations": ([P, P, P, P, U64, ctypes.POINTER(U64), P], I32),
    "pm4g_variants": ([P, P, P, ctypes.POINTER(P)], I32),
    "pm4g_variants_size": ([P, ctypes.POINTER(U64), ctypes.POINTER(U64)], I32),
    "pm4g_variants_get": ([P, P, P, P, P, P, P], I32),
    "pm4g_variants_case_index": ([P, P, P], I32),
    "pm4g_variants_destroy": ([P], I32),
    "pm4g_analyze": ([P, ctypes.POINTER(pm4g_outputs), P, P], I32),
    "pm4g_sort_analyze": ([P, ctypes.POINTER(pm4g_outputs), P, P], I32),
    "pm4g_filter_time": ([P, I64, I64, I32, P, ctypes.POINTER(P)], I32),
    "pm4g_filter_attr": ([P, I32, ctypes.POINTER(pm4g_pred), I32, I32, P, ctypes.POINTER(P)], I32),
    "pm4g_filter_cases": ([P, ctypes.POINTER(pm4g_case_pred), I32, P, ctypes.POINTER(P)], I32),
    "pm4g_filter_variants": ([P, P, P, I64, I32, P, ctypes.POINTER(P)], I32),
    "pm4g_comm_unique_id": ([P, ctypes.POINTER(ctypes.c_size_t)], I32),
    "pm4g_comm_create": ([P, I32, I32, ctypes.POINTER(P)], I32),
    "pm4g_comm_destroy": ([P], I32),
    "pm4g_variants_merge": ([ctypes.POINTER(P), I32, I32, P, ctypes.POINTER(P)], I32),
    "pm4g_sum_u64": ([P, I32, U64, P, P], I32),
    "pm4g_tables_partial": ([P, P, P], I32),
    "pm4g_tables_finalize": ([P, U32, P, P, P, P, P, P], I32),
    "pm4g_last_error": ([], ctypes.c_char_p),
    "pm4g_version": ([], ctypes.c_char_p),
    "pm4g_launch_count": ([], U64),
    "pm4g_mem_stats": ([ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U64)], I32),
    "pm4g_mem_release": ([], I32),
    "pm4g_prof_enable": ([I32], I32),
    "pm4g_prof_reset": ([], I32),
    "pm4g_prof_collect": ([ctypes.POINTER(I32)], I32),
    "pm4g_prof_n_records": ([], I32),
    "pm4g_prof_record": ([I32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double)], I32),
    "pm4g_prof_entry": ([I32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(U64),
                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], I32),
}

_lib = None


def lib():
    """Load libpm4g.so (built by paper_2204_04898_b200.build).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2204_04898_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int):
    if st != PM4G_OK:
        raise Pm4gError(st, lib().pm4g_last_error().decode())


def _ptr(t):
    # a plain int: ctypes converts it for c_void_p arguments and fields
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def _stream(stream):
    if stream is None:   # the current stream's raw handle (torch.cuda.current_stream() costs ~15 us a call)
        return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))
    return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _dev():
    return torch.device("cuda", torch._C._cuda_getDevice())


def act_bytes_for(n_activities: int) -> int:
    return 1 if n_activities <= 256 else (2 if n_activities <= 65536 else 4)


# ================================================================ log
@dataclass
class Extra:
    kind: int                 # PM4G_KIND_*
    data: torch.Tensor        # [n] u32 codes (int32/uint32), int64 or float64
    valid: torch.Tensor | None = None   # [n] uint8 (1 = present)
    dict_size: int = 0


def pm4g_log_create(case: torch.Tensor, act: torch.Tensor, ts: torch.Tensor, n_activities: int,
                    n_case_codes: int | None = None, case_lo: int = 0, case_hi: int = 0,
                    extra: list[Extra] | None = None, borrow: bool = False, stream=None,
                    time_filter: tuple[int, int] | None = None) -> "Log":
    """Columns are CUDA tensors (device input) or CPU tensors (PM4G_HOST_INPUT: copied H2D
    inside the call).  case: 4-byte codes; act: 1/2/4-byte codes; ts: int64.
    time_filter=(t1, t2): pm4g_log_create_filtered (create + events-mode time filter, one pass)."""
    n = int(case.numel())
    host = not case.is_cuda
    for t in (case, act, ts):
        assert t.is_contiguous() and t.numel() == n and t.is_cuda == (not host)
    assert case.element_size() == 4 and ts.dtype == torch.int64
    if n_case_codes is None:
        n_case_codes = int(case.to(torch.int64).max().item()) + 1 if n else 1
    ex = extra or []
    cols = (pm4g_column * max(1, len(ex)))()
    for i, x in enumerate(ex):
        cols[i] = pm4g_column(x.kind, _ptr(x.data), _ptr(x.valid), x.dict_size)
    d = pm4g_log_desc(n, _ptr(case), _ptr(act), act.element_size(), _ptr(ts), n_case_codes,
                      case_lo, case_hi, n_activities, len(ex), cols,
                      (PM4G_HOST_INPUT if host else 0) | (PM4G_BORROW if borrow else 0))
    out = ctypes.c_void_p()
    if time_filter is None:
        _check(lib().pm4g_log_create(ctypes.byref(d), _stream(stream), ctypes.byref(out)))
    else:
        _check(lib().pm4g_log_create_filtered(ctypes.byref(d), int(time_filter[0]), int(time_filter[1]),
                                              _stream(stream), ctypes.byref(out)))
    keep = (case, act, ts, ex) if borrow else None
    return Log(out, n_activities, act.element_size(), keep)


class Log:
    def __init__(self, handle, n_activities: int, act_bytes: int, keepalive=None):
        self.h = handle
        self.A = n_activities
        self.act_bytes = act_bytes
        self._keep = keepalive

    def close(self):
        if self.h:
            lib().pm4g_log_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> pm4g_log_info:
        i = pm4g_log_info()
        _check(lib().pm4g_log_info_get(self.h, ctypes.byref(i)))
        return i

    @property
    def n(self) -> int:
        return self.info().n_events

    def sort(self, stream=None) -> "Log":
        _check(lib().pm4g_sort(self.h, _stream(stream)))
        return self

    def sorted_columns(self, stream=None):
        n = self.n
        dev = _dev()
        c = torch.empty(n, dtype=torch.uint32, device=dev)
        a = torch.empty(n, dtype=torch.uint32, device=dev)
        t = torch.empty(n, dtype=torch.int64, device=dev)
        _check(lib().pm4g_sorted_columns(self.h, _ptr(c), _ptr(a), _ptr(t), _stream(stream)))
        return c, a, t

    def dfg(self, comm=None, stream=None, with_mean=True):
        A, dev = self.A, _dev()
        cnt = torch.empty(A * A, dtype=torch.int64, device=dev)
        sm = torch.empty(A * A, dtype=torch.int64, device=dev)
        mean = torch.empty(A * A, dtype=torch.float64, device=dev) if with_mean else None
        _check(lib().pm4g_dfg(self.h, _ptr(cnt), _ptr(sm), _ptr(mean), _comm(comm), _stream(stream)))
        return cnt.view(A, A), sm.view(A, A), (mean.view(A, A) if with_mean else None)

    def dfg_minmax(self, comm=None, stream=None):
        """NEXT-2: per-edge (min, max) pair duration, u64 as int64 tensors [A, A]."""
        A, dev = self.A, _dev()
        mn = torch.empty(A * A, dtype=torch.int64, device=dev)
        mx = torch.empty(A * A, dtype=torch.int64, device=dev)
        _check(lib().pm4g_dfg_minmax(self.h, _ptr(mn), _ptr(mx), _comm(comm), _stream(stream)))
        return mn.view(A, A), mx.view(A, A)

    def efg(self, comm=None, stream=None):
        """NEXT-3: eventually-follows graph + temporal profile.  Returns a dict of
        [A, A] tensors: cnt, sum (u64 as int64), sumsq_lo / sumsq_hi (the u128
        sum of squared durations), mean, stdev."""
        A, dev = self.A, _dev()
        cnt = torch.empty(A * A, dtype=torch.int64, device=dev)
        sm = torch.empty(A * A, dtype=torch.int64, device=dev)
        sq = torch.empty(2 * A * A, dtype=torch.int64, device=dev)
        mean = torch.empty(A * A, dtype=torch.float64, device=dev)
        sd = torch.empty(A * A, dtype=torch.float64, device=dev)
        _check(lib().pm4g_efg(self.h, _ptr(cnt), _ptr(sm), _ptr(sq), _ptr(mean), _ptr(sd), _comm(comm),
                              _stream(stream)))
        return {"cnt": cnt.view(A, A), "sum": sm.view(A, A), "sumsq_lo": sq[:A * A].view(A, A),
                "sumsq_hi": sq[A * A:].view(A, A), "mean": mean.view(A, A), "stdev": sd.view(A, A)}

    def start_end(self, comm=None, stream=None):
        A, dev = self.A, _dev()
        st = torch.empty(A, dtype=torch.int64, device=dev)
        en = torch.empty(A, dtype=torch.int64, device=dev)
        _check(lib().pm4g_start_end(self.h, _ptr(st), _ptr(en), _comm(comm), _stream(stream)))
        return st, en

    def case_durations(self, stream=None):
        C = self.info().n_cases
        dev = _dev()
        cc = torch.empty(C, dtype=torch.uint32, device=dev)
        ne = torch.empty(C, dtype=torch.uint32, device=dev)
        du = torch.empty(C, dtype=torch.int64, device=dev)
        nc = U64(0)
        _check(lib().pm4g_case_durations(self.h, _ptr(cc), _ptr(ne), _ptr(du), C, ctypes.byref(nc),
                                         _stream(stream)))
        return cc, ne, du

    def variants(self, comm=None, stream=None) -> "VariantTable":
        out = ctypes.c_void_p()
        _check(lib().pm4g_variants(self.h, _comm(comm), _stream(stream), ctypes.byref(out)))
        return VariantTable(out)

    def case_capacity(self) -> int:
        """Host-known upper bound on n_cases (no device synchronisation)."""
        c = U64(0)
        _check(lib().pm4g_case_capacity(self.h, ctypes.byref(c)))
        return c.value

    def analyze(self, comm=None, stream=None, tables=True, cases=True, variants=True, out=None,
                minmax=False, _entry="pm4g_analyze"):
        """Fused pass.  ``out``: optional dict of tensors, filled on first use and reused
        by later calls (per-case arrays are sized by case_capacity(), valid up to
        info().n_cases).  ``minmax``: also the per-edge min / max durations."""
        A, dev = self.A, _dev()
        C = self.case_capacity() if cases else 0
        o = out if out is not None else {}
        def need(k, size, dt):
            if k not in o or o[k].numel() < size:
                o[k] = torch.empty(size, dtype=dt, device=dev)
        want = set()
        if tables:
            for k, sz, dt in (("cnt", A * A, torch.int64), ("dur_sum", A * A, torch.int64),
                              ("mean", A * A, torch.float64), ("start", A, torch.int64), ("end", A, torch.int64)):
                need(k, sz, dt)
                want.add(k)
        if minmax:
            for k in ("dur_min", "dur_max"):
                need(k, A * A, torch.int64)
                want.add(k)
        if cases:
            for k, dt in (("case_code", torch.uint32), ("n_events", torch.uint32), ("dur", torch.int64)):
                need(k, C, dt)
                want.add(k)
        vh = ctypes.c_void_p()
        g = lambda k: _ptr(o[k]) if k in want else None  # noqa: E731
        outs = pm4g_outputs(g("cnt"), g("dur_sum"), g("mean"), g("start"), g("end"),
                            g("case_code"), g("n_events"), g("dur"),
                            min((o[k].numel() for k in ("case_code", "n_events", "dur") if k in want), default=0),
                            ctypes.pointer(vh) if variants else None, g("dur_min"), g("dur_max"))
        _check(getattr(lib(), _entry)(self.h, ctypes.byref(outs), _comm(comm), _stream(stream)))
        res = {k: o[k] for k in want}
        if variants:
            res["variants"] = VariantTable(vh)
        return res

    def sort_analyze(self, comm=None, stream=None, tables=True, cases=True, variants=True, out=None,
                     minmax=False):
        """pm4g_sort_analyze: sort() then analyze() in one call (same results; the sort's
        host check is folded into the analysis' synchronisation)."""
        return self.analyze(comm=comm, stream=stream, tables=tables, cases=cases, variants=variants,
                            out=out, minmax=minmax, _entry="pm4g_sort_analyze")

    def filter_time(self, t1: int, t2: int, mode: int = PM4G_TIME_EVENTS, stream=None) -> "Log":
        out = ctypes.c_void_p()
        _check(lib().pm4g_filter_time(self.h, int(t1), int(t2), int(mode), _stream(stream), ctypes.byref(out)))
        return Log(out, self.A, self.act_bytes)

    def filter_attr(self, column: int = PM4G_COL_ACTIVITY, codes=None, lo=None, hi=None,
                    level: int = PM4G_LEVEL_EVENTS, keep: bool = True, stream=None) -> "Log":
        codes_arr = None
        if codes is not None:
            vals = [int(c) for c in codes]
            codes_arr = (U32 * max(1, len(vals)))(*vals)
            pred = pm4g_pred(PM4G_PRED_IN_SET, ctypes.cast(codes_arr, P), len(vals), 0, 0, 0.0, 0.0)
        elif isinstance(lo, float) or isinstance(hi, float):
            pred = pm4g_pred(PM4G_PRED_RANGE_F64, None, 0, 0, 0, float(lo), float(hi))
        else:
            pred = pm4g_pred(PM4G_PRED_RANGE_I64, None, 0, int(lo), int(hi), 0.0, 0.0)
        out = ctypes.c_void_p()
        _check(lib().pm4g_filter_attr(self.h, int(column), ctypes.byref(pred), int(level),
                                      1 if keep else 0, _stream(stream), ctypes.byref(out)))
        return Log(out, self.A, self.act_bytes)

    def repartition(self, bounds, comm, stream=None) -> "Log":
        """NEXT-4: all-to-all by case range over NCCL; this rank receives the rows with
        bounds[rank] <= case < bounds[rank + 1] of every rank's (ingested) log."""
        arr = (U32 * len(bounds))(*[int(b) for b in bounds])
        out = ctypes.c_void_p()
        _check(lib().pm4g_repartition(self.h, ctypes.cast(arr, P), _comm(comm), _stream(stream), ctypes.byref(out)))
        return Log(out, self.A, self.act_bytes)

    def partition_by_case(self, bounds, stream=None) -> list:
        """The same split on one device: one new ingested log per case range."""
        R = len(bounds) - 1
        arr = (U32 * len(bounds))(*[int(b) for b in bounds])
        outs = (P * R)()
        _check(lib().pm4g_partition_by_case(self.h, ctypes.cast(arr, P), R, _stream(stream),
                                            ctypes.cast(outs, ctypes.POINTER(P))))
        return [Log(ctypes.c_void_p(outs[i]), self.A, self.act_bytes) for i in range(R)]

    def filter_cases(self, kind: int, codes=None, lo: int = 0, hi: int = 0, keep: bool = True,
                     stream=None) -> "Log":
        """NEXT-1 whole-case filter (formatted log): PM4G_CASE_START_IN / END_IN (codes),
        SIZE / THROUGHPUT (lo, hi inclusive), PATHS (codes = flattened (a, b) pairs)."""
        vals = [int(c) for c in (codes or [])]
        arr = (U32 * max(1, len(vals)))(*vals)
        pred = pm4g_case_pred(int(kind), ctypes.cast(arr, P) if vals else None, len(vals), int(lo), int(hi))
        out = ctypes.c_void_p()
        _check(lib().pm4g_filter_cases(self.h, ctypes.byref(pred), 1 if keep else 0, _stream(stream),
                                       ctypes.byref(out)))
        return Log(out, self.A, self.act_bytes)

    def filter_variants(self, seqs, keep: bool = True, stream=None) -> "Log":
        """filter_by_variants: keep / remove the cases whose exact activity
        sequence is one of ``seqs`` (iterable of code sequences)."""
        seqs = [[int(x) for x in q] for q in seqs]
        off = [0]
        for q in seqs:
            off.append(off[-1] + len(q))
        flat = [x for q in seqs for x in q]
        off_arr = (U64 * len(off))(*off)
        act_arr = (U32 * max(1, len(flat)))(*flat)
        out = ctypes.c_void_p()
        _check(lib().pm4g_filter_variants(self.h, ctypes.cast(off_arr, P), ctypes.cast(act_arr, P),
                                          len(seqs), 1 if keep else 0, _stream(stream), ctypes.byref(out)))
        return Log(out, self.A, self.act_bytes)


# ================================================================ variants
class VariantTable:
    def __init__(self, handle):
        self.h = handle

    def close(self):
        if self.h:
            lib().pm4g_variants_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self):
        v, t = U64(0), U64(0)
        _check(lib().pm4g_variants_size(self.h, ctypes.byref(v), ctypes.byref(t)))
        return v.value, t.value

    def get(self, stream=None) -> dict:
        V, T = self.size()
        dev = _dev()
        o = {"count": torch.empty(V, dtype=torch.int64, device=dev),
             "len": torch.empty(V, dtype=torch.uint32, device=dev),
             "rep_case": torch.empty(V, dtype=torch.uint32, device=dev),
             "seq_off": torch.empty(V + 1, dtype=torch.int64, device=dev),
             "seq_act": torch.empty(T, dtype=torch.uint32, device=dev)}
        _check(lib().pm4g_variants_get(self.h, _ptr(o["count"]), _ptr(o["len"]), _ptr(o["rep_case"]),
                                       _ptr(o["seq_off"]), _ptr(o["seq_act"]), _stream(stream)))
        return o

    def case_index(self, n_cases: int, stream=None) -> torch.Tensor:
        out = torch.empty(n_cases, dtype=torch.uint32, device=_dev())
        _check(lib().pm4g_variants_case_index(self.h, _ptr(out), _stream(stream)))
        return out

    def as_dict(self) -> dict:
        """{activity tuple: count} on the host (for tests / presentation)."""
        o = {k: v.cpu() for k, v in self.get().items()}
        torch.cuda.synchronize()
        off, acts, cnt = o["seq_off"].tolist(), o["seq_act"].tolist(), o["count"].tolist()
        return {tuple(acts[off[i]:off[i + 1]]): cnt[i] for i in range(len(cnt))}


def pm4g_variants_merge(parts: list, local_part: int = -1, stream=None) -> VariantTable:
    arr = (P * len(parts))(*[p.h for p in parts])
    out = ctypes.c_void_p()
    _check(lib().pm4g_variants_merge(arr, len(parts), int(local_part), _stream(stream), ctypes.byref(out)))
    return VariantTable(out)


def pm4g_log_concat(logs: list, case_lo: int, case_hi: int, stream=None) -> Log:
    """Concatenate ingested logs (in order) into one log with case range [case_lo, case_hi)."""
    arr = (P * len(logs))(*[lg.h for lg in logs])
    out = ctypes.c_void_p()
    _check(lib().pm4g_log_concat(arr, len(logs), int(case_lo), int(case_hi), _stream(stream), ctypes.byref(out)))
    return Log(out, logs[0].A, logs[0].act_bytes)


def pm4g_sum_u64(parts: torch.Tensor, stream=None) -> torch.Tensor:
    """parts: [R, len] int64/uint64 CUDA tensor -> [len] sum (the C1 reduction)."""
    R, L = parts.shape
    out = torch.empty(L, dtype=parts.dtype, device=parts.device)
    _check(lib().pm4g_sum_u64(_ptr(parts.contiguous()), R, L, _ptr(out), _stream(stream)))
    return out


def pm4g_tables_partial(log: Log, stream=None) -> torch.Tensor:
    A = log.A
    packed = torch.empty(2 * A * A + 2 * A, dtype=torch.int64, device=_dev())
    _check(lib().pm4g_tables_partial(log.h, _ptr(packed), _stream(stream)))
    return packed


def pm4g_tables_finalize(packed: torch.Tensor, A: int, stream=None):
    dev = packed.device
    cnt = torch.empty(A * A, dtype=torch.int64, device=dev)
    sm = torch.empty(A * A, dtype=torch.int64, device=dev)
    mean = torch.empty(A * A, dtype=torch.float64, device=dev)
    st = torch.empty(A, dtype=torch.int64, device=dev)
    en = torch.empty(A, dtype=torch.int64, device=dev)
    _check(lib().pm4g_tables_finalize(_ptr(packed), A, _ptr(cnt), _ptr(sm), _ptr(mean), _ptr(st), _ptr(en),
                                      _stream(stream)))
    return cnt.view(A, A), sm.view(A, A), mean.view(A, A), st, en


# ================================================================ comm
class Comm:
    """NCCL communicator owned by libpm4g; torch.distributed only carries the id."""

    def __init__(self, handle, nranks, rank):
        self.h, self.nranks, self.rank = handle, nranks, rank

    def close(self):
        if self.h:
            lib().pm4g_comm_destroy(self.h)
            self.h = None


def pm4g_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    sz = ctypes.c_size_t(0)
    _check(lib().pm4g_comm_unique_id(buf, ctypes.byref(sz)))
    return buf.raw[: sz.value]


def pm4g_comm_create(uid: bytes, nranks: int, rank: int) -> Comm:
    buf = ctypes.create_string_buffer(bytes(uid).ljust(128, b"\0"), 128)
    out = ctypes.c_void_p()
    _check(lib().pm4g_comm_create(buf, nranks, rank, ctypes.byref(out)))
    return Comm(out, nranks, rank)


def _comm(c):
    return c.h if c is not None else None


# ================================================================ diagnostics
def pm4g_launch_count() -> int:
    return int(lib().pm4g_launch_count())


def pm4g_mem_stats() -> dict:
    """Device memory the library holds: live blocks / bytes and cached bytes."""
    b, n, c = U64(0), U64(0), U64(0)
    _check(lib().pm4g_mem_stats(ctypes.byref(b), ctypes.byref(n), ctypes.byref(c)))
    return {"live_blocks": int(b.value), "live_bytes": int(n.value), "cached_bytes": int(c.value)}


def pm4g_mem_release():
    _check(lib().pm4g_mem_release())


def pm4g_prof_enable(on: bool = True):
    _check(lib().pm4g_prof_enable(1 if on else 0))


def pm4g_prof_reset():
    _check(lib().pm4g_prof_reset())


def pm4g_prof_collect() -> dict:
    """{kernel name: (launches, total ms, algorithmic bytes)}; synchronises."""
    n = I32(0)
    _check(lib().pm4g_prof_collect(ctypes.byref(n)))
    out = {}
    for i in range(n.value):
        nm, la, ms, by = ctypes.c_char_p(), U64(0), ctypes.c_double(0), ctypes.c_double(0)
        _check(lib().pm4g_prof_entry(i, ctypes.byref(nm), ctypes.byref(la), ctypes.byref(ms), ctypes.byref(by)))
        out[nm.value.decode()] = (la.value, ms.value, by.value)
    return out


def pm4g_prof_records() -> list:
    """[(name, start_ms, dur_ms)] of the last pm4g_prof_collect, in launch order."""
    out = []
    for i in range(int(lib().pm4g_prof_n_records())):
        nm, t0, d = ctypes.c_char_p(), ctypes.c_double(0), ctypes.c_double(0)
        _check(lib().pm4g_prof_record(i, ctypes.byref(nm), ctypes.byref(t0), ctypes.byref(d)))
        out.append((nm.value.decode(), t0.value, d.value))
    return out


pm4g_sort = Log.sort
pm4g_dfg = Log.dfg
pm4g_start_end = Log.start_end
pm4g_case_durations = Log.case_durations
pm4g_variants = Log.variants
pm4g_analyze = Log.analyze
pm4g_filter_time = Log.filter_time
pm4g_filter_attr = Log.filter_attr
pm4g_filter_cases = Log.filter_cases
pm4g_filter_variants = Log.filter_variants
pm4g_dfg_minmax = Log.dfg_minmax
pm4g_efg = Log.efg
pm4g_repartition = Log.repartition
pm4g_partition_by_case = Log.partition_by_case
pm4g_case_capacity = Log.case_capacity
