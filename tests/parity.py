"""Parity helpers: run the CUDA path through the C-ABI binding and compare with O1.

Used by tests/test_gpu_*.py and __graft_entry__.smoke().  Integer outputs must
match bit for bit; fp64 means within 1e-12 relative (north_star tolerance).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2204_04898_b200 import pm4g

MEAN_RTOL = 1e-12


def to_device_cols(case, act, ts, A, device="cuda"):
    case_t = torch.as_tensor(np.asarray(case, dtype=np.int64)).to(torch.uint32).contiguous()
    act_np = np.asarray(act, dtype=np.int64)
    ab = pm4g.act_bytes_for(A)
    adt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[ab]
    act_t = torch.as_tensor(act_np).to(torch.int32).to(adt) if ab != 1 else torch.as_tensor(act_np).to(torch.uint8)
    ts_t = torch.as_tensor(np.asarray(ts, dtype=np.int64)).contiguous()
    if device is None:
        return case_t, act_t.contiguous(), ts_t
    return case_t.to(device), act_t.contiguous().to(device), ts_t.to(device)


def gpu_run(case, act, ts, A, n_case_codes=None, case_lo=0, case_hi=0, sort=True, fused=True,
            sort_analyze=False):
    """Build a log on cuda:0, sort it, and return every output on the host
    (sort_analyze: one pm4g_sort_analyze call instead of pm4g_sort + pm4g_analyze)."""
    c, a, t = to_device_cols(case, act, ts, A)
    if n_case_codes is None:
        n_case_codes = (int(np.max(np.asarray(case, dtype=np.int64))) + 1) if len(case) else 1
    log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=n_case_codes, case_lo=case_lo, case_hi=case_hi)
    if not sort_analyze:
        log.sort()
    out = collect(log, fused=fused, sort_analyze=sort_analyze)
    log.close()
    return out


def collect(log, fused=True, sort_analyze=False):
    A = log.A
    res = {}
    if sort_analyze:
        o = log.sort_analyze()
        vt = o.pop("variants")
    elif fused:
        o = log.analyze()
        vt = o.pop("variants")
    else:
        cnt, sm, mean = log.dfg()
        st, en = log.start_end()
        cc, ne, du = log.case_durations()
        o = dict(cnt=cnt, dur_sum=sm, mean=mean, start=st, end=en, case_code=cc, n_events=ne, dur=du)
        vt = log.variants()
    C = log.info().n_cases
    v = vt.get()
    ci = vt.case_index(C)
    torch.cuda.synchronize()
    res["cnt"] = o["cnt"].view(-1).cpu().numpy().view(np.uint64).reshape(A, A)
    res["sum"] = o["dur_sum"].view(-1).cpu().numpy().reshape(A, A)
    res["mean"] = o["mean"].view(-1).cpu().numpy().reshape(A, A)
    res["start"] = o["start"].cpu().numpy().view(np.uint64)
    res["end"] = o["end"].cpu().numpy().view(np.uint64)
    res["case_code"] = o["case_code"][:C].cpu().numpy()
    res["n_events"] = o["n_events"][:C].cpu().numpy()
    res["dur"] = o["dur"][:C].cpu().numpy()
    res["v_count"] = v["count"].cpu().numpy().view(np.uint64)
    res["v_len"] = v["len"].cpu().numpy()
    res["v_rep"] = v["rep_case"].cpu().numpy()
    res["v_off"] = v["seq_off"].cpu().numpy().view(np.uint64)
    res["v_act"] = v["seq_act"].cpu().numpy()
    res["case_variant"] = ci.cpu().numpy()
    sc, sa, stt = log.sorted_columns()
    torch.cuda.synchronize()
    res["sorted_case"], res["sorted_act"], res["sorted_ts"] = sc.cpu().numpy(), sa.cpu().numpy(), stt.cpu().numpy()
    vt.close()
    return res


def assert_parity(g: dict, r: "oracle.OracleResult", check_sorted: bool = True):
    assert np.array_equal(g["cnt"], r.cnt), "DFG counts differ"
    assert np.array_equal(g["sum"], r.sum), "DFG duration sums differ"
    nz = r.cnt > 0
    assert np.all(g["mean"][~nz] == 0.0)
    if nz.any():
        ref = r.mean[nz]
        err = np.abs(g["mean"][nz] - ref) / np.maximum(np.abs(ref), 1e-300)
        assert np.all((err <= MEAN_RTOL) | (g["mean"][nz] == ref)), f"mean rel err {err.max()}"
    assert np.array_equal(g["start"], r.start), "start activities differ"
    assert np.array_equal(g["end"], r.end), "end activities differ"
    assert np.array_equal(g["case_code"], r.case_code), "case codes differ"
    assert np.array_equal(g["n_events"], r.n_events), "events per case differ"
    assert np.array_equal(g["dur"], r.dur), "case durations differ"
    assert np.array_equal(g["v_count"], r.v_count), "variant counts differ"
    assert np.array_equal(g["v_len"], r.v_len), "variant lengths differ"
    assert np.array_equal(g["v_rep"], r.v_rep), "variant representatives differ"
    assert np.array_equal(g["v_off"], r.v_off), "variant offsets differ"
    assert np.array_equal(g["v_act"], r.v_act), "variant sequences differ"
    assert np.array_equal(g["case_variant"], r.case_variant), "case -> variant differs"
    if check_sorted:
        assert np.array_equal(g["sorted_case"], r.sorted_case), "sorted case column differs"
        assert np.array_equal(g["sorted_act"], r.sorted_act), "sorted activity column differs"
        assert np.array_equal(g["sorted_ts"], r.sorted_ts), "sorted timestamps differ"


def check_log(case, act, ts, A, **kw):
    r = oracle.run(case, act, ts, A)
    g = gpu_run(case, act, ts, A, **kw)
    assert_parity(g, r)
    return g, r
