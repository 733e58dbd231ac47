"""Whole-log bit-exact parity at BASELINE.json's full sizes ("each
reported number is checked against O1 first").

* 100M (configs[3], with its 2% timestamp ties): the bench's call,
  pm4g_sort_analyze, on the whole 10^8-event log; O1 runs once on the whole log
  (single process, ~35 s) and EVERY output is compared element by element --
  DFG counts / sums / means, start / end, all 10M per-case rows, the variant
  table in order with its sequences, every case's variant index and the whole
  formatted log (sorted case / activity / timestamp columns).
* 1B + events-mode time filter (configs[4], the north-star workload on one
  GPU): the GPU formats and analyses the filtered 8e8-row log in one piece.  O1
  runs on 16 contiguous case-range shards of the same log (R19: no case
  crosses a shard; the generator draws every shard's rows in the global
  ingest order restricted to its cases) in 8 worker processes, and the shard
  results are merged by the plain definitions: integer tables summed (exact,
  modulo 2^64 for the sums, R8), per-case rows concatenated in code order,
  variants keyed by their exact sequence (counts summed, representative = the
  smallest case code, R11), means recomputed as sum / count (R6).  Every output
  is compared, the formatted log shard by shard.
"""
from __future__ import annotations

import multiprocessing as mp

import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, T0_MS, generate
from tests.parity import assert_parity, collect
from paper_2204_04898_b200 import pm4g

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _device_log(spec, lo=0, hi=None):
    L = generate(spec, lo, hi, device="cuda")
    case = L.case.to(torch.uint32).contiguous()
    act = L.act.to(torch.uint8).contiguous()
    return L, case, act, L.ts.contiguous()


def test_100M_whole_log_bit_exact():
    spec = CONFIGS["100M"]
    A = spec.n_activities
    L, case, act, ts = _device_log(spec)
    log = pm4g.pm4g_log_create(case, act, ts, A, n_case_codes=spec.n_cases, borrow=True)
    g = collect(log, sort_analyze=True)
    log.close()
    c, a, t = case.cpu().numpy(), act.cpu().numpy(), ts.cpu().numpy()
    del L, case, act, ts
    torch.cuda.empty_cache()
    assert (np.diff(np.sort(t)) == 0).any()          # the log has timestamp ties
    r = oracle.run(c, a, t, A)
    assert not r.overflow
    assert r.n_cases == spec.n_cases and g["case_code"].size == spec.n_cases
    assert_parity(g, r)


# ------------------------------------------------------------------ 1B + filter, sharded O1
_SHARDS: list = []     # per shard: (case, act, ts) host arrays of the kept rows (fork-inherited)
_GPU: dict = {}        # the GPU's whole-log outputs (fork-inherited)


def _o1_shard(j):
    """O1 on shard j; compares the shard's slice of the GPU's per-case rows and
    formatted log here and returns the shard's tables and variants for the merge."""
    c, a, t, row0, case0 = _SHARDS[j]
    A = _GPU["A"]
    r = oracle.run(c, a, t, A)
    C = r.n_cases
    g = _GPU
    ok = {
        "case_code": np.array_equal(g["case_code"][case0:case0 + C], r.case_code),
        "n_events": np.array_equal(g["n_events"][case0:case0 + C], r.n_events),
        "dur": np.array_equal(g["dur"][case0:case0 + C], r.dur),
        "sorted_case": np.array_equal(g["sorted_case"][row0:row0 + c.size], r.sorted_case),
        "sorted_act": np.array_equal(g["sorted_act"][row0:row0 + c.size], r.sorted_act),
        "sorted_ts": np.array_equal(g["sorted_ts"][row0:row0 + c.size], r.sorted_ts),
    }
    return dict(ok=ok, C=C, n=c.size, cnt=r.cnt, sum=r.sum.view(np.uint64), start=r.start, end=r.end,
                v_count=r.v_count, v_rep=r.v_rep, v_off=r.v_off, v_act=r.v_act, case_variant=r.case_variant,
                overflow=r.overflow, t=r.t_sort + r.t_loop)


def test_1B_filter_whole_log_bit_exact():
    spec = CONFIGS["1B"]
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs a 180 GB B200")
    A = spec.n_activities
    t1, t2 = T0_MS + int(36.5 * 86_400_000), T0_MS + int(328.5 * 86_400_000)
    L, case, act, ts = _device_log(spec)
    log = pm4g.pm4g_log_create(case, act, ts, A, n_case_codes=spec.n_cases, borrow=True)
    f = log.filter_time(t1, t2)
    log.close()
    del L, case, act, ts
    g = collect(f, sort_analyze=True)
    n_kept = f.n
    f.close()
    torch.cuda.empty_cache()
    g["A"] = A
    _GPU.clear()
    _GPU.update(g)

    # the same log as R = 16 case-range shards (R19), filtered row by row
    R = 16
    _SHARDS.clear()
    row0 = case0 = 0
    bounds = [spec.n_cases * k // R for k in range(R + 1)]
    for j in range(R):
        Ls = generate(spec, bounds[j], bounds[j + 1], device="cuda")
        keep = (Ls.ts >= t1) & (Ls.ts <= t2)
        ck = Ls.case[keep]
        c = ck.cpu().numpy().astype(np.uint32)
        _SHARDS.append((c, Ls.act[keep].cpu().numpy().astype(np.uint8), Ls.ts[keep].cpu().numpy(), row0, case0))
        row0 += c.size
        case0 += int(torch.unique(ck).numel())
        del Ls, keep, ck
    torch.cuda.empty_cache()
    assert row0 == n_kept

    with mp.get_context("fork").Pool(8) as pool:
        parts = pool.map(_o1_shard, range(R))

    for j, p in enumerate(parts):
        assert not p["overflow"]
        assert all(p["ok"].values()), f"shard {j}: {p['ok']}"
    assert sum(p["C"] for p in parts) == g["case_code"].size
    # tables: summed over shards (u64 / int64 modulo 2^64, R8), mean = sum / cnt (R6)
    cnt = sum(p["cnt"].astype(np.uint64) for p in parts)
    sm = sum(p["sum"] for p in parts).view(np.int64)
    assert np.array_equal(g["cnt"], cnt) and np.array_equal(g["sum"], sm)
    nz = cnt > 0
    mean = np.zeros_like(g["mean"])
    mean[nz] = sm[nz].astype(np.float64) / cnt[nz].astype(np.float64)
    assert np.array_equal(g["mean"], mean)
    assert np.array_equal(g["start"], sum(p["start"] for p in parts))
    assert np.array_equal(g["end"], sum(p["end"] for p in parts))
    # variants: exact sequences, counts summed, representative = smallest case (R11)
    merged = {}
    local = []
    for p in parts:
        keys = []
        for i in range(p["v_count"].size):
            k = p["v_act"][p["v_off"][i]:p["v_off"][i + 1]].tobytes()
            keys.append(k)
            cnt_i, rep_i = merged.get(k, (0, 1 << 32))
            merged[k] = (cnt_i + int(p["v_count"][i]), min(rep_i, int(p["v_rep"][i])))
        local.append(keys)
    order = sorted(merged.items(), key=lambda kv: (-kv[1][0], kv[1][1]))
    pos = {k: i for i, (k, _) in enumerate(order)}
    assert g["v_count"].tolist() == [v[0] for _, v in order]
    assert g["v_rep"].tolist() == [v[1] for _, v in order]
    want_act = np.concatenate([np.frombuffer(k, np.uint32) for k, _ in order])
    assert np.array_equal(g["v_act"], want_act)
    assert np.array_equal(g["v_len"], np.array([len(k) // 4 for k, _ in order], np.uint32))
    case_variant = np.concatenate([np.array([pos[k] for k in keys], np.uint32)[p["case_variant"]]
                                   for keys, p in zip(local, parts)])
    assert np.array_equal(g["case_variant"], case_variant)


def test_wide_key_microseconds_whole_log_bit_exact():
    """The wide path at scale: the 100M recipe at 2e7 events / 2e6 cases with
    timestamps in MICROseconds (ms * 1000 + a per-row offset < 1000): a year
    spans 45 ts bits, 2e6 cases need 21 case bits -> a 66-bit composite key.
    pm4g_sort_analyze vs O1 on the whole log, every output."""
    spec = CONFIGS["100M"].with_(n_cases=2_000_000, n_events=20_000_000)
    A = spec.n_activities
    L, case, act, ts = _device_log(spec)
    ts_us = ts * 1000 + (torch.arange(ts.numel(), device=ts.device) * 7919) % 1000
    log = pm4g.pm4g_log_create(case, act, ts_us, A, n_case_codes=spec.n_cases, borrow=True)
    info = log.info()
    assert info.key_bits > 64 and 45 <= info.ts_bits <= 46 and info.case_bits == 21
    g = collect(log, sort_analyze=True)
    log.close()
    c, a, t = case.cpu().numpy(), act.cpu().numpy(), ts_us.cpu().numpy()
    r = oracle.run(c, a, t, A)
    assert_parity(g, r)
