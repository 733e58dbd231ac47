"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot run 10^8-10^9 events in a test, so these tests check
(a) properties that hold at any size (S:282, S:332, S:359, S:422, S:206,
    telescoping of duration sums),
(b) closed forms from the generator's planted structure on the no-tie twin
    (DFG counts = sum_v m_v pairs(v), start/end, the variant multiset), and
(c) sampled cases one by one against O1: their formatted rows, events per
    case, duration and variant sequence.
"""
import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from paper_2204_04898_b200 import pm4g

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(spec, no_ties):
    L = generate(spec, device="cuda", no_ties=no_ties)
    case = L.case.to(torch.uint32)
    act = L.act.to(torch.uint8 if spec.n_activities <= 256 else torch.int16)
    log = pm4g.pm4g_log_create(case, act, L.ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
    log.sort()
    o = log.analyze()
    return L, log, o


def _planted_tables(L, A):
    """Expected tables of the no-tie twin: pool cases from the planted assignment
    (sum_v m_v pairs(v)); the few cases drawn as fresh random walks (lengths the
    pool does not cover) through O1 on exactly their events."""
    m = torch.bincount(L.case_variant[L.case_variant >= 0], minlength=len(L.pool_seqs)).cpu().numpy()
    cnt = np.zeros((A, A), np.int64)
    start = np.zeros(A, np.int64)
    end = np.zeros(A, np.int64)
    want = {}
    walk = torch.nonzero(L.case_variant < 0).flatten() + L.case_lo
    if walk.numel():
        sel = torch.isin(L.case, walk)
        r = oracle.run(L.case[sel].cpu().numpy(), L.act[sel].cpu().numpy(), L.ts[sel].cpu().numpy(), A)
        cnt += r.cnt.astype(np.int64).reshape(A, A)
        start += r.start.astype(np.int64)
        end += r.end.astype(np.int64)
        want.update(r.variants())
    for v, seq in enumerate(L.pool_seqs):
        if m[v] == 0:
            continue
        for a, b in zip(seq, seq[1:]):
            cnt[a, b] += m[v]
        start[seq[0]] += m[v]
        end[seq[-1]] += m[v]
        want[tuple(seq)] = want.get(tuple(seq), 0) + int(m[v])
    return cnt, start, end, want


@pytest.mark.parametrize("name", ["100M"])
def test_full_size_no_tie_closed_form(name):
    spec = CONFIGS[name]
    A = spec.n_activities
    L, log, o = _run(spec, no_ties=True)
    assert int((L.case_variant < 0).sum()) < spec.n_cases // 1000   # nearly all from the pool
    cnt, start, end, want = _planted_tables(L, A)
    got_cnt = o["cnt"].cpu().numpy().reshape(A, A)
    assert np.array_equal(got_cnt, cnt)
    assert np.array_equal(o["start"].cpu().numpy(), start) and np.array_equal(o["end"].cpu().numpy(), end)
    v = o["variants"].as_dict()
    assert v == want


def _sample_check(L, log, o, spec, k=1500, seed=0):
    """k random cases: rows / n_events / duration / variant vs O1 on exactly those cases."""
    A = spec.n_activities
    C = log.info().n_cases
    rng = np.random.default_rng(seed)
    pick = np.sort(rng.choice(spec.n_cases, size=min(k, spec.n_cases), replace=False))

    def member(codes):   # rows whose case is in `codes` (a lookup table: torch.isin sorts n values)
        m = torch.zeros(spec.n_cases, dtype=torch.bool, device=L.case.device)
        m[torch.as_tensor(codes, device=L.case.device)] = True
        return m[L.case.to(torch.int64)]

    sel = member(pick)
    c, a, t = L.case[sel].cpu().numpy(), L.act[sel].cpu().numpy(), L.ts[sel].cpu().numpy()
    r = oracle.run(c, a, t, A)
    # GPU per-case outputs are in case-code order; the workload's codes are dense
    cc = o["case_code"][:C].cpu().numpy()
    assert cc.size == spec.n_cases and np.array_equal(cc[pick], pick.astype(np.uint32))
    assert np.array_equal(o["n_events"][:C].cpu().numpy()[pick], r.n_events)
    assert np.array_equal(o["dur"][:C].cpu().numpy()[pick], r.dur)
    # formatted rows of the sampled cases
    sc, sa, st = log.sorted_columns()
    offs = torch.cumsum(o["n_events"][:C].to(torch.int64), 0) - o["n_events"][:C].to(torch.int64)
    rows = torch.cat([torch.arange(int(offs[p]), int(offs[p]) + int(o["n_events"][p]), device=sc.device)
                      for p in pick[:200]])
    s200 = member(pick[:200])
    sub = oracle.run(L.case[s200].cpu().numpy(), L.act[s200].cpu().numpy(), L.ts[s200].cpu().numpy(), A)
    # (u32 columns viewed as i32 to gather: codes < 2^31)
    assert np.array_equal(sa.view(torch.int32)[rows].to(torch.int64).cpu().numpy(), sub.sorted_act)
    assert np.array_equal(st[rows].cpu().numpy(), sub.sorted_ts)
    assert np.array_equal(sc.view(torch.int32)[rows].to(torch.int64).cpu().numpy(), sub.sorted_case)
    del sc, sa, st
    # variant of each sampled case = its exact sequence (the oracle's per-case sequence)
    vt = o["variants"].get()
    ci = o["variants"].case_index(C).cpu().numpy()
    off, acts = vt["seq_off"].cpu().numpy(), vt["seq_act"].cpu().numpy()
    for j, p in enumerate(pick[:300]):
        vi = ci[p]
        seq = acts[off[vi]:off[vi + 1]].tolist()
        want = r.v_act[r.v_off[r.case_variant[j]]:r.v_off[r.case_variant[j] + 1]].tolist()
        assert seq == want


def _invariants(L, log, o, spec):
    A = spec.n_activities
    C = log.info().n_cases
    N = L.n
    cnt = o["cnt"].cpu().numpy()
    sm = o["dur_sum"].cpu().numpy()
    assert int(cnt.sum()) == N - C
    assert int(o["start"].sum()) == C and int(o["end"].sum()) == C
    vt = o["variants"].get()
    assert int(vt["count"].sum()) == C
    assert int(o["n_events"][:C].to(torch.int64).sum()) == N
    assert int(sm.astype(np.int64).sum()) == int(o["dur"][:C].sum())  # telescoping
    mean = o["mean"].cpu().numpy()
    nz = cnt > 0
    assert np.allclose(mean[nz], sm[nz] / cnt[nz], rtol=1e-12, atol=0)


@pytest.mark.parametrize("name", ["100M"])
def test_full_size_sampled_and_invariants(name):
    spec = CONFIGS[name]
    L, log, o = _run(spec, no_ties=False)
    _invariants(L, log, o, spec)
    _sample_check(L, log, o, spec)


def test_1b_single_gpu_with_time_filter():
    """BASELINE.json configs[4] shape (1B events, 50M cases, 256 activities) on one GPU:
    events-mode time filter [T0 + 36.5 d, T0 + 328.5 d], then sort + analyze;
    invariants at full size and sampled cases vs O1 on the filtered rows."""
    from gen.synth import T0_MS
    spec = CONFIGS["1B"]
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs a 180 GB B200")
    L = generate(spec, device="cuda")
    case = L.case.to(torch.uint32)
    act = L.act.to(torch.uint8)
    ts = L.ts
    t1, t2 = T0_MS + int(36.5 * 86_400_000), T0_MS + int(328.5 * 86_400_000)
    log = pm4g.pm4g_log_create(case, act, ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
    f = log.filter_time(t1, t2).sort()
    o = f.analyze()
    keep = (ts >= t1) & (ts <= t2)
    N = int(keep.sum())
    assert f.n == N
    C = f.info().n_cases
    assert int(o["cnt"].sum()) == N - C
    assert int(o["start"].sum()) == C == int(o["variants"].get()["count"].sum())
    assert int(o["n_events"][:C].to(torch.int64).sum()) == N
    # sampled cases vs the oracle on their filtered rows
    rng = np.random.default_rng(1)
    cc = o["case_code"][:C].to(torch.int64)
    pick_idx = np.sort(rng.choice(C, size=500, replace=False))
    pick = cc[torch.as_tensor(pick_idx, device=cc.device)].to(torch.int64)
    sel = keep & torch.isin(L.case, pick)
    r = oracle.run(L.case[sel].cpu().numpy(), L.act[sel].cpu().numpy(), L.ts[sel].cpu().numpy(), spec.n_activities)
    assert np.array_equal(o["n_events"][:C].cpu().numpy()[pick_idx], r.n_events)
    assert np.array_equal(o["dur"][:C].cpu().numpy()[pick_idx], r.dur)


def test_shard_above_2_30_events():
    """A single shard past the former 2^30 - 1 limit (1.2e9 events, 60M cases, 256
    activities): the look-back status words carry 31-bit counts, so every radix
    pass, the format's case ranks and the scans stay exact.  Invariants at full
    size and 1,000 sampled cases vs O1 (logs replicated to scale)."""
    import types
    if torch.cuda.get_device_properties(0).total_memory < 120e9:
        pytest.skip("needs a 180 GB B200")
    spec = CONFIGS["1B"].with_(n_cases=60_000_000, n_events=1_200_000_000)
    assert spec.n_events > (1 << 30)
    G = generate(spec, device="cuda")
    # keep only compact columns (the generator's int64 temporaries would crowd out the sort)
    case = G.case.to(torch.uint32)
    L = types.SimpleNamespace(case=case.view(torch.int32), act=G.act.to(torch.uint8), ts=G.ts, n=G.n)
    del G
    torch.cuda.empty_cache()
    log = pm4g.pm4g_log_create(case, L.act, L.ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
    log.sort()
    o = log.analyze()
    assert log.n == spec.n_events
    _invariants(L, log, o, spec)
    _sample_check(L, log, o, spec, k=1000, seed=3)
