"""Multi-GPU merge logic on ONE GPU (fake collective).

R case-range shards are processed independently on cuda:0; their packed
integer tables are summed with pm4g_sum_u64 (what C1's NCCL allreduce does) and
their variant tables are merged with pm4g_variants_merge (what C2 does after
its allgather).  The result must equal the oracle on the whole log, bit for bit
-- i.e. the merge is exact and independent of R.
"""
import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from paper_2204_04898_b200 import pm4g
from paper_2204_04898_b200.dist import make_comm, shard_ranges
from tests.parity import assert_parity, collect, to_device_cols

pytestmark = pytest.mark.gpu


def _shard_log(spec, lo, hi):
    L = generate(spec, lo, hi)
    c, a, t = to_device_cols(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    log = pm4g.pm4g_log_create(c, a, t, spec.n_activities, n_case_codes=spec.n_cases, case_lo=lo, case_hi=hi)
    return log.sort()


@pytest.mark.parametrize("name", ["tiny", "bpic2019"])
@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_merge_equals_whole(name, R):
    spec = CONFIGS[name]
    A = spec.n_activities
    L = generate(spec)
    full = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), A)
    logs = [_shard_log(spec, lo, hi) for lo, hi in shard_ranges(spec.n_cases, R)]
    packed = torch.stack([pm4g.pm4g_tables_partial(lg) for lg in logs])
    total = pm4g.pm4g_sum_u64(packed)
    cnt, sm, mean, st, en = pm4g.pm4g_tables_finalize(total, A)
    parts = [lg.variants() for lg in logs]
    merged = pm4g.pm4g_variants_merge(parts)
    v = merged.get()
    torch.cuda.synchronize()
    assert np.array_equal(cnt.cpu().numpy().view(np.uint64), full.cnt)
    assert np.array_equal(sm.cpu().numpy(), full.sum)
    nz = full.cnt > 0
    assert np.allclose(mean.cpu().numpy()[nz], full.mean[nz], rtol=1e-12, atol=0)
    assert np.array_equal(st.cpu().numpy().view(np.uint64), full.start)
    assert np.array_equal(en.cpu().numpy().view(np.uint64), full.end)
    assert np.array_equal(v["count"].cpu().numpy().view(np.uint64), full.v_count)
    assert np.array_equal(v["rep_case"].cpu().numpy(), full.v_rep)
    assert np.array_equal(v["len"].cpu().numpy(), full.v_len)
    assert np.array_equal(v["seq_off"].cpu().numpy().view(np.uint64), full.v_off)
    assert np.array_equal(v["seq_act"].cpu().numpy(), full.v_act)
    # per-case outputs stay sharded; concatenated by rank they are the global cases dataframe
    cc = np.concatenate([lg.case_durations()[0].cpu().numpy() for lg in logs])
    du = np.concatenate([lg.case_durations()[2].cpu().numpy() for lg in logs])
    assert np.array_equal(cc, full.case_code) and np.array_equal(du, full.dur)
    # what each rank gets for its own cases from the NCCL path: the global variant
    # index of every local case (merge with local_part = rank)
    cv = []
    for r, lg in enumerate(logs):
        mr = pm4g.pm4g_variants_merge(parts, local_part=r)
        cv.append(mr.case_index(lg.info().n_cases).cpu().numpy())
        mr.close()
    assert np.array_equal(np.concatenate(cv), full.case_variant)


def test_weak_hash_cross_shard_merge(monkeypatch):
    """Collisions across shards (4-bit keys) are still merged exactly."""
    monkeypatch.setenv("PM4G_DEBUG_WEAK_HASH", "1")
    spec = CONFIGS["tiny"]
    L = generate(spec)
    full = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    logs = [_shard_log(spec, lo, hi) for lo, hi in shard_ranges(spec.n_cases, 3)]
    merged = pm4g.pm4g_variants_merge([lg.variants() for lg in logs])
    assert merged.as_dict() == full.variants()


@pytest.mark.parametrize("env", [("PM4G_DEBUG_NO_COOP", "1"), ("PM4G_DEBUG_VARIANT_CAP", "64")])
def test_merge_one_pass_fallbacks(monkeypatch, env):
    """The merge's one-pass grouping (weighted items, order = representative case)
    through its other exits: the radix ordering when the cooperative grid is
    refused, and the table regrowth after an overflow."""
    monkeypatch.setenv(*env)
    spec = CONFIGS["bpic2019"]
    L = generate(spec)
    full = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    logs = [_shard_log(spec, lo, hi) for lo, hi in shard_ranges(spec.n_cases, 3)]
    parts = [lg.variants() for lg in logs]
    assert pm4g.pm4g_variants_merge(parts).as_dict() == full.variants()
    mr = pm4g.pm4g_variants_merge(parts, local_part=1)
    lo, hi = shard_ranges(spec.n_cases, 3)[1]
    cv = mr.case_index(logs[1].info().n_cases).cpu().numpy()
    sel = (full.case_code >= lo) & (full.case_code < hi)
    assert np.array_equal(cv, full.case_variant[sel])


def test_world_one_communicator_path():
    """comm != NULL with nranks = 1 runs the comm code path (no NCCL) and agrees."""
    spec = CONFIGS["tiny"]
    L = generate(spec)
    c, a, t = to_device_cols(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    log = pm4g.pm4g_log_create(c, a, t, spec.n_activities, n_case_codes=spec.n_cases).sort()
    comm = make_comm(0, 1)
    o = log.analyze(comm=comm)
    v = o["variants"].as_dict()
    full = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    assert v == full.variants()
    ci = o["variants"].case_index(log.info().n_cases).cpu().numpy()
    assert np.array_equal(ci, full.case_variant)
    assert np.array_equal(o["cnt"].cpu().numpy().view(np.uint64).reshape(full.cnt.shape), full.cnt)
    comm.close()
