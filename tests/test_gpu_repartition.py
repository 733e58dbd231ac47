"""NEXT-4: global repartition by case range and columnar ingest.

The all-to-all is checked on one device through the same data movement the
NCCL path performs: every source slice of an unsorted global table is split by
case range (pm4g_partition_by_case) and each destination concatenates its
pieces in source order (pm4g_log_concat).  Each destination's results must equal
the oracle on the global table restricted to its case range (row order of the
global table: the stable tie-break, R2).  pm4g_repartition itself runs here at
world size 1 (NCCL needs one GPU per rank)."""
import numpy as np
import pytest
import torch

import oracle
from gen.synth import CONFIGS, generate
from tests.parity import assert_parity, collect, to_device_cols
from paper_2204_04898_b200 import pm4g
from paper_2204_04898_b200.dist import shard_ranges, make_comm

pytestmark = pytest.mark.gpu


def _source_logs(case, act, ts, A, ncodes, n_src, extra=None):
    """The global table ingested in n_src contiguous row slices (arbitrary cases each)."""
    cuts = np.linspace(0, case.size, n_src + 1).astype(int)
    logs = []
    for a, b in zip(cuts, cuts[1:]):
        c, ac, t = to_device_cols(case[a:b], act[a:b], ts[a:b], A)
        ex = None
        if extra is not None:
            v, valid = extra
            ex = [pm4g.Extra(kind=pm4g.PM4G_KIND_I64, data=torch.as_tensor(v[a:b]).cuda(),
                             valid=torch.as_tensor(valid[a:b].astype(np.uint8)).cuda())]
        logs.append(pm4g.pm4g_log_create(c, ac, t, A, n_case_codes=ncodes, extra=ex))
    return logs


@pytest.mark.parametrize("name,n_src,R", [("tiny", 3, 2), ("bpic2019", 4, 3), ("roadtraffic", 2, 5)])
def test_partition_concat_equals_oracle(name, n_src, R):
    spec = CONFIGS[name]
    L = generate(spec)
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    rng = np.random.default_rng(R)
    cost = rng.integers(0, 3000, case.size).astype(np.int64)
    valid = rng.random(case.size) > 0.1
    srcs = _source_logs(case, act, ts, A, L.n_case_codes, n_src, extra=(cost, valid))
    ranges = shard_ranges(spec.n_cases, R)
    bounds = [ranges[0][0]] + [hi for _, hi in ranges]
    pieces = [s.partition_by_case(bounds) for s in srcs]
    for r, (lo, hi) in enumerate(ranges):
        dst = pm4g.pm4g_log_concat([p[r] for p in pieces], lo, hi)
        sel = (case >= lo) & (case < hi)
        assert dst.n == int(sel.sum())
        # the extra column travelled with its rows: an event-level range filter on it
        f = dst.filter_attr(0, lo=1001, hi=2500)
        keep = sel & valid & (cost >= 1001) & (cost <= 2500)
        assert_parity(collect(f.sort()), oracle.run(case[keep], act[keep], ts[keep], A))
        assert_parity(collect(dst.sort()), oracle.run(case[sel], act[sel], ts[sel], A))


def test_repartition_world_one_and_errors():
    spec = CONFIGS["tiny"]
    L = generate(spec)
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    c, a, t = to_device_cols(case, act, ts, A)
    log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=spec.n_cases)
    comm = make_comm(0, 1)
    out = log.repartition([0, spec.n_cases], comm)
    assert_parity(collect(out.sort()), oracle.run(case, act, ts, A))
    for bad in ([5, spec.n_cases], [0, 10]):                 # a case outside the bounds
        with pytest.raises(pm4g.Pm4gError) as e:
            log.partition_by_case(bad)
        assert e.value.status == pm4g.PM4G_EINVAL
    with pytest.raises(pm4g.Pm4gError):
        log.sort().partition_by_case([0, spec.n_cases])      # needs an ingested log
    comm.close()


def test_read_parquet_roundtrip(tmp_path):
    """P:75-88 columnar ingest: string ids / activities (first-occurrence codes),
    a timestamp column and nullable extra attributes, vs the oracle on the codes."""
    import pyarrow as pa
    import pyarrow.parquet as pq
    from paper_2204_04898_b200.io import read_parquet
    L = generate(CONFIGS["tiny"])
    case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
    rng = np.random.default_rng(0)
    cost = pa.array([None if rng.random() < 0.2 else int(x) for x in rng.integers(0, 5000, case.size)], pa.int64())
    res = pa.array([f"r{int(x)}" for x in rng.integers(0, 7, case.size)])
    tbl = pa.table({"case:concept:name": pa.array([f"case-{int(x):05d}" for x in case]),
                    "concept:name": pa.array([f"act {int(x)}" for x in act]),
                    "time:timestamp": pa.array(ts, pa.timestamp("ms")),
                    "cost": cost, "org:resource": res})
    p = tmp_path / "log.parquet"
    pq.write_table(tbl, p)
    log, cdict, adict, edicts = read_parquet(str(p), extra=("cost", "org:resource"))
    # expected codes: first-occurrence order of each string column
    def first_occ(xs):
        d = {}
        return np.array([d.setdefault(x, len(d)) for x in xs], dtype=np.int64), list(d)
    ec, ecd = first_occ([f"case-{int(x):05d}" for x in case])
    ea, ead = first_occ([f"act {int(x)}" for x in act])
    assert cdict == ecd and adict == ead
    assert_parity(collect(log.sort()), oracle.run(ec, ea, ts, len(ead)))
    # the nullable extra: nulls never match
    f = log.filter_attr(0, lo=1000, hi=4000, level=pm4g.PM4G_LEVEL_CASES)
    cv = np.array([-1 if v is None else v for v in cost.to_pylist()])
    keep = oracle.filter_attr(ec, cv, lo=1000, hi=4000, valid=(cv >= 0), level=1)
    assert_parity(collect(f.sort()), oracle.run(ec[keep], ea[keep], ts[keep], len(ead)))
