"""Device-timed measurements of SURVEY.md 8(f)'s NEXT rows on a formatted log
of a BASELINE.json workload (default: the 100M config, one GPU).

    python tools/bench_next.py [--config 100M] [--reps 10]

Times, with CUDA events on the launching stream after warm-up:
  * analyze (DFG + start/end + durations + variants) without / with min/max
    (NEXT-2: the marginal cost of the extremes);
  * pm4g_dfg_minmax alone;
  * every NEXT-1 whole-case filter (START_IN, END_IN, SIZE, THROUGHPUT, PATHS)
    and filter_variants (top-10 variants), output log included;
  * for reference, the A10 case-level time filter on the same formatted log;
  * NEXT-3 efg (eventually-follows graph + temporal profile) with its pair count.
Prints one JSON object per line: {"op", "ms", "events", "G_events_per_s", ...}.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen.synth import CONFIGS, T0_MS, generate  # noqa: E402
from paper_2204_04898_b200 import pm4g  # noqa: E402


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="100M")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    spec = CONFIGS[args.config]
    L = generate(spec, device="cuda")
    act = L.act.to(torch.uint8 if spec.n_activities <= 256 else torch.int16)
    case32 = L.case.to(torch.uint32)
    log = pm4g.pm4g_log_create(case32, act, L.ts, spec.n_activities,
                               n_case_codes=spec.n_cases, borrow=True)
    n = log.n

    def emit(op, ms, **kw):
        print(json.dumps({"op": op, "config": args.config, "ms": round(ms, 4), "events": n,
                          "G_events_per_s": round(n / (ms / 1e3) / 1e9, 3), **kw}), flush=True)

    # NEXT-4 on the ingested log: the 8-way case-range split (an all-to-all's send
    # side) and the concatenation a destination performs; and Parquet ingest
    R = 8
    bounds = [spec.n_cases * r // R for r in range(R + 1)]

    def split():
        for p in log.partition_by_case(bounds):
            p.close()
    emit("partition_by_case 8 ranges (NEXT-4)", timed(split, max(3, args.reps // 2), warm=1))
    parts = log.partition_by_case(bounds)

    def concat():
        pm4g.pm4g_log_concat(parts, 0, spec.n_cases).close()
    emit("log_concat 8 parts (NEXT-4)", timed(concat, max(3, args.reps // 2), warm=1))
    for p in parts:
        p.close()
    try:
        import tempfile
        import time as _t
        import pyarrow as pa
        import pyarrow.parquet as pq
        from paper_2204_04898_b200.io import read_parquet
        m = min(n, 10_000_000)
        tbl = pa.table({"case:concept:name": pa.array(L.case[:m].cpu().numpy()),
                        "concept:name": pa.array(L.act[:m].cpu().numpy()),
                        "time:timestamp": pa.array(L.ts[:m].cpu().numpy(), pa.timestamp("ms"))})
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "log.parquet")
            pq.write_table(tbl, path)
            read_parquet(path)[0].close()
            torch.cuda.synchronize()
            t0 = _t.perf_counter()
            lg = read_parquet(path)[0]
            torch.cuda.synchronize()
            dt = _t.perf_counter() - t0
            lg.close()
        print(json.dumps({"op": "read_parquet -> log (NEXT-4, host wall clock incl. parse + H2D + validate)",
                          "config": args.config, "ms": round(dt * 1e3, 2), "events": m,
                          "M_events_per_s": round(m / dt / 1e6, 1)}), flush=True)
    except ImportError:
        pass

    log.sort()
    torch.cuda.synchronize()

    def analyze(minmax):
        o = log.analyze(minmax=minmax)
        o["variants"].close()

    emit("analyze", timed(lambda: analyze(False), args.reps))
    emit("analyze+minmax", timed(lambda: analyze(True), args.reps))
    emit("dfg_minmax", timed(lambda: log.dfg_minmax(), args.reps))

    # EFG: pairs = sum over cases of m (m - 1) / 2
    C = log.info().n_cases
    cc, ne, du = log.case_durations()
    m = ne[:C].to(torch.int64)
    pairs = int((m * (m - 1) // 2).sum())
    ms = timed(lambda: log.efg(), max(3, args.reps // 2), warm=2)
    emit("efg + temporal profile", ms, pairs=pairs, G_pairs_per_s=round(pairs / (ms / 1e3) / 1e9, 3))

    vt = log.variants()
    d = vt.as_dict()
    vt.close()
    top = sorted(d.items(), key=lambda kv: -kv[1])[:10]
    kept_top = sum(c for _, c in top)
    cases = [
        ("filter_cases START_IN {0,1}", dict(kind=pm4g.PM4G_CASE_START_IN, codes=[0, 1])),
        ("filter_cases END_IN {0,1}", dict(kind=pm4g.PM4G_CASE_END_IN, codes=[0, 1])),
        ("filter_cases SIZE [5,15]", dict(kind=pm4g.PM4G_CASE_SIZE, lo=5, hi=15)),
        ("filter_cases THROUGHPUT [1d,30d]", dict(kind=pm4g.PM4G_CASE_THROUGHPUT, lo=86_400_000, hi=30 * 86_400_000)),
        ("filter_cases PATHS 3 pairs", dict(kind=pm4g.PM4G_CASE_PATHS, codes=[0, 1, 1, 2, 2, 3])),
    ]
    for name, kw in cases:
        kept = [0]

        def run():
            f = log.filter_cases(**kw)
            kept[0] = f.n
            f.close()
        emit(name, timed(run, args.reps), kept_events=kept[0])

    def runv():
        f = log.filter_variants([list(s) for s, _ in top])
        f.close()
    emit("filter_variants top-10", timed(runv, args.reps), kept_cases=kept_top)

    def runt():
        f = log.filter_time(T0_MS + 90 * 86_400_000, T0_MS + 270 * 86_400_000, pm4g.PM4G_TIME_CASES_INTERSECTING)
        f.close()
    emit("filter_time CASES_INTERSECTING (A10, reference)", timed(runt, args.reps))
    log.close()


if __name__ == "__main__":
    main()
