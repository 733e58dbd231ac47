#!/usr/bin/env python
"""bench.py -- events/s of the PM4Py-GPU hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 100M] [--impl pm4g|reference]

One step = one pass of the hot path over one batch (the config's log shard):
  A0 pm4g_log_create (validate + metadata, columns borrowed in HBM)
  [A1 events-mode time filter, only with --filter: pm4g_log_create_filtered
   validates and filters in one pass; the sort's first radix pass drops the rows]
  A2-A4 pm4g_sort (composite key, onesweep LSD radix sort, case segments)
  A5-A9 pm4g_analyze (fused DFG + start/end + case durations + variant keys,
        then the variant group-count / verify / order)
  A11 with N > 1: NCCL allreduce of the tables + allgather/merge of variants.
Default workload: BASELINE.json configs[3], the synthetic 100M-event log
(10M cases, 64 activities, fully shuffled rows -> full radix sort), one such
shard per GPU (weak scaling: rank r holds case codes [r*10M, (r+1)*10M) of a
global log of N*100M events).  Inputs (1.3 GB/GPU) are larger than L2.

Rank 0 prints ONE JSON line.  `value` = total input events of all ranks / max
over ranks of the device time of the K timed steps (CUDA events around the loop
only; a second K-step loop with an event pair around every kernel gives the
per-kernel table and the roofline, `instrumented_ms_per_step`).  `--graph` runs
pm4g_sort_analyze's segments between its host round trips as CUDA graphs.  `e2e` = the same metric
from HOST buffers (pinned) with a D2H read of every result, inside the timed
region.  For steps of >= 64 MB the H2D copy of step k+1's columns is a torch
copy_ into one of two device column sets on an ingest stream (own host thread),
followed by pm4g_log_create borrowing them, all under step k's compute and D2H;
smaller steps pass the pinned host columns to pm4g_log_create with
PM4G_HOST_INPUT (the copy is then inside the C-ABI call).  `roofline` = the
dominant kernel (k_onesweep, the radix scatter pass) -- algorithmic bytes /
CUDA-event time of its launches in the instrumented loop, against
MEASURED_PEAKS.json hbm_gbs.  `cpu_baseline` = the oracle (single-threaded C++)
timed per stage on the whole config at N = 1 (default), whose every output is
then compared element by element with a GPU step on the same log
(`verified.o1_whole_log_bit_exact`; a line whose outputs are not bit-exact
carries "valid": false).  `--impl reference` times the oracle alone (the
reference arm for this tier).
"""
from __future__ import annotations

import argparse
import concurrent.futures
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

METRIC = "events/sec for sort+DFG+variants at 1/2/4/8 B200; achieved HBM GB/s vs peak"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [x for x in sm if mx and x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workload
def make_shard(cfg: str, rank: int, world: int, device, strong: bool = False):
    """weak: each rank holds a full config-sized shard of a world x larger log;
    strong: the config's log is split across the world by case range (R19)."""
    from gen.synth import CONFIGS
    from gen.synth import generate
    from paper_2204_04898_b200.dist import shard_ranges
    base = CONFIGS[cfg]
    if strong:
        spec = base
        lo, hi = shard_ranges(base.n_cases, world)[rank]
    else:
        spec = base.with_(n_cases=base.n_cases * world,
                          n_events=None if base.n_events is None else base.n_events * world)
        lo, hi = rank * base.n_cases, (rank + 1) * base.n_cases
    L = generate(spec, lo, hi, device=device)
    case = L.case.to(torch.uint32)
    act = L.act.to(L.act_dtype()) if L.act_dtype() != torch.uint8 else L.act.to(torch.uint8)
    ts = L.ts.contiguous()
    meta = dict(n_case_codes=L.n_case_codes, case_lo=lo, case_hi=hi, A=L.n_activities)
    del L
    return case.contiguous(), act.contiguous(), ts, meta, spec


def ingest(pm4g, case, act, ts, meta, host=False, stream=None, filt=None):
    """pm4g_log_create: columns (device, borrowed; or pinned host, copied H2D) -> validated log.
    With filt = (t1, t2): pm4g_log_create_filtered -- the same validation pass also applies the
    events-mode time filter (A1) to the log's metadata; the sort's first pass drops the rows."""
    return pm4g.pm4g_log_create(case, act, ts, meta["A"], n_case_codes=meta["n_case_codes"],
                                case_lo=meta["case_lo"], case_hi=meta["case_hi"], borrow=not host,
                                stream=stream, time_filter=filt)


def run_step(pm4g, case, act, ts, meta, comm, out, filt=None, host=False, trace=None, info=None, log=None):
    tick = (lambda nm: trace.append((nm, time.perf_counter()))) if trace is not None else (lambda nm: None)
    tick("start")
    fused = log is None and filt is not None   # validation + filter in one pass
    if log is None:
        log = ingest(pm4g, case, act, ts, meta, host, filt=filt)
    tick("log_create")
    if filt is not None and not fused:
        f = log.filter_time(filt[0], filt[1], pm4g.PM4G_TIME_EVENTS)
        log.close()
        log = f
        tick("filter_time")
    res = log.sort_analyze(comm=comm, out=out)   # pm4g_sort + pm4g_analyze in one call
    tick("sort+analyze")
    if info is not None:
        i = log.info()
        info.update(n=int(i.n_events), C=int(i.n_cases))
    v = res["variants"]
    log.close()
    tick("close")
    return res, v


def check_invariants(pm4g, case, act, ts, meta, comm, out, filt, dist, dev, keep=None) -> dict:
    """One extra step outside the timed region, its outputs checked against
    identities that hold for any log (S:282, S:332, S:359, S:422, S:206 and the
    telescoping of duration sums): the bench reports whether they held."""
    info = {}
    res, v = run_step(pm4g, case, act, ts, meta, comm, out, filt, info=info)
    n, C = info["n"], info["C"]
    tab = v.get()
    M = 1 << 64
    vals = [n, C, int(res["n_events"][:C].to(torch.int64).sum()), int(res["dur"][:C].sum()) if C else 0]
    if dist:
        g = [None] * dist.get_world_size()
        dist.all_gather_object(g, vals)
        vals = [sum(x[k] for x in g) for k in range(4)]
    N, Ct, ne, dsum = vals
    ok = {
        "sum_dfg_count_eq_events_minus_cases": int(res["cnt"].sum()) == N - Ct,
        "sum_start_eq_cases": int(res["start"].sum()) == Ct,
        "sum_end_eq_cases": int(res["end"].sum()) == Ct,
        "sum_variant_counts_eq_cases": int(tab["count"].sum()) == Ct,
        "sum_case_events_eq_events": ne == N,
        "sum_dfg_durations_eq_sum_case_durations": int(res["dur_sum"].sum()) % M == dsum % M,
    }
    if keep is not None:   # every output of this step on the host, for the O1 comparison
        import numpy as np
        A = meta["A"]
        keep.update(cnt=res["cnt"].cpu().numpy().view(np.uint64).reshape(A, A),
                    sum=res["dur_sum"].cpu().numpy().reshape(A, A), mean=res["mean"].cpu().numpy().reshape(A, A),
                    start=res["start"].cpu().numpy().view(np.uint64), end=res["end"].cpu().numpy().view(np.uint64),
                    case_code=res["case_code"][:C].cpu().numpy(), n_events=res["n_events"][:C].cpu().numpy(),
                    dur=res["dur"][:C].cpu().numpy(), v_count=tab["count"].cpu().numpy().view(np.uint64),
                    v_len=tab["len"].cpu().numpy(), v_rep=tab["rep_case"].cpu().numpy(),
                    v_off=tab["seq_off"].cpu().numpy().view(np.uint64), v_act=tab["seq_act"].cpu().numpy(),
                    case_variant=v.case_index(C).cpu().numpy())
    v.close()
    return {"all": all(ok.values()), **ok}


def workload_config(cfg: str, n_local: int, cases: int, A: int, world: int, filt: bool,
                    n_total: int | None = None) -> dict:
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": f"synthetic-{cfg}: {n_local:,} events / {cases:,} cases / {A} activities per GPU, "
                        f"fully shuffled rows (full radix sort)" + (", events-mode time filter" if filt else ""),
            "events_per_gpu": n_local, "global_events": n_total if n_total is not None else n_local * world,
            "parallelism": f"case-sharded x{world}",
            "l2": "inputs (13 B/event) larger than L2; no flush needed",
            "step": "log_create+sort+analyze(DFG,start/end,durations,variants)" + ("+filter" if filt else "")}


def cpu_baseline(cfg, cases: int, device, gpu_out=None):
    """O1 (single-threaded C++) on the first `cases` cases of the workload, timed
    per stage (stable sort, then the loop).  With the whole config (cases >=
    n_cases, the default at N = 1) and gpu_out (every output of a GPU step on
    the same log), every output is compared element by element: SURVEY.md 8(d)
    "each reported number is checked against O1 first"."""
    import numpy as np
    import oracle
    from gen.synth import CONFIGS, generate
    spec = CONFIGS[cfg]
    k = min(cases, spec.n_cases)
    L = generate(spec, 0, k, device=device)
    c, a, t = L.case.cpu().numpy(), L.act.cpu().numpy(), L.ts.cpu().numpy()
    del L
    oracle.build()
    t0 = time.perf_counter()
    r = oracle.run(c, a, t, spec.n_activities)
    dt = time.perf_counter() - t0
    whole = k == spec.n_cases
    out = {"value": c.size / dt, "unit": "events/s", "cores": 1, "kind": "oracle",
           "sample": (f"the whole {cfg} workload" if whole else f"first {k:,} cases of the {cfg} workload") +
                     f" ({c.size:,} events); single-threaded O1, {dt:.2f} s (stable sort {r.t_sort:.2f} s, "
                     f"loop {r.t_loop:.2f} s)",
           "stage_s": {"sort": round(r.t_sort, 3), "loop": round(r.t_loop, 3), "total": round(dt, 3)}}
    if gpu_out:
        g = gpu_out
        if whole:
            checks = {
                "dfg_count": np.array_equal(g["cnt"], r.cnt), "dfg_sum": np.array_equal(g["sum"], r.sum),
                "dfg_mean": np.array_equal(g["mean"], r.mean),
                "start": np.array_equal(g["start"], r.start), "end": np.array_equal(g["end"], r.end),
                "case_code": np.array_equal(g["case_code"], r.case_code),
                "n_events": np.array_equal(g["n_events"], r.n_events), "dur": np.array_equal(g["dur"], r.dur),
                "variant_count": np.array_equal(g["v_count"], r.v_count),
                "variant_len": np.array_equal(g["v_len"], r.v_len),
                "variant_rep": np.array_equal(g["v_rep"], r.v_rep),
                "variant_off": np.array_equal(g["v_off"], r.v_off),
                "variant_seq": np.array_equal(g["v_act"], r.v_act),
                "case_variant": np.array_equal(g["case_variant"], r.case_variant)}
            out["o1_whole_log_bit_exact"] = {"all": all(checks.values()), **checks}
        else:
            out["per_case_parity_on_sample"] = bool(np.array_equal(g["n_events"][:k], r.n_events) and
                                                    np.array_equal(g["dur"][:k], r.dur))
    return out


# ------------------------------------------------------------------ reference arm
def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from gen.synth import CONFIGS, generate
    spec = CONFIGS[args.config]
    cases = args.ref_cases
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    L = generate(spec, 0, min(cases, spec.n_cases), device=dev)
    c, a, t = L.case.cpu().numpy(), L.act.cpu().numpy(), L.ts.cpu().numpy()
    oracle.build()
    for _ in range(args.warmup):
        oracle.run(c, a, t, spec.n_activities)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run(c, a, t, spec.n_activities)
    dt = time.perf_counter() - t0
    v = c.size * args.steps / dt
    full_n = spec.n_events if spec.n_events is not None else int(c.size)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "events/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": workload_config(args.config, full_n, spec.n_cases, spec.n_activities, 1, args.filter),
            "cpu_baseline": {"value": v, "unit": "events/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {min(cases, spec.n_cases):,} cases ({c.size:,} events) of "
                                       f"the {args.config} workload per step; single-threaded O1"},
            "e2e": {"value": v, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="100M")
    ap.add_argument("--impl", default="pm4g", choices=["pm4g", "reference"])
    ap.add_argument("--filter", action="store_true", help="events-mode time filter in the step (1B-style)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--cpu-cases", type=int, default=0,
                    help="oracle sample: the first K cases (default 0 = the whole config, compared element by "
                         "element with a GPU step)")
    ap.add_argument("--ref-cases", type=int, default=50_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stages", action="store_true", help="print the per-kernel table to stderr")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="weak: a config-sized shard per GPU (default); strong: the config's log split across "
                         "the GPUs (default for the 1B config, the north-star layout)")
    ap.add_argument("--emulate", default=None, metavar="R/N",
                    help="one GPU runs rank R's shard of an N-way split (per-GPU time of an N-GPU run, "
                         "without the NCCL merge)")
    ap.add_argument("--graph", action="store_true",
                    help="run pm4g_sort_analyze's segments between its host round trips as CUDA graphs "
                         "(PM4G_GRAPH=1; the per-kernel events become event-record nodes)")
    args = ap.parse_args()
    if args.graph:
        os.environ["PM4G_GRAPH"] = "1"   # read by libpm4g at its first sort_analyze
    if args.impl == "reference":
        return reference_arm(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.graph:   # the legacy default stream cannot be captured: run the steps on a stream of their own
        torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_2204_04898_b200 import pm4g
    comm = None
    if world > 1:
        uid = [pm4g.pm4g_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = pm4g.pm4g_comm_create(uid[0], world, rank)

    scaling = args.scaling or ("strong" if args.config == "1B" else "weak")
    shard_rank, shard_world = rank, world
    if args.emulate:
        if world != 1:
            raise SystemExit("--emulate runs on one process")
        shard_rank, shard_world = (int(x) for x in args.emulate.split("/"))
    case, act, ts, meta, spec = make_shard(args.config, shard_rank, shard_world, dev, strong=scaling == "strong")
    n_local = int(case.numel())
    filt = None
    if args.filter:
        from gen.synth import T0_MS
        filt = (T0_MS + int(36.5 * 86_400_000), T0_MS + int(328.5 * 86_400_000))
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    out = {}
    for _ in range(args.warmup):
        _, v = run_step(pm4g, case, act, ts, meta, comm, out, filt)
        v.close()
    torch.cuda.synchronize()

    # ---------------- timed region (device time, CUDA events on the launching stream)
    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.2)
    # K steps timed with events around the whole loop only (value, ms_per_step);
    # then K more with an event pair around every kernel (the per-kernel table and
    # the roofline): those events cost GPU and host time of their own (~30% of a
    # tiny step), so they stay out of the headline timing
    l0 = pm4g.pm4g_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        _, v = run_step(pm4g, case, act, ts, meta, comm, out, filt)
        v.close()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = pm4g.pm4g_launch_count() - l0
    pm4g.pm4g_prof_reset()
    pm4g.pm4g_prof_enable(True)
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    trace = []
    for i in range(args.steps):
        _, v = run_step(pm4g, case, act, ts, meta, comm, out, filt,
                        trace=trace if (args.stages and i == args.steps - 1) else None)
        v.close()
    i1.record(stream)
    torch.cuda.synchronize()
    pm4g.pm4g_prof_enable(False)
    prof = pm4g.pm4g_prof_collect()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    ms_instr = i0.elapsed_time(i1)
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    n_total = n_local
    if dist:   # shards hold about, not exactly, the same number of events
        t = torch.tensor([n_local], device=dev, dtype=torch.int64)
        dist.all_reduce(t)
        n_total = int(t.item())
    value = n_total * args.steps / (ms / 1e3)

    # ---------------- end to end through the C-ABI with host buffers
    e2e = None
    if args.e2e_steps > 0:
        hc, ha, ht = case.cpu().pin_memory(), act.cpu().pin_memory(), ts.cpu().pin_memory()
        torch.cuda.synchronize()
        d2h = 0
        hosts = {}

        # Ingest of step k+1 -- the H2D copy of its columns from pinned memory into one of two
        # device column sets, then pm4g_log_create (validation) on them -- runs on its own
        # stream and host thread while step k sorts / analyses / copies its results back: the
        # copy engine, not the SMs, bounds this path (PCIe, 13 B/event in).  A column set is
        # refilled only after the step that read it has drained (event on the compute stream).
        ing_stream = torch.cuda.Stream(device=dev)
        pool = concurrent.futures.ThreadPoolExecutor(1, initializer=torch.cuda.set_device, initargs=(dev,))
        pending = []
        pipelined = n_local * 13 >= (64 << 20)
        dcols = [tuple(torch.empty_like(x, device=dev) for x in (hc, ha, ht)) for _ in range(2 if pipelined else 0)]
        drained = [None, None]
        n_ingest = [0]

        def ingest_async():
            slot = n_ingest[0] % 2
            n_ingest[0] += 1
            wait = drained[slot]

            def work():
                with torch.cuda.stream(ing_stream):
                    if wait is not None:
                        ing_stream.wait_event(wait)
                    for d, h in zip(dcols[slot], (hc, ha, ht)):
                        d.copy_(h, non_blocking=True)
                    return slot, ingest(pm4g, *dcols[slot], meta, False, ing_stream, filt=filt)
            if pipelined:
                pending.append(pool.submit(work))
            else:   # small steps: pm4g_log_create copies the pinned host columns itself
                f = concurrent.futures.Future()
                f.set_result((slot, ingest(pm4g, hc, ha, ht, meta, True, filt=filt)))
                pending.append(f)

        def e2e_step(prefetch):
            nonlocal d2h
            slot, log = pending.pop(0).result()
            if prefetch:
                ingest_async()
            res, v = run_step(pm4g, None, None, None, meta, comm, out, None, log=log)   # (filtered at ingest)
            drained[slot] = torch.cuda.Event()
            drained[slot].record(stream)
            tabs = v.get()
            d2h = 0
            for k in ("cnt", "dur_sum", "mean", "start", "end", "case_code", "n_events", "dur"):
                x = res[k]
                if k not in hosts or hosts[k].numel() != x.numel():
                    hosts[k] = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
                hosts[k].copy_(x, non_blocking=True)
                d2h += x.numel() * x.element_size()
            for k, x in tabs.items():   # pinned buffers kept across steps (no host allocation in the loop)
                hk = "v_" + k
                if hk not in hosts or hosts[hk].dtype != x.dtype or hosts[hk].numel() < x.numel():
                    hosts[hk] = torch.empty(max(1, 2 * x.numel()), dtype=x.dtype, pin_memory=True)
                hosts[hk][: x.numel()].copy_(x.reshape(-1), non_blocking=True)
                d2h += x.numel() * x.element_size()
            v.close()

        ingest_async()
        e2e_step(False)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        ing_stream.wait_event(f0)
        ingest_async()
        for k in range(args.e2e_steps):
            e2e_step(k + 1 < args.e2e_steps)
        f1.record(stream)
        torch.cuda.synchronize()
        pool.shutdown()
        ems = f0.elapsed_time(f1)
        if dist:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n_total * args.e2e_steps / (ems / 1e3), "unit": "events/s",
               "h2d_bytes_per_step": n_local * (4 + act.element_size() + 8), "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / args.e2e_steps,
               "overlap": ("double-buffered: step k+1's H2D + validation (own stream and host thread) "
                           "runs under step k's sort/analyze and D2H") if pipelined else "none (small step)"}

    # ---------------- roofline of the dominant kernel
    peak, peak_src = _peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roof = None
    if "k_onesweep" in prof:
        la, kms, kbytes = prof["k_onesweep"]
        achieved = kbytes / (kms / 1e3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                tj = json.load(open(tf))
                ent = tj.get("k_onesweep")
                if ent and ent.get("config") == args.config:
                    traffic = ent["dram_bytes_per_launch"]
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "kernel": "k_onesweep", "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": kbytes / la, "launches": la,
                "avg_launch_ms": kms / la, "share_of_step": round(kms / ms_instr, 4), "peak_source": peak_src,
                "measured_in": "a second K-step loop with an event pair around every kernel"}
    step_bytes = sum(b for (_, _, b) in prof.values())
    stages = {k: {"launches": la, "ms": round(m, 3), "GB/s": round(b / (m / 1e3) / 1e9, 1) if m > 0 else None}
              for k, (la, m, b) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    if args.stages and rank == 0:
        for k, s in stages.items():
            print(f"{k:28s} {s}", file=sys.stderr)
        if trace:
            print("host trace of the last step (ms since step start):", file=sys.stderr)
            for nm, tt in trace:
                print(f"  {1e3 * (tt - trace[0][1]):9.3f}  {nm}", file=sys.stderr)
        recs = pm4g.pm4g_prof_records()
        per = len(recs) // max(1, args.steps)
        last = recs[-per:] if per else []
        if last:
            t00, prev_end = last[0][1], last[0][1]
            print("timeline of the last timed step (start ms, gap before, duration ms):", file=sys.stderr)
            for nm, t0, d in last:
                print(f"  {t0 - t00:9.3f} gap {t0 - prev_end:8.3f}  {d:8.3f}  {nm}", file=sys.stderr)
                prev_end = t0 + d

    # the oracle sees cases [0, k) of the config: comparable with this rank's outputs
    # when the rank holds the config from case 0 and no filter runs
    comparable = (rank == 0 and not args.no_cpu_baseline and filt is None and meta["case_lo"] == 0
                  and world == 1 and shard_world == 1)
    kept = {} if comparable else None
    verified = check_invariants(pm4g, case, act, ts, meta, comm, out, filt, dist, dev, kept)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        del case, act, ts
        torch.cuda.empty_cache()
        cpu = cpu_baseline(args.config, args.cpu_cases or 1 << 62, dev, kept)
        if "o1_whole_log_bit_exact" in cpu:
            verified["o1_whole_log_bit_exact"] = cpu["o1_whole_log_bit_exact"]["all"]
            verified["all"] = verified["all"] and verified["o1_whole_log_bit_exact"]
        if not verified["all"]:
            print("bench: outputs NOT verified (see 'verified'); the line is flagged invalid", file=sys.stderr)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "instrumented_ms_per_step": ms_instr / args.steps,
            "scaling": scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": workload_config(args.config, n_local, meta["case_hi"] - meta["case_lo"], meta["A"], world,
                                      filt is not None, n_total),
            "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof, "verified": verified,
            "cpu_baseline": cpu, "valid": bool(verified["all"]),
            "hbm_pipeline": {"algorithmic_GB_per_step": step_bytes / args.steps / 1e9,
                             "achieved_GB_per_s": step_bytes / (ms / 1e3) / 1e9,
                             "frac_of_peak": step_bytes / (ms / 1e3) / 1e9 / peak},
            "stages": stages,
        }
        line["config"]["scaling_layout"] = (f"{scaling}: " + ("the config's log split across the GPUs by case range"
                                                       if scaling == "strong" else "one config-sized shard per GPU"))
        if args.emulate:
            line["config"]["emulated_shard"] = (f"rank {shard_rank} of {shard_world} on one GPU "
                                                "(per-GPU step of that run, without the NCCL merge)")
        if args.graph:
            line["config"]["cuda_graphs"] = ("pm4g_sort_analyze's launches between its host round trips "
                                             "captured and replayed as CUDA graphs (PM4G_GRAPH=1)")
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
