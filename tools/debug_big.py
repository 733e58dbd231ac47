"""Debug helper: run sort+analyze on a (scaled) config, optionally time-filtered, report the failing stage."""
import sys, time
import torch
from gen.synth import CONFIGS, generate, T0_MS
from paper_2204_04898_b200 import pm4g

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
filt = len(sys.argv) > 3 and sys.argv[3] == "filter"
spec = CONFIGS[name]
if scale != 1.0:
    spec = spec.with_(n_cases=int(spec.n_cases * scale), n_events=int(spec.n_events * scale))
L = generate(spec, device="cuda")
act = L.act.to(torch.uint8 if spec.n_activities <= 256 else torch.int16)
log = pm4g.pm4g_log_create(L.case.to(torch.uint32), act, L.ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
if filt:
    t1, t2 = T0_MS + int(36.5 * 86_400_000), T0_MS + int(328.5 * 86_400_000)
    log = log.filter_time(t1, t2)
    torch.cuda.synchronize(); print("filter ok", log.n, flush=True)
log.sort(); torch.cuda.synchronize(); print("sort ok", flush=True)
for step in ("dfg", "start_end", "case_durations", "variants"):
    getattr(log, step)(); torch.cuda.synchronize(); print(step, "ok", flush=True)
o = log.analyze(); torch.cuda.synchronize(); print("analyze ok", o["variants"].size(), flush=True)
