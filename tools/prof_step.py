"""One filter + sort + analyze on a (scaled) config, for ncu captures."""
import sys
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
act = L.act.to(torch.uint8)
case = L.case.to(torch.uint32)
ts = L.ts
torch.cuda.synchronize()
log = pm4g.pm4g_log_create(case, act, ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
if filt:
    log = log.filter_time(T0_MS + int(36.5 * 86_400_000), T0_MS + int(328.5 * 86_400_000))
log.sort()
o = log.analyze()
torch.cuda.synchronize()
print("ok", log.n)
