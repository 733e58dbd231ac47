"""Experiment: k_aggregate time by output set at a given config scale (A=256 vs A=64)."""
import sys
import torch
from gen.synth import CONFIGS, generate
from paper_2204_04898_b200 import pm4g

name, scale = sys.argv[1], float(sys.argv[2])
spec = CONFIGS[name]
if scale != 1.0:
    spec = spec.with_(n_cases=int(spec.n_cases * scale), n_events=int(spec.n_events * scale))
L = generate(spec, device="cuda")
act = L.act.to(torch.uint8)
log = pm4g.pm4g_log_create(L.case.to(torch.uint32), act, L.ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
log.sort()
for label, kw in (("all", {}), ("tables", dict(cases=False, variants=False)),
                  ("cases", dict(tables=False, variants=False)), ("variants", dict(tables=False, cases=False))):
    for _ in range(2):
        log.analyze(**kw)
    torch.cuda.synchronize()
    pm4g.pm4g_prof_enable(True); pm4g.pm4g_prof_reset()
    for _ in range(5):
        log.analyze(**kw)
    torch.cuda.synchronize()
    st = pm4g.pm4g_prof_collect()
    pm4g.pm4g_prof_enable(False)
    print(name, scale, label, {k: round(v[1] / v[0], 3) for k, v in st.items() if k == "k_aggregate"}, flush=True)
