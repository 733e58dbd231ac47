"""Experiment: time each aggregate flavour separately on the 100M workload."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_04898_b200 import pm4g
from bench import make_shard

cfg = sys.argv[1] if len(sys.argv) > 1 else "100M"
case, act, ts, meta, spec = make_shard(cfg, 0, 1, torch.device("cuda"))
log = pm4g.pm4g_log_create(case, act, ts, meta["A"], n_case_codes=meta["n_case_codes"], borrow=True).sort()
C = log.info().n_cases
for name, fn in [("dfg(tables)", lambda: log.dfg()), ("start_end(tables)", lambda: log.start_end()),
                 ("case_durations", lambda: log.case_durations()), ("variants", lambda: log.variants().close())]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    pm4g.pm4g_prof_reset(); pm4g.pm4g_prof_enable(True)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    pm4g.pm4g_prof_enable(False)
    prof = pm4g.pm4g_prof_collect()
    print(name, {k: round(v[1] / 5, 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1])[:6]})
