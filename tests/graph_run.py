"""pm4g_sort_analyze with PM4G_GRAPH=1 (CUDA-graph segments), repeated so the
executable graphs are instantiated, then updated in place, vs the oracle.
Run by tests/test_gpu_graphs.py in a subprocess (the mode is read once per process)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PM4G_GRAPH"] = "1"

import torch  # noqa: E402

import oracle  # noqa: E402
from gen.synth import CONFIGS, generate  # noqa: E402
from tests.parity import assert_parity, gpu_run  # noqa: E402

torch.cuda.set_stream(torch.cuda.Stream())   # graphs need a capturable (non-default) stream
for name in sys.argv[1:]:
    L = generate(CONFIGS[name])
    c, a, t = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    r = oracle.run(c, a, t, L.n_activities)
    for rep in range(3):
        assert_parity(gpu_run(c, a, t, L.n_activities, n_case_codes=L.n_case_codes, sort_analyze=True), r)
# a case longer than the in-shared-memory ranking takes (the exact fallback runs
# after the graph segments, eagerly) and timestamp ties
import numpy as np  # noqa: E402
rng = np.random.default_rng(3)
n = 60_000
c = rng.integers(0, 4000, n)
c[:5000] = 77
a = rng.integers(0, 9, n)
t = rng.integers(0, 10**6, n)
t[::5] = 123
r = oracle.run(c, a, t, 9)
for rep in range(3):
    assert_parity(gpu_run(c, a, t, 9, n_case_codes=4000, sort_analyze=True), r)
# the lazily filtered log (validation + events-mode time filter in one pass; the
# sort's first pass drops the rows) and a wide-key log (case + ts bits > 64)
from paper_2204_04898_b200 import pm4g  # noqa: E402
from tests.parity import collect, to_device_cols  # noqa: E402
L = generate(CONFIGS["bpic2019"])
c, a, t = L.case.numpy(), L.act.numpy(), L.ts.numpy()
t1, t2 = int(t.min()) + 30 * 86_400_000, int(t.max()) - 30 * 86_400_000
keep = oracle.filter_time(c, t, t1, t2, oracle.EVENTS)
r = oracle.run(c[keep], a[keep], t[keep], L.n_activities)
dc, da, dt = to_device_cols(c, a, t, L.n_activities)
for rep in range(3):
    log = pm4g.pm4g_log_create(dc, da, dt, L.n_activities, n_case_codes=L.n_case_codes, time_filter=(t1, t2))
    assert_parity(collect(log, sort_analyze=True), r)
    log.close()
n = 40_000
c = rng.integers(0, 2**24, n)
t = rng.integers(-(2**60), 2**60, n)
a = rng.integers(0, 7, n)
r = oracle.run(c, a, t, 7)
for rep in range(3):
    assert_parity(gpu_run(c, a, t, 7, n_case_codes=2**24, sort_analyze=True), r)
print("graph_run ok")
