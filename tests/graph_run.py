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
print("graph_run ok")
