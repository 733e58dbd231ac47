"""pm4g_sort_analyze in CUDA-graph mode (PM4G_GRAPH=1, SURVEY.md 8(d) "small configs
with and without CUDA-graph capture"): every output equals the oracle, on the first
call (graphs instantiated) and on repeated calls (graphs updated in place), for
logs whose variant tables take the single-CTA and the cooperative ordering."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_graph_mode_parity():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "graph_run.py"), "tiny", "roadtraffic", "bpic2019"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert "graph_run ok" in r.stdout, (r.stdout + r.stderr)[-4000:]
