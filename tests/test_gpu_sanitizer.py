"""compute-sanitizer over the hot path on tests/sanitize_run.py --
L1, the tiny config, both time-filter paths, the format fallback and the general
variant engine:

* memcheck: no out-of-bounds / misaligned access; with every handle closed the
  library holds no live block (sanitize_run checks pm4g_mem_stats) and, its reuse
  cache released, leaks no device memory (counted for allocations made by
  libpm4g only -- the interpreter's own tensors die with the process, and the
  library's per-thread pinned host staging words live for the process);
* synccheck: no barrier reached by part of a block or warp;
* racecheck: no shared-memory hazard other than two documented, benign ones:
  - k_format's slot claim `s_perm[s0 + r] = p`: rows with equal keys (ties)
    claim the same slot on purpose; whichever store lands, the slot holds a row
    of that key, and phase 5 lays the tied rows out in ingest order from the
    key alone;
  - k_aggregate's staged case offsets `st.off[...]`: written by the producer
    warp, read by the consumers after the stage's mbarrier completes (arrive
    with release semantics after __syncwarp; consumers wait with acquire) --
    racecheck does not model mbarrier synchronisation.
"""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = [
    pytest.mark.gpu, pytest.mark.slow,
    # opt-in: the GPU pool this repo is tested on has closed compute-sanitizer
    # (runs under it left GPUs needing a reset), so the default GPU suite skips
    # these; PM4G_SANITIZER=1 runs them where the tool is allowed
    pytest.mark.skipif(os.environ.get("PM4G_SANITIZER") != "1",
                       reason="compute-sanitizer runs are opt-in (PM4G_SANITIZER=1)"),
]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
CSRC = os.path.join(ROOT, "paper_2204_04898_b200", "csrc")

# (source text of the first access, source text of the second access)
BENIGN = [
    ("s_perm[s0 + r] = (uint16_t)p;", "s_perm[s0 + r] = (uint16_t)p;"),
    ("st.off[j] = ", "st.off["),
]


def _run(tool, extra):
    cmd = [SAN, "--tool", tool, "--print-limit", "100000", *extra,
           sys.executable, os.path.join(ROOT, "tests", "sanitize_run.py")]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, env=env, cwd=ROOT)
    out = r.stdout + r.stderr
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert "sanitize_run ok" in out, out[-6000:]
    return out


def _src(loc):
    f, ln = loc.rsplit(":", 1)
    path = os.path.join(CSRC, os.path.basename(f))
    with open(path) as fh:
        return fh.read().splitlines()[int(ln) - 1]


def test_memcheck():
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    out = _run("memcheck", ["--leak-check", "full"])
    assert "Invalid" not in out and "Misaligned" not in out, out[-6000:]
    # device allocations made by libpm4g (its per-thread pinned host staging words,
    # cudaHostAlloc'ed once and kept for the process, are not leaks)
    leaks = [b for b in out.split("========= Leaked")[1:] if "libpm4g.so" in b and "cudaHostAlloc" not in b]
    assert not leaks, "libpm4g allocations leaked:\n" + "\n".join(b[:1500] for b in leaks[:5])


def test_synccheck():
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    out = _run("synccheck", [])
    assert "ERROR SUMMARY: 0 errors" in out, out[-6000:]


def test_racecheck():
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    out = _run("racecheck", ["--racecheck-report", "hazard"])
    bad = []
    for block in out.split("hazard detected")[1:]:
        locs = re.findall(r"(?:Write|Read) Thread \([^)]*\) at .*? in ([a-z_]+\.cuh?:\d+)", block)[:2]
        if len(locs) < 2:
            continue
        a, b = (_src(x).strip() for x in locs)
        if not any((p in a and q in b) or (p in b and q in a) for p, q in BENIGN):
            bad.append((locs, a, b))
    assert not bad, "unexpected shared-memory hazards: " + repr(bad[:10])
