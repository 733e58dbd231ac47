"""Per-tile phase counters of the radix passes ("What bounds a pass").

    PM4G_NVCC_EXTRA=-DPM4G_OS_PROF python -m paper_2204_04898_b200.build --force
    python tools/osprof.py [config]

Thread 0 of every CTA reads clock64 at the phase boundaries of each tile (rank,
totals + scan + permutation, look-back, write-out) and counts its look-back
round trips; the sums over one sort (all passes) are printed per tile.
Needs a build with PM4G_OS_PROF (the symbol pm4g_debug_osprof exists only then).
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from gen.synth import CONFIGS, generate  # noqa: E402
from paper_2204_04898_b200 import pm4g  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "100M"
spec = CONFIGS[name]
L = generate(spec, device="cuda")
act, case, ts = L.act.to(torch.uint8), L.case.to(torch.uint32), L.ts
fn = pm4g.lib().pm4g_debug_osprof
buf = (ctypes.c_ulonglong * 8)()
for it in range(3):
    log = pm4g.pm4g_log_create(case, act, ts, spec.n_activities, n_case_codes=spec.n_cases, borrow=True)
    fn(buf)
    log.sort()
    torch.cuda.synchronize()
    fn(buf)
    v = list(buf)
    tot = sum(v[:4])
    print("tiles %d, cycles per tile: rank %.0f | totals+scan+permute %.0f | look-back %.0f | write-out %.0f"
          " | fractions %s | look-back round trips per tile %.2f"
          % (v[5], v[0] / v[5], v[1] / v[5], v[2] / v[5], v[3] / v[5], [round(x / tot, 3) for x in v[:4]], v[4] / v[5]))
    log.close()
