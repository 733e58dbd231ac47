"""One small invocation of every hot-path entry point, for compute-sanitizer
(tests/test_gpu_sanitizer.py runs it under memcheck / racecheck / synccheck).

L1 and the tiny config: validate, lazy + materialised time
filters, sort, sort_analyze with the format fallback, every aggregate, the
variant grouping (one-pass and the general engine), checked against the oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gen.synth import CONFIGS, generate  # noqa: E402
from tests.parity import assert_parity, collect, gpu_run, to_device_cols  # noqa: E402
from paper_2204_04898_b200 import pm4g  # noqa: E402


def main():
    torch.cuda.set_device(0)
    case, act, ts = [0, 1, 2, 0, 1, 2, 0, 2], [0, 0, 0, 1, 2, 1, 2, 2], [0, 5, 0, 10, 15, 50, 20, 100]
    assert_parity(gpu_run(case, act, ts, 3), oracle.run(case, act, ts, 3))
    L = generate(CONFIGS["tiny"])
    c, a, t = L.case.numpy(), L.act.numpy(), L.ts.numpy()
    A = L.n_activities
    assert_parity(gpu_run(c, a, t, A, n_case_codes=L.n_case_codes, sort_analyze=True), oracle.run(c, a, t, A))
    t1, t2 = int(t.min()) + 30 * 86_400_000, int(t.max()) - 30 * 86_400_000
    keep = oracle.filter_time(c, t, t1, t2, oracle.EVENTS)
    for lazy in ("0", "1"):
        os.environ["PM4G_NO_LAZY_FILTER"] = "1" if lazy == "0" else "0"
        dc, da, dt = to_device_cols(c, a, t, A)
        log = pm4g.pm4g_log_create(dc, da, dt, A, n_case_codes=L.n_case_codes)
        f = log.filter_time(t1, t2, pm4g.PM4G_TIME_EVENTS).sort()
        assert_parity(collect(f), oracle.run(c[keep], a[keep], t[keep], A))
        f.close()
        log.close()
    # long cases: the exact format fallback
    rng = np.random.default_rng(7)
    n = 6000
    cc = rng.integers(0, 300, n)
    cc[:2500] = 5
    cc = cc[rng.permutation(n)]
    aa = rng.integers(0, 7, n)
    tt = rng.integers(0, 50, n)
    assert_parity(gpu_run(cc, aa, tt, 7, n_case_codes=300, sort_analyze=True), oracle.run(cc, aa, tt, 7))
    # collisions: the general round-based variant engine
    os.environ["PM4G_DEBUG_WEAK_HASH"] = "1"
    assert_parity(gpu_run(c, a, t, A, n_case_codes=L.n_case_codes), oracle.run(c, a, t, A))
    os.environ["PM4G_DEBUG_WEAK_HASH"] = "0"
    torch.cuda.synchronize()
    # every handle is closed: the library holds no device memory but its reuse cache
    m = pm4g.pm4g_mem_stats()
    assert m["live_blocks"] == 0, f"library blocks still live after every handle closed: {m}"
    pm4g.pm4g_mem_release()
    print("sanitize_run ok", m)


if __name__ == "__main__":
    main()
