"""R ranks as threads of one process on cuda:0 through libpm4g's NCCL code path,
with PM4G_NCCL_LIB pointing at the loopback NCCL (tests/fake_nccl).  Each rank
checks, against the oracle on the whole log: the allreduced DFG / start-end and
min / max tables, the allgathered + merged variant table, its cases' global
variant index, the EFG, and a repartition of row slices into case ranges.
Prints "OK R" or raises."""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_2204_04898_b200 import pm4g  # noqa: E402
from paper_2204_04898_b200.dist import shard_ranges  # noqa: E402
from tests.parity import to_device_cols  # noqa: E402


def u64(t):
    return t.contiguous().view(-1).cpu().numpy().view(np.uint64)


def rank_main(r, R, uid, name, errs):
    try:
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            comm = pm4g.pm4g_comm_create(uid, R, r)
            spec = CONFIGS[name]
            L = generate(spec)
            case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
            full = oracle.run(case, act, ts, A)
            lo, hi = shard_ranges(spec.n_cases, R)[r]
            sel = (case >= lo) & (case < hi)
            c, a, t = to_device_cols(case[sel], act[sel], ts[sel], A)
            log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=spec.n_cases, case_lo=lo, case_hi=hi).sort()
            o = log.analyze(comm=comm, minmax=True)
            st.synchronize()
            assert np.array_equal(u64(o["cnt"]).reshape(A, A), full.cnt), "C1 counts"
            assert np.array_equal(o["dur_sum"].cpu().numpy().reshape(A, A), full.sum), "C1 sums"
            assert np.array_equal(u64(o["start"]), full.start) and np.array_equal(u64(o["end"]), full.end)
            mn, mx = oracle.dfg_minmax(case, act, ts, A)
            assert np.array_equal(u64(o["dur_min"]), mn.reshape(-1)) and np.array_equal(u64(o["dur_max"]), mx.reshape(-1))
            vt = o["variants"].get()
            st.synchronize()
            assert np.array_equal(u64(vt["count"]), full.v_count), "C2 counts"
            assert np.array_equal(vt["rep_case"].cpu().numpy(), full.v_rep), "C2 reps"
            assert np.array_equal(vt["seq_act"].cpu().numpy(), full.v_act), "C2 sequences"
            ci = o["variants"].case_index(log.info().n_cases).cpu().numpy()
            mine = np.isin(full.case_code, np.unique(case[sel]))
            assert np.array_equal(ci, full.case_variant[mine]), "per-case global variant index"
            e = log.efg(comm=comm)
            re = oracle.efg(case, act, ts, A)
            st.synchronize()
            for kg, kr in (("cnt", "cnt"), ("sum", "sum"), ("sumsq_lo", "sq_lo"), ("sumsq_hi", "sq_hi")):
                assert np.array_equal(u64(e[kg]), re[kr].reshape(-1)), "EFG " + kg
            # repartition: rank r ingests row slice r of the table, receives its case range
            cuts = np.linspace(0, case.size, R + 1).astype(int)
            rs = slice(cuts[r], cuts[r + 1])
            c2, a2, t2 = to_device_cols(case[rs], act[rs], ts[rs], A)
            src = pm4g.pm4g_log_create(c2, a2, t2, A, n_case_codes=spec.n_cases)
            bounds = [b[0] for b in shard_ranges(spec.n_cases, R)] + [spec.n_cases]
            got = src.repartition(bounds, comm)
            assert got.n == int(sel.sum()), "repartition row count"
            o2 = got.sort().analyze(comm=None, variants=False)
            part = oracle.run(case[sel], act[sel], ts[sel], A)
            st.synchronize()
            assert np.array_equal(u64(o2["cnt"]).reshape(A, A), part.cnt), "repartition content"
            assert np.array_equal(o2["case_code"][:part.n_cases].cpu().numpy(), part.case_code)
            comm.close()
    except BaseException as ex:  # noqa: BLE001
        errs.append(f"rank {r}: {type(ex).__name__}: {ex}")


def main():
    R = int(sys.argv[1])
    name = sys.argv[2] if len(sys.argv) > 2 else "tiny"
    uid = pm4g.pm4g_comm_unique_id()
    errs = []
    th = [threading.Thread(target=rank_main, args=(r, R, uid, name, errs)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs or any(t.is_alive() for t in th):
        print("FAILED", errs, flush=True)
        return 1
    print(f"OK {R}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
