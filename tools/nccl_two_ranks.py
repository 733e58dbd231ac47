"""N ranks through the real NCCL path: one GPU per rank (LOCAL_RANK), or all on
one GPU where NCCL allows it (NCCL 2.28 refuses duplicate devices: "invalid
usage", reported as PM4G_ENCCL -- then the script only checks that).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_two_ranks.py

Each rank holds a case-range shard of the tiny / bpic2019 workload; analyze()
with a 2-rank pm4g communicator must reproduce the oracle on the whole log
(C1 allreduce, C2 allgather + merge, per-case global variant index), and
repartition() of row slices must reproduce each rank's case range.  The
bootstrap (unique id) goes over gloo.  Prints one line per rank.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_2204_04898_b200 import pm4g  # noqa: E402
from paper_2204_04898_b200.dist import shard_ranges  # noqa: E402
from tests.parity import to_device_cols  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count())
    uid = [pm4g.pm4g_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    try:
        comm = pm4g.pm4g_comm_create(uid[0], world, rank)
    except pm4g.Pm4gError as e:
        print(f"rank {rank}: NCCL communicator refused: {e}", flush=True)
        return 0
    ok = True
    for name in ("tiny", "bpic2019"):
        spec = CONFIGS[name]
        L = generate(spec)
        case, act, ts, A = L.case.numpy(), L.act.numpy(), L.ts.numpy(), L.n_activities
        lo, hi = shard_ranges(spec.n_cases, world)[rank]
        sel = (case >= lo) & (case < hi)
        c, a, t = to_device_cols(case[sel], act[sel], ts[sel], A)
        log = pm4g.pm4g_log_create(c, a, t, A, n_case_codes=spec.n_cases, case_lo=lo, case_hi=hi).sort()
        o = log.analyze(comm=comm)
        full = oracle.run(case, act, ts, A)
        torch.cuda.synchronize()
        ok &= np.array_equal(o["cnt"].cpu().numpy().view(np.uint64).reshape(A, A), full.cnt)
        ok &= np.array_equal(o["dur_sum"].cpu().numpy().reshape(A, A), full.sum)
        ok &= o["variants"].as_dict() == full.variants()
        mine = oracle.run(case[sel], act[sel], ts[sel], A)
        ci = o["variants"].case_index(log.info().n_cases).cpu().numpy()
        ok &= np.array_equal(ci, full.case_variant[np.isin(full.case_code, mine.case_code)])
        # repartition: rank r ingests rows [r/world, (r+1)/world) of the table, receives its case range
        cuts = np.linspace(0, case.size, world + 1).astype(int)
        rs = slice(cuts[rank], cuts[rank + 1])
        c2, a2, t2 = to_device_cols(case[rs], act[rs], ts[rs], A)
        src = pm4g.pm4g_log_create(c2, a2, t2, A, n_case_codes=spec.n_cases)
        bounds = [r[0] for r in shard_ranges(spec.n_cases, world)] + [spec.n_cases]
        mine2 = src.repartition(bounds, comm).sort()
        o2 = mine2.analyze(variants=False)
        torch.cuda.synchronize()
        ok &= np.array_equal(o2["cnt"].cpu().numpy().view(np.uint64).reshape(A, A), mine.cnt)
        ok &= mine2.n == int(sel.sum())
    print(f"rank {rank}: two-rank NCCL parity {'OK' if ok else 'FAILED'}", flush=True)
    comm.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
