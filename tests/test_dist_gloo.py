"""N > 1 host logic on CPU with torch.distributed/gloo, world_size 2 (no GPU).

Covers what the multi-GPU path does on the host: the case-range sharding
(S:228-231), shard-independent generation, the unique-id bootstrap, and the
merge algebra the NCCL collectives implement (integer tables are
summed, variant tables are unioned with summed counts and min representative).
The per-shard results here come from the oracle, so the test pins that
sharding + merge reproduces the single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_04898_b200.dist import broadcast_unique_id, shard_range, shard_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from gen.synth import CONFIGS, generate
        spec = CONFIGS[cfg]
        lo, hi = shard_range(spec.n_cases, rank, world)
        L = generate(spec, lo, hi)
        r = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
        A = spec.n_activities
        # C1: one allreduce of the packed integer table [cnt | sum | start | end]
        packed = torch.from_numpy(np.concatenate([r.cnt.view(np.int64).ravel(), r.sum.ravel(),
                                                  r.start.view(np.int64), r.end.view(np.int64)]))
        dist.all_reduce(packed)
        # C2: allgather of the per-shard variant tables, merged by sequence
        mine = [(tuple(r.v_act[r.v_off[i]:r.v_off[i + 1]].tolist()), int(r.v_count[i]), int(r.v_rep[i]))
                for i in range(r.v_count.size)]
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        merged = {}
        for part in allv:
            for seq, c, rep in part:
                oc, orep = merged.get(seq, (0, 1 << 62))
                merged[seq] = (oc + c, min(orep, rep))
        # bootstrap: rank 0's opaque id reaches every rank unchanged
        uid = broadcast_unique_id(b"pm4g-uid-%d" % port if rank == 0 else None, rank)
        per_case = (r.case_code.min() if r.n_cases else -1, r.case_code.max() if r.n_cases else -1, r.n_cases)
        q.put((rank, packed.numpy(), merged, uid, per_case, (lo, hi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["tiny"])
def test_two_rank_shard_and_merge_equals_single(cfg):
    import oracle
    from gen.synth import CONFIGS, generate
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = CONFIGS[cfg]
    L = generate(spec)
    full = oracle.run(L.case.numpy(), L.act.numpy(), L.ts.numpy(), spec.n_activities)
    A = spec.n_activities
    want = np.concatenate([full.cnt.view(np.int64).ravel(), full.sum.ravel(),
                           full.start.view(np.int64), full.end.view(np.int64)])
    for rank, packed, merged, uid, per_case, rng in res:
        assert np.array_equal(packed, want)                       # allreduce result on every rank
        wantv = {tuple(full.v_act[full.v_off[i]:full.v_off[i + 1]].tolist()): (int(full.v_count[i]), int(full.v_rep[i]))
                 for i in range(full.v_count.size)}
        assert merged == wantv                                    # allgather + merge result
        assert uid == b"pm4g-uid-%d" % port
    # shards are disjoint, ordered, cover every case
    (_, _, _, _, pc0, r0), (_, _, _, _, pc1, r1) = res
    assert r0[1] == r1[0] and r0[0] == 0 and r1[1] == spec.n_cases
    assert pc0[2] + pc1[2] == full.n_cases and pc0[1] < pc1[0]


def test_shard_ranges_partition():
    for C in (0, 1, 7, 150_370, 10_000_000):
        for R in (1, 2, 3, 4, 8):
            rs = shard_ranges(C, R)
            assert rs[0][0] == 0 and rs[-1][1] == C
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_generator_is_shard_independent():
    """The union of the shards is the log (same rows, per-case identical), for any R."""
    from gen.synth import CONFIGS, generate
    spec = CONFIGS["tiny"]
    L = generate(spec)
    key = lambda c, a, t: sorted(zip(c.tolist(), a.tolist(), t.tolist()))  # noqa: E731
    whole = key(L.case, L.act, L.ts)
    for R in (2, 3, 4):
        parts = [generate(spec, lo, hi) for lo, hi in shard_ranges(spec.n_cases, R)]
        got = key(torch.cat([p.case for p in parts]), torch.cat([p.act for p in parts]),
                  torch.cat([p.ts for p in parts]))
        assert got == whole
