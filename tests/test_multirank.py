"""world_size-2 gloo tests of the N > 1 path (CPU): sharding plan, pool
seeding disjointness, no data-path collective, max-over-ranks timing."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, pools, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_1004_3114_b200.sharding import pool_segments, shard

    sh = shard(total, world, rank, 99)
    # this rank's generation (CPU oracle standing in for the rank's GPU)
    vals = O.bank_fill(sh.count, pools, seed=sh.seed, pool_exponent=8, throwaway_f=1,
                       n_arrays=4, dtype=O.F32)
    # timing reduction as bench.py does it: max over ranks
    t = torch.tensor([float(10 + rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # gather for verification only (not part of generation)
    counts = [None] * world
    dist.all_gather_object(counts, (sh.count, sh.offset, sh.seed, vals[:4].tolist(),
                                    pool_segments(sh.count, pools)[-1]))
    if rank == 0:
        q.put((float(t.item()), counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,pools", [(2 * 7 * 300 + 3, 7), (1001, 4)])
def test_two_rank_shards_are_disjoint_and_cover_the_job(total, pools):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, pools, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, info = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == 11.0  # max over ranks
    (c0, o0, s0, v0, seg0), (c1, o1, s1, v1, seg1) = info
    assert c0 + c1 == total and o0 == 0 and o1 == c0
    assert (s0, s1) == (99, 100)  # C4: GPU g seeded 99 + g
    assert v0 != v1
    assert seg0[0] + seg0[1] == c0 and seg1[0] + seg1[1] == c1


def test_shard_plan_matches_c4():
    from paper_1004_3114_b200.sharding import shard

    total = 1 << 36
    for world in (1, 2, 4, 8):
        sh = [shard(total, world, r, 99) for r in range(world)]
        assert sum(s.count for s in sh) == total
        assert len({s.seed for s in sh}) == world
        assert all(s.count == total // world for s in sh)


def test_pool_segments_match_c3_layout():
    from paper_1004_3114_b200.sharding import pool_segments

    seg = pool_segments(1 << 34, 1184)
    assert seg[0] == (0, 14510025) and seg[767][1] == 14510025 and seg[768][1] == 14510024
    assert seg[-1][0] + seg[-1][1] == 1 << 34
    assert np.all(np.diff([s for s, _ in seg]) > 0)
