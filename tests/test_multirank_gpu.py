"""Two ranks on ONE GPU (gloo, both on cuda:0): each rank drives the GPU
library for its C4 shard (pools seeded 99 + rank, an even share of the
total) and its values equal the oracle's bank fill for that seed.  The
ranks never wait on each other's kernels (no collective on the data path);
only the max-over-ranks timing reduction and a barrier use gloo."""
import os
import socket
import sys

import pytest

pytestmark = pytest.mark.gpu

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
    import numpy as np
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import paper_1004_3114_b200 as W
    from paper_1004_3114_b200.sharding import shard

    torch.cuda.set_device(0)
    sh = shard(total, world, rank, 99)
    g = W.WallaceState(W.WallaceConfig(pool_exponent=10, throwaway_f=1, seed=sh.seed,
                                       n_arrays=4, dtype="f32", pools=pools))
    out = torch.empty(sh.count, dtype=torch.float32, device="cuda:0")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    g.fill(out)
    ev1.record()
    torch.cuda.synchronize()
    ref = O.bank_fill(sh.count, pools, seed=sh.seed, pool_exponent=10, throwaway_f=1,
                      n_arrays=4, dtype=O.F32)
    ok = bool(np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32)))
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res = [None] * world
    dist.all_gather_object(res, (rank, sh.seed, sh.count, ok, g.kernel_launches()))
    if rank == 0:
        q.put((float(t.item()), res))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_gpu_drive_the_library_per_shard():
    import torch.multiprocessing as mp

    total, pools = 2 * 37 * 3 * 4095 + 5, 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, pools, q)) for r in range(2)]
    for p in procs:
        p.start()
    tmax, res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax > 0
    (r0, s0, c0, ok0, l0), (r1, s1, c1, ok1, l1) = res
    assert (s0, s1) == (99, 100) and c0 + c1 == total
    assert ok0 and ok1, "a rank's shard differs from the oracle bank fill"
    assert l0 >= 1 and l1 >= 1  # each rank launched the library's kernels
