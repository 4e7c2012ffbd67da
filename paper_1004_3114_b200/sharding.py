"""Multi-GPU sharding of the generator.

The work shards into independent, distinctly seeded pools: GPU g of a
C4-style run owns pools UniformState(seed_base + g, c) for c < pools and an
even share of the total count.  There is no collective on the generation
path; torch.distributed is used only to time the job (barrier + max over
ranks of the device time), as bench.py does.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class RankShard:
    rank: int
    world: int
    seed: int          # UniformState seed of this rank's pools
    stream0: int       # pool c uses stream0 + c
    count: int         # normals this rank generates per step
    offset: int        # where this rank's block sits in the job's output


def shard(total: int, world: int, rank: int, seed_base: int, *, seed_per_rank: bool = True
          ) -> RankShard:
    """Split `total` normals over `world` ranks: ranks < total % world take
    one more; rank g seeds its pools with seed_base + g (C4: 99 + g)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    seed = seed_base + rank if seed_per_rank else seed_base
    return RankShard(rank, world, seed, 0, count, offset)


def pool_segments(count: int, pools: int):
    """Pool-major layout of one bank fill (wrng_gpu.h): pool p owns
    [start_p, start_p + len_p), len_p = count // pools + (p < count % pools)."""
    base, extra = divmod(count, pools)
    out, start = [], 0
    for p in range(pools):
        ln = base + (1 if p < extra else 0)
        out.append((start, ln))
        start += ln
    return out
