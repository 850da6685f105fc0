"""Summand sharding of the multi-GPU path: contiguous blocks of
summands per rank, sizes differing by at most one (equal-rank configs)."""


def shard_bounds(S: int, world: int, rank: int):
    """[lo, hi) of the summands rank `rank` of `world` holds."""
    if not (0 <= rank < world) or S < 1:
        raise ValueError("bad shard request")
    return (rank * S) // world, ((rank + 1) * S) // world
