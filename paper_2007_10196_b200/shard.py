"""Member sharding across GPUs.

Component grids of a combination family are independent within a step, so the
family shards by member: each rank evolves a subset, all ranks share the
per-step family wave speed (an all-reduce(max) of 5 doubles inside the step
graph, sgwg_evolve) and the combination sum is all-reduced at output times.
Assignment is deterministic LPT (largest member first onto the least-loaded
rank; ties to the lowest rank), members kept in sorted order within a rank so
each rank's partial combination sum follows the reference's member order
(combine.hpp:115-120).
"""
from __future__ import annotations

from typing import List, Sequence


def member_points(levels: Sequence[Sequence[int]], root: Sequence[int], bc: Sequence[int]) -> List[int]:
    """points of each member (GridGeometry::make, grid.hpp:127-128)."""
    out = []
    for lv in levels:
        n = 1
        for k, l in enumerate(lv):
            n *= (root[k] << int(l)) + (1 if bc[k] == 1 else 0)
        out.append(n)
    return out


def lpt_shards(points: Sequence[int], nranks: int) -> List[List[int]]:
    """Deterministic longest-processing-time assignment of member indices."""
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    order = sorted(range(len(points)), key=lambda i: (-points[i], i))
    load = [0] * nranks
    shards: List[List[int]] = [[] for _ in range(nranks)]
    for i in order:
        r = min(range(nranks), key=lambda q: (load[q], q))
        shards[r].append(i)
        load[r] += points[i]
    return [sorted(s) for s in shards]


def shard_balance(points: Sequence[int], shards: Sequence[Sequence[int]]) -> float:
    """max-rank load / mean load (1.0 = perfect)."""
    loads = [sum(points[i] for i in s) for s in shards]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean else 1.0
