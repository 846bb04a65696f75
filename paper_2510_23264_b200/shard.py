"""Item sharding of the scoring pass over ranks (one process per GPU).

A score is a mean over independent prompt items (proj/src/patching.cpp:229-238),
so each rank evaluates every edge on a contiguous block of items, keeps the
per-edge partial sums of the metric (double), and one all-reduce (NCCL inside
libcqg.so, cqg_init_comm) sums them; dividing by the total item count gives
the reference's mean. This module is the host-side statement of that
partition, shared by bench.py and the multi-rank tests.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def item_block(rank: int, world: int, items: int) -> Tuple[int, int]:
    """[lo, hi) of the items owned by `rank` (contiguous, sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return rank * items // world, (rank + 1) * items // world


def partial_sums(shard_means: np.ndarray, shard_items: int) -> np.ndarray:
    """Per-edge sums over a shard from the shard's per-edge means."""
    return np.asarray(shard_means, np.float64) * float(shard_items)


def combine(total_sums: np.ndarray, items: int) -> np.ndarray:
    """Mean over all items from the all-reduced per-edge sums."""
    if items <= 0:
        raise ValueError("empty dataset")
    return np.asarray(total_sums, np.float64) / float(items)
