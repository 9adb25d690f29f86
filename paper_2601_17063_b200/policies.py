"""Policy-level types of the drop-in surface (pkg/src/moecache/policies.py:20-48).

The B200 engine evaluates every policy (LRU, LFU, Belady, ML, FIFO, ARC,
LeCaR) inside its replay kernels; per-access ``CachePolicy`` objects are not
provided.  Victim rules are implemented in
csrc/mcb_kernels.cu (k_replay) as argmin of (key, expert id) over
resident \\ pinned.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional


class PolicyError(Exception):
    pass


class NoEvictableError(PolicyError):
    """Every resident expert is pinned (or unscorable); no victim can be chosen."""


@dataclass(frozen=True)
class PolicyDecision:
    loaded: int
    was_hit: bool
    evicted: Optional[int] = None


def lecar_update(weights, ghost_kind: str, elapsed: int, learning_rate: float, discount: float):
    """LeCaR's regret update after a ghost hit (policies.py:305-327): a hit in
    the LRU ghost list rewards the LFU weight and vice versa; returns the
    renormalised (w_lru, w_lfu).  The replay kernels apply the same update
    with host-made factors exp(learning_rate * discount**elapsed)."""
    w_lru, w_lfu = weights
    factor = math.exp(learning_rate * discount ** elapsed)
    if ghost_kind == "lru":
        w_lfu *= factor
    elif ghost_kind == "lfu":
        w_lru *= factor
    else:
        raise ValueError(f"ghost_kind must be 'lru' or 'lfu', got {ghost_kind!r}")
    total = w_lru + w_lfu
    return (w_lru / total, w_lfu / total)
