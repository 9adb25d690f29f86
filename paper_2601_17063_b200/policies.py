"""Policy-level types of the drop-in surface (pkg/src/moecache/policies.py:20-48).

The B200 engine evaluates the four north-star policies (LRU, LFU, Belady,
ML) inside its replay kernel; per-access ``CachePolicy`` objects are not
provided.  Victim rules are implemented in
csrc/mcb_kernels.cu (k_replay) as argmin of (key, expert id) over
resident \\ pinned.
"""
from __future__ import annotations

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
