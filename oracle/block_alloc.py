"""Restatement of the reference's paged-pool accounting plus the physical-id policy
-- TEST INFRASTRUCTURE ONLY.

Counts follow ``CachePool`` (/root/reference/pkg/src/epdsim/engine.py:156-191):
incremental ``allocate(rid, n)`` that fails when ``n > free``, ``release(rid)`` that
returns the held count and is idempotent.  The reference has no block ids; the ids
restated here are the builder's documented policy: the lowest free id first,
in ascending order, released ids return to the free set.  Written with a sorted list +
bisect, independently of the heap in ``paper_2505_12658_b200/pools.py``.
"""

from __future__ import annotations

import bisect
from typing import Dict, List


class OracleBlockPool:
    def __init__(self, capacity: int):
        self.capacity = capacity
        self.free: List[int] = list(range(capacity))
        self.ids: Dict[str, List[int]] = {}

    def allocate(self, rid: str, n: int) -> List[int]:
        if n < 0:
            raise ValueError("n must be >= 0")
        if n > len(self.free):
            raise MemoryError(f"pool exhausted allocating {n} blocks for {rid}")
        taken, self.free = self.free[:n], self.free[n:]
        if n:
            self.ids.setdefault(rid, []).extend(taken)
        return taken

    def release(self, rid: str) -> int:
        ids = self.ids.pop(rid, [])
        for b in ids:
            bisect.insort(self.free, b)
        return len(ids)

    def held(self, rid: str) -> int:
        return len(self.ids.get(rid, ()))
