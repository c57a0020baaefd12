"""S2: physical paged cache pools.

``PhysicalCachePool`` subclasses the reference ``CachePool`` (engine.py:156-191) and
keeps its exact count semantics -- incremental ``allocate`` that raises
``MemoryError`` when full, idempotent ``release``, ``held``, ``can_allocate``,
``free_blocks``, ``allocated_blocks`` -- and adds what a real executor needs:

  * physical block ids per request, handed out lowest-id-first from a min-heap and
    returned on release (the reference keeps only counts, engine.py:164);
  * a slot per request (a row of the device block table), also lowest-first;
  * a dirty set so the device block table is updated only for requests whose block
    list changed since the last batch.

``allocated_blocks`` is a running counter instead of the reference's O(#holders) sum
(engine.py:166-168); the value is identical.
"""

from __future__ import annotations

import heapq
from typing import Dict, List, Set

from ._epdsim import EN


class PhysicalCachePool(EN.CachePool):
    def __init__(self, block_size: int, capacity_blocks: int, max_slots: int = 0,
                 physical_blocks: int = None):
        super().__init__(block_size, capacity_blocks)
        # Blocks that exist on the device.  Normally == capacity; tests that co-locate
        # several instances on one GPU cap it (ids are lowest-first, so a lightly loaded
        # pool never reaches the cap) and exceeding it is a hard error, not a MemoryError
        # the scheduler would treat as backpressure.
        self.physical_blocks = capacity_blocks if physical_blocks is None else physical_blocks
        self._free: List[int] = list(range(capacity_blocks))  # sorted list is a valid heap
        self._allocated = 0
        self.ids: Dict[str, List[int]] = {}
        self.max_slots = max_slots
        self._free_slots: List[int] = list(range(max_slots))
        self.slot: Dict[str, int] = {}
        self.dirty: Set[str] = set()

    # -- reference count semantics ------------------------------------------
    @property
    def allocated_blocks(self) -> int:
        return self._allocated

    def allocate(self, rid: str, n_blocks: int) -> None:
        new_holder = n_blocks > 0 and rid not in self.ids
        if new_holder and self.max_slots and not self._free_slots and self.can_allocate(n_blocks):
            # checked before any state changes; not a MemoryError, because the reference
            # would have admitted this request (its pool only counts blocks)
            raise RuntimeError(f"no free block-table slot for {rid}: {self.max_slots} "
                               f"concurrent holders (raise max_slots)")
        super().allocate(rid, n_blocks)  # validates, raises MemoryError, updates counts
        if n_blocks == 0:
            return
        self._allocated += n_blocks
        lst = self.ids.get(rid)
        if lst is None:
            lst = self.ids[rid] = []
            if self.max_slots:
                self.slot[rid] = heapq.heappop(self._free_slots)
        pop = heapq.heappop
        free = self._free
        lst.extend(pop(free) for _ in range(n_blocks))
        if lst[-1] >= self.physical_blocks or max(lst[-n_blocks:]) >= self.physical_blocks:
            raise RuntimeError(f"block id {max(lst)} beyond the {self.physical_blocks} "
                               f"physical blocks of this pool (raise the device pool limit)")
        self.dirty.add(rid)

    def release(self, rid: str) -> int:
        n = super().release(rid)
        self._allocated -= n
        ids = self.ids.pop(rid, None)
        if ids:
            push = heapq.heappush
            for b in ids:
                push(self._free, b)
        s = self.slot.pop(rid, None)
        if s is not None:
            heapq.heappush(self._free_slots, s)
        self.dirty.discard(rid)
        return n

    # -- physical view -------------------------------------------------------
    def block_ids(self, rid: str) -> List[int]:
        return self.ids.get(rid, [])

    def consistent(self) -> bool:
        """Physical ids agree with the reference counts (used by invariant checks)."""
        if sum(len(v) for v in self.ids.values()) != self._allocated:
            return False
        if any(len(self.ids.get(r, ())) != n for r, n in self.alloc.items()):
            return False
        held = [b for v in self.ids.values() for b in v]
        return len(set(held)) == len(held) and len(held) + len(self._free) == self.capacity_blocks
