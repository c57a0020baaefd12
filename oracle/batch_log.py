"""Golden scheduler logs captured from the reference ``epdsim`` -- TEST INFRASTRUCTURE.

``capture(...)`` replays a trace through the unmodified reference ``run_trace``
(cluster.py:491-497) and records, by wrapping the two seams:
  * every batch: (iid, decode_entries, prefill_chunks, encode_entries, repr(latency))
    -- the recipe of BASELINE.md section 2 (iid recovered from
    ``reqs[first rid].current_instance``, set at cluster.py:282,426);
  * every migration job: (kind, source, target, rid, kv_bytes, image_bytes, kv_blocks,
    image_blocks) at ``_start_migration`` (cluster.py:392-421);
  * every pool event (instance, pool, op, rid, n) so block-id maps can be restated
    by ``block_alloc.OracleBlockPool``.
The wrappers only observe; the reference decides everything.
"""

from __future__ import annotations

import hashlib
import json
from contextlib import contextmanager
from typing import Dict, List


def digest(log) -> str:
    return hashlib.sha256(json.dumps(log).encode()).hexdigest()[:16]


@contextmanager
def _patched(obj, name, new):
    old = getattr(obj, name)
    setattr(obj, name, new)
    try:
        yield old
    finally:
        setattr(obj, name, old)


def capture(epdsim, spec, model, hw, slo, trace) -> Dict:
    C = epdsim.cluster
    EN = epdsim.engine
    batches: List = []
    migrations: List = []
    pool_events: List = []

    orig_lat = C.batch_latency

    def lat(batch, reqs, m, h):
        v = orig_lat(batch, reqs, m, h)
        first = (batch.decode_entries or batch.prefill_chunks or batch.encode_entries)[0][0]
        batches.append((reqs[first].current_instance, tuple(batch.decode_entries),
                        tuple(batch.prefill_chunks), tuple(batch.encode_entries), repr(v)))
        return v

    orig_start = C.Cluster._start_migration

    def start(self, r, inst, kind):
        orig_start(self, r, inst, kind)
        j = self.jobs[r.rid]
        migrations.append((j.kind, j.source, j.target, j.rid, j.kv_bytes, j.image_bytes,
                           j.kv_blocks, j.image_blocks))

    class LoggedPool(EN.CachePool):
        owner = None
        kind = None

        def allocate(self, rid, n):
            super().allocate(rid, n)
            if n:
                pool_events.append((self.owner, self.kind, "alloc", rid, n))

        def release(self, rid):
            n = super().release(rid)
            if n:
                pool_events.append((self.owner, self.kind, "release", rid, n))
            return n

    orig_init = EN.InstanceState.__init__

    def init(self, iid, itype, kv_cap, img_cap, budgets, policy=EN.STAGE_LEVEL):
        orig_init(self, iid, itype, kv_cap, img_cap, budgets, policy)
        for kind in ("kv", "image"):
            old = getattr(self, kind + "_pool")
            p = LoggedPool(old.block_size, old.capacity_blocks)
            p.owner, p.kind = iid, kind
            setattr(self, kind + "_pool", p)

    with _patched(C, "batch_latency", lat), \
            _patched(C.Cluster, "_start_migration", start), \
            _patched(EN.InstanceState, "__init__", init):
        report = C.run_trace(spec, model, hw, slo, trace, check_invariants=True)
    return {"batches": batches, "migrations": migrations, "pool_events": pool_events,
            "aggregates": report.aggregates}


def block_maps(pool_events, capacities: Dict) -> Dict:
    """Restate physical block ids from pool events: {(iid, kind, rid, k): ids} for the
    k-th allocation episode of rid on that pool, using OracleBlockPool."""
    from .block_alloc import OracleBlockPool
    pools = {key: OracleBlockPool(cap) for key, cap in capacities.items()}
    episodes: Dict = {}
    out: Dict = {}
    for owner, kind, op, rid, n in pool_events:
        p = pools[(owner, kind)]
        if op == "alloc":
            k = episodes.get((owner, kind, rid), 0)
            p.allocate(rid, n)
            out[(owner, kind, rid, k)] = list(p.ids[rid])
        else:
            p.release(rid)
            episodes[(owner, kind, rid)] = episodes.get((owner, kind, rid), 0) + 1
    return out
