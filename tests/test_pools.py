"""S2 tests on CPU: PhysicalCachePool keeps the reference CachePool's count semantics
(engine.py:156-191) and hands out the documented physical ids.

The reference cluster is run with its pools swapped for PhysicalCachePool; decisions must
stay bit-identical to the golden logs and every allocation's ids must equal the oracle
restatement (oracle/block_alloc.py) replayed on the reference's own pool events.
"""

import pytest

from oracle.batch_log import block_maps, digest
from oracle.block_alloc import OracleBlockPool
from paper_2505_12658_b200._epdsim import C, E, EN
from paper_2505_12658_b200.pools import PhysicalCachePool
from parity_util import golden_trace, load_golden


def test_count_semantics_match_reference_pool():
    ref = EN.CachePool(16, 10)
    phy = PhysicalCachePool(16, 10, max_slots=4)
    for rid, n in [("a", 3), ("b", 0), ("a", 2), ("c", 5)]:
        ref.allocate(rid, n)
        phy.allocate(rid, n)
        assert (ref.allocated_blocks, ref.free_blocks, ref.held(rid)) == \
               (phy.allocated_blocks, phy.free_blocks, phy.held(rid))
    for pool in (ref, phy):
        with pytest.raises(MemoryError):
            pool.allocate("d", 1)
        with pytest.raises(ValueError):
            pool.allocate("d", -1)
        assert not pool.can_allocate(1)
    assert phy.block_ids("a") == [0, 1, 2, 3, 4] and phy.block_ids("c") == [5, 6, 7, 8, 9]
    assert ref.release("a") == phy.release("a") == 5
    assert ref.release("a") == phy.release("a") == 0  # idempotent
    phy.allocate("e", 2)
    assert phy.block_ids("e") == [0, 1]  # lowest ids first
    assert phy.slot["e"] == 0 and phy.slot["c"] == 1  # "b" allocated 0 blocks: no slot
    assert phy.consistent()


def test_physical_limit_is_a_hard_error():
    phy = PhysicalCachePool(16, 100, physical_blocks=4)
    phy.allocate("a", 4)
    with pytest.raises(RuntimeError):
        phy.allocate("b", 1)


class _PhysCluster(C.Cluster):
    """Reference cluster with physical pools; records ids per allocation episode."""

    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.alloc_log = {}
        episodes = {}
        for iid, inst in self.instances.items():
            for kind in ("kv", "image"):
                old = getattr(inst, kind + "_pool")
                new = PhysicalCachePool(old.block_size, old.capacity_blocks,
                                        max_slots=4096 if kind == "kv" else 0)
                log, ep = self.alloc_log, episodes

                def alloc(rid, n, _new=new, _iid=iid, _kind=kind, _orig=new.allocate):
                    _orig(rid, n)
                    if n:
                        k = ep.get((_iid, _kind, rid), 0)
                        log[(_iid, _kind, rid, k)] = list(_new.ids[rid])

                def rel(rid, _new=new, _iid=iid, _kind=kind, _orig=new.release):
                    n = _orig(rid)
                    if n:
                        ep[(_iid, _kind, rid)] = ep.get((_iid, _kind, rid), 0) + 1
                    return n

                new.allocate, new.release = alloc, rel
                setattr(inst, kind + "_pool", new)


@pytest.mark.parametrize("name", ["config1_2000rps", "tiny_EP1_D1", "tiny_E1_P1_D1",
                                  "tiny_E1_PD1", "qwen_EP1_D1"])
def test_block_ids_match_oracle_policy(name):
    g = load_golden(name)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(g["method"]))
    log = []
    orig = C.batch_latency

    def lat(batch, reqs, m, h):
        v = orig(batch, reqs, m, h)
        first = (batch.decode_entries or batch.prefill_chunks or batch.encode_entries)[0][0]
        log.append((reqs[first].current_instance, tuple(batch.decode_entries),
                    tuple(batch.prefill_chunks), tuple(batch.encode_entries), repr(v)))
        return v

    C.batch_latency = lat
    try:
        cl = _PhysCluster(spec, E.ModelProfile(**g["model"]), E.HardwareProfile(*g["hw"]),
                          E.SloSpec(*g["slo"]))
        cl.run(golden_trace(E, g), check_invariants=True)
    finally:
        C.batch_latency = orig
    assert digest(log) == g["sha"]  # decisions unchanged by the physical pools
    caps = {}
    for iid, (kvb, imb) in g["capacities"].items():
        caps[(iid, "kv")] = kvb
        caps[(iid, "image")] = imb
    expect = block_maps([tuple(e) for e in g["pool_events"]], caps)
    assert cl.alloc_log == expect


def test_oracle_pool_matches_reference_counts():
    ref = EN.CachePool(16, 6)
    o = OracleBlockPool(6)
    for op in [("a", 2), ("b", 3), ("a", 1), ("rel", "b"), ("c", 3)]:
        if op[0] == "rel":
            assert ref.release(op[1]) == o.release(op[1])
        else:
            ref.allocate(*op)
            o.allocate(*op)
        for rid in "abc":
            assert ref.held(rid) == o.held(rid)
    assert o.ids["c"] == [2, 3, 4]
