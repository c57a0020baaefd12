"""Migration copy planning (host logic, CPU): for every EP / PD job the reference created
in the golden fixtures (cluster.py:392-421), ``plan_transfer`` moves exactly the job's
bytes -- ``kv_bytes + image_bytes`` (cluster.py:411-413, migration.py:63-64) -- with
whole blocks except a token-exact (KV) / row-exact (image) last block, and reads only
blocks the source holds."""

import types

import pytest

from paper_2505_12658_b200 import get_shape
from paper_2505_12658_b200._epdsim import MC
from paper_2505_12658_b200.cluster import copy_bytes, instance_devices, plan_transfer
from parity_util import load_golden


def _pool(rid, n, first=0, slot=3):
    return types.SimpleNamespace(ids={rid: list(range(first, first + n))}, slot={rid: slot})


@pytest.mark.parametrize("name,shape", [("tiny_EP1_D1", "tiny"), ("tiny_E1_P1_D1", "tiny"),
                                        ("tiny_E1_PD1", "tiny"), ("qwen_EP1_D1", "qwen2-vl-7b")])
def test_plan_moves_exactly_the_job_bytes(name, shape):
    s = get_shape(shape)
    g = load_golden(name)
    assert g["migrations"]
    for kind, src, dst, rid, kv_bytes, image_bytes, kv_blocks, image_blocks in g["migrations"]:
        kv_len = int(kv_bytes) // s.kv_bytes_per_token
        vt = int(image_bytes) // (s.hidden * 2)
        job = types.SimpleNamespace(rid=rid, kind=kind, kv_bytes=kv_bytes,
                                    image_bytes=image_bytes, kv_blocks=kv_blocks,
                                    image_blocks=image_blocks)
        r = types.SimpleNamespace(kv_len=kv_len, plan=types.SimpleNamespace(visual_tokens=vt))
        plan = plan_transfer(job, r, s, _pool(rid, kv_blocks, 0, 1), _pool(rid, kv_blocks, 100, 2),
                             _pool(rid, image_blocks, 7), _pool(rid, image_blocks, 50))
        moved = sum(copy_bytes(len(a), blk, grp, tail) for w, a, b, blk, grp, tail in plan
                    if w != "last_tok")
        assert moved == kv_bytes + image_bytes, (rid, kind)
        for w, a, b, blk, grp, tail in plan:
            assert len(a) == len(b) and blk % grp == 0 and 0 < tail <= grp
            if w == "kv":
                assert len(a) == MC.kv_blocks_needed(kv_len) <= kv_blocks
                assert a == list(range(len(a))) and b == list(range(100, 100 + len(b)))
            elif w == "image":
                assert len(a) == MC.image_blocks_needed(vt) <= image_blocks
            else:
                assert kind == "pd" and (a, b) == ([1], [2])
        assert any(w == "last_tok" for w, *_ in plan) == (kind == "pd")


def test_placement_round_robin_in_construction_order():
    iids = ["E0", "E1", "P0", "P1", "P2", "D0", "D1", "D2"]
    place = instance_devices(iids, [f"cuda:{i}" for i in range(8)])
    assert [place[i].index for i in iids] == list(range(8))
    place = instance_devices(["EP0", "D0"], ["cuda:0"])
    assert {d.index for d in place.values()} == {0}
