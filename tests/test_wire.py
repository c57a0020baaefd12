"""Migration control-message wire format (wire.py): exact round trips,
page tables preserved, malformed input rejected; and the message for a real reference
migration carries the block maps the physical pools produce."""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_12658_b200.wire import BlockMap, MigrationMessage  # noqa: E402


def _msg(n_kv=43, n_img=0):
    maps = [BlockMap("kv", 8 << 20, tuple(range(100, 100 + n_kv)),
                     tuple(range(7, 7 + 2 * n_kv, 2)))]
    if n_img:
        maps.append(BlockMap("image", 4718592, tuple(range(n_img)), tuple(range(5, 5 + n_img))))
    return MigrationMessage("pd", "req-00017", 1, 2, 686, 31999, n_kv * (8 << 20), 7,
                            tuple(maps))


@pytest.mark.parametrize("n_kv,n_img", [(0, 0), (1, 0), (43, 0), (869, 4)])
def test_round_trip(n_kv, n_img):
    m = _msg(n_kv, n_img)
    b = m.to_bytes()
    assert MigrationMessage.from_bytes(b) == m
    # header + rid + prompt ids + per map header + 8 bytes per block
    assert len(b) == 46 + len(m.rid) + 4 + sum(29 + 8 * len(x.src_ids) for x in m.maps)


def test_rejects_bad_input():
    b = _msg().to_bytes()
    with pytest.raises(ValueError):
        MigrationMessage.from_bytes(b"XXXX" + b[4:])
    with pytest.raises(ValueError):
        MigrationMessage.from_bytes(b + b"\0")
    with pytest.raises(ValueError):
        BlockMap("kv", 1, (1, 2), (3,))
    with pytest.raises(ValueError):
        MigrationMessage("xx", "r", 0, 1, 0, 0, 0).to_bytes()
