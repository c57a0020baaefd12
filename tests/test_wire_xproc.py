"""The migration control message (wire.py, f4) consumed by a separate process.

Two processes (gloo, CPU): the source holds a block pool and, for every migration job the
reference created in a golden fixture, sends the control message bytes followed by the
payload it gathers by the message's source page table (token-exact last block); the target
knows nothing but its own pool -- it decodes the message and scatters the payload by the
target page table.  Checked: the target pool equals the source's blocks at the mapped ids,
byte for byte within the valid tail, the payload size equals the job's bytes
(cluster.py:411-413), and EP messages carry the request's prompt token ids."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

KV_TOK_BYTES = 4096   # tiny model: 2 layers x K,V x 4 heads x 128 x bf16 per token
HEAD_BYTES = 256      # 128 dims x bf16
BLOCK = 16 * KV_TOK_BYTES


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _messages():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from parity_util import load_golden
    from paper_2505_12658_b200 import get_shape
    from paper_2505_12658_b200.inputs import prompt_tokens
    from paper_2505_12658_b200.wire import BlockMap, MigrationMessage
    s = get_shape("tiny")
    g = load_golden("tiny_E1_P1_D1")
    rng = np.random.default_rng(3)
    out = []
    for kind, src, dst, rid, kv_bytes, img_bytes, kv_blocks, img_blocks in g["migrations"]:
        maps = []
        if kv_bytes:
            kv_len = int(kv_bytes) // s.kv_bytes_per_token
            n = -(-kv_len // 16)
            valid = kv_len - (n - 1) * 16
            maps.append(BlockMap("kv", s.kv_block_elems * 2,
                                 tuple(int(x) for x in rng.choice(200, n, replace=False)),
                                 tuple(int(x) for x in rng.choice(200, n, replace=False)),
                                 16 * s.head_dim * 2, valid * s.head_dim * 2))
        if img_bytes:
            vt = int(img_bytes) // (s.hidden * 2)
            n = -(-vt // 576)
            blk = s.image_block_elems * 2
            maps.append(BlockMap("image", blk,
                                 tuple(int(x) for x in rng.choice(40, n, replace=False)),
                                 tuple(int(x) for x in rng.choice(40, n, replace=False)),
                                 blk, (vt - (n - 1) * 576) * s.hidden * 2))
        prompt = tuple(int(t) for t in prompt_tokens(0, rid, 37, s.vocab)) if kind == "ep" else ()
        out.append(MigrationMessage(kind, rid, 0, 1, 0, -1, int(kv_bytes + img_bytes), 0,
                                    tuple(maps), prompt))
    return out


def _pools(seed):
    from paper_2505_12658_b200 import get_shape
    s = get_shape("tiny")
    rng = np.random.default_rng(seed)
    return {"kv": rng.integers(0, 255, (200, s.kv_block_elems * 2), dtype=np.uint8),
            "image": rng.integers(0, 255, (40, s.image_block_elems * 2), dtype=np.uint8)}


def _segments(m):
    """(block position, byte offset, length) runs the map moves, in payload order."""
    g = m.group_bytes or m.block_bytes
    for i in range(len(m.src_ids)):
        if i + 1 < len(m.src_ids) or (m.tail_bytes or g) == g:
            yield i, 0, m.block_bytes
        else:
            for k in range(m.block_bytes // g):
                yield i, k * g, m.tail_bytes


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from paper_2505_12658_b200.wire import MigrationMessage
    if rank == 0:  # source: message, then the payload gathered by the source page table
        pools = _pools(11)
        for msg in _messages():
            b = np.frombuffer(msg.to_bytes(), dtype=np.uint8)
            dist.send(torch.tensor([b.size]), 1)
            dist.send(torch.from_numpy(b.copy()), 1)
            parts = [pools[m.pool][m.src_ids[i], o:o + n] for m in msg.maps
                     for i, o, n in _segments(m)]
            pay = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
            dist.send(torch.tensor([pay.size]), 1)
            if pay.size:
                dist.send(torch.from_numpy(pay), 1)
        dist.send(torch.tensor([-1]), 1)
        out[0] = "sent"
    else:  # target: only its own pools; everything else comes from the message
        pools = _pools(99)
        got, prompts, sizes = [], {}, []
        while True:
            n = torch.zeros(1, dtype=torch.int64)
            dist.recv(n, 0)
            if n.item() < 0:
                break
            b = torch.zeros(n.item(), dtype=torch.uint8)
            dist.recv(b, 0)
            msg = MigrationMessage.from_bytes(b.numpy().tobytes())
            k = torch.zeros(1, dtype=torch.int64)
            dist.recv(k, 0)
            pay = torch.zeros(k.item(), dtype=torch.uint8)
            if k.item():
                dist.recv(pay, 0)
            pay = pay.numpy()
            off = 0
            for m in msg.maps:
                for i, o, nb in _segments(m):
                    pools[m.pool][m.dst_ids[i], o:o + nb] = pay[off:off + nb]
                    off += nb
            assert off == pay.size == msg.payload_bytes
            sizes.append((msg.payload_bytes, sum(m.bytes for m in msg.maps)))
            if msg.kind == "ep":
                prompts[msg.rid] = msg.prompt_ids
            got.append(msg)
        out[1] = ({k: v for k, v in pools.items()}, got, prompts, sizes)
    dist.destroy_process_group()


def test_message_consumed_by_another_process():
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(port, out), nprocs=2, join=True)
    pools, got, prompts, sizes = out[1]
    want = _messages()
    assert got == want
    assert all(a == b for a, b in sizes)
    src = _pools(11)
    exp = _pools(99)
    for msg in want:  # the target pool = the source's blocks at the mapped ids (valid bytes)
        for m in msg.maps:
            for i, o, n in _segments(m):
                exp[m.pool][m.dst_ids[i], o:o + n] = src[m.pool][m.src_ids[i], o:o + n]
    for k in exp:
        assert np.array_equal(pools[k], exp[k])
    assert prompts and all(len(p) == 37 for p in prompts.values())
