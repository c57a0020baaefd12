"""Migration control message with page tables.

HydraInfer's migration control information carries the request's KV and image page tables
(PAPER.md:379); the reference's ``MigrationJob`` (migration.py:41-61) carries only byte and
block counts.  ``MigrationMessage`` is the control message a source instance sends to the
target when a pull-based migration starts (cluster.py:316-324): which blocks to read
(source page table), where they go (the target's freshly reserved blocks), the request
state the target needs to continue (cached length, last generated token), and the content
descriptor of the request (the synthetic-input seed; a production trace would carry token
ids and image handles here).  The byte format is fixed little-endian and versioned, so it
can cross processes (CUDA-IPC pools on separate ranks) or hosts unchanged:

    header   magic b"HYMG", u16 version (2), u8 kind (0 = EP images, 1 = PD KV),
             u8 n_maps, u32 source instance index, u32 target instance index,
             i64 kv_len, i32 last_token, u64 payload bytes, u64 seed, u16 len(rid), rid utf-8,
             u32 n_prompt, n_prompt x i32 prompt token ids (the request's text content; an
             EP target prefills with them)
    per map  u8 pool (0 = KV, 1 = image), u32 n, u64 block_bytes, u64 group_bytes,
             u64 tail_bytes, n x i32 source ids, n x i32 target ids -- the last block moves
             only the first tail_bytes of each group_bytes group (token-exact,
             hy_copy_blocks_tail), so sum over maps = payload bytes
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import List, Tuple

MAGIC = b"HYMG"
VERSION = 2
KINDS = {"ep": 0, "pd": 1}
POOLS = {"kv": 0, "image": 1}
_HDR = struct.Struct("<4sHBBIIqiQQH")
_MAP = struct.Struct("<BIQQQ")


@dataclass(frozen=True)
class BlockMap:
    pool: str                 # "kv" or "image"
    block_bytes: int
    src_ids: Tuple[int, ...]  # source page table (physical block ids, in sequence order)
    dst_ids: Tuple[int, ...]  # target page table
    group_bytes: int = 0      # 0: whole blocks (group = block)
    tail_bytes: int = 0       # valid bytes per group of the last block (0: whole group)

    def __post_init__(self):
        if self.pool not in POOLS:
            raise ValueError(f"pool must be one of {sorted(POOLS)}")
        if len(self.src_ids) != len(self.dst_ids):
            raise ValueError("source and target page tables differ in length")
        g = self.group_bytes or self.block_bytes
        if g <= 0 or self.block_bytes % g or not 0 <= self.tail_bytes <= g:
            raise ValueError("group_bytes must divide block_bytes; 0 <= tail_bytes <= group")

    @property
    def bytes(self) -> int:
        """Bytes this map moves (the last block token-exact)."""
        n = len(self.src_ids)
        if n == 0:
            return 0
        g = self.group_bytes or self.block_bytes
        return (n - 1) * self.block_bytes + (self.block_bytes // g) * (self.tail_bytes or g)


@dataclass(frozen=True)
class MigrationMessage:
    kind: str                 # "ep" (image embeddings E -> P) or "pd" (KV P -> D)
    rid: str
    source: int               # instance indices in the cluster's instance order
    target: int
    kv_len: int
    last_token: int
    payload_bytes: int        # job.kv_bytes + job.image_bytes (cluster.py:411-413)
    seed: int = 0
    maps: Tuple[BlockMap, ...] = field(default_factory=tuple)
    prompt_ids: Tuple[int, ...] = ()

    def to_bytes(self) -> bytes:
        if self.kind not in KINDS:
            raise ValueError(f"kind must be one of {sorted(KINDS)}")
        rid = self.rid.encode()
        out = [_HDR.pack(MAGIC, VERSION, KINDS[self.kind], len(self.maps), self.source,
                         self.target, self.kv_len, self.last_token, self.payload_bytes,
                         self.seed, len(rid)), rid]
        npr = len(self.prompt_ids)
        out.append(struct.pack(f"<I{npr}i", npr, *self.prompt_ids))
        for m in self.maps:
            n = len(m.src_ids)
            out.append(_MAP.pack(POOLS[m.pool], n, m.block_bytes, m.group_bytes, m.tail_bytes))
            out.append(struct.pack(f"<{n}i{n}i", *m.src_ids, *m.dst_ids))
        return b"".join(out)

    @staticmethod
    def from_bytes(buf: bytes) -> "MigrationMessage":
        (magic, ver, kind, n_maps, source, target, kv_len, last_token, payload, seed,
         rid_len) = _HDR.unpack_from(buf, 0)
        if magic != MAGIC:
            raise ValueError("not a migration message")
        if ver != VERSION:
            raise ValueError(f"unsupported message version {ver}")
        off = _HDR.size
        rid = buf[off:off + rid_len].decode()
        off += rid_len
        (npr,) = struct.unpack_from("<I", buf, off)
        off += 4
        prompt = struct.unpack_from(f"<{npr}i", buf, off)
        off += 4 * npr
        maps: List[BlockMap] = []
        inv_pool = {v: k for k, v in POOLS.items()}
        for _ in range(n_maps):
            pool, n, bb, gb, tb = _MAP.unpack_from(buf, off)
            off += _MAP.size
            ids = struct.unpack_from(f"<{n}i{n}i", buf, off)
            off += 8 * n
            maps.append(BlockMap(inv_pool[pool], bb, tuple(ids[:n]), tuple(ids[n:]), gb, tb))
        if off != len(buf):
            raise ValueError("trailing bytes after the last block map")
        inv_kind = {v: k for k, v in KINDS.items()}
        return MigrationMessage(inv_kind[kind], rid, source, target, kv_len, last_token,
                                payload, seed, tuple(maps), tuple(prompt))
