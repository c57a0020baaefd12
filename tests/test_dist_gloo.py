"""Multi-process (world_size 2, gloo, CPU) test of the N>1 bench path: each rank takes its
round-robin shard of the trace (independent units, no data-path collective), replays it
through the reference scheduler, and the scalar metrics are all-reduced exactly as
bench.py does on GPUs."""

import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    from paper_2505_12658_b200._epdsim import C, E
    d = bench.Dist()
    base, slo = bench.base_trace(E, 40 * world)
    mine = bench.shard(E, E.scale_to_rate(base, 20.0 * world), d.rank, d.world)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    rep = C.run_trace(spec, E.MODEL_PRESETS["llava-1.5-7b"], E.DEFAULT_HARDWARE, slo, mine)
    meets = sum(1 for m in rep.requests if E.meets_slo(m))
    tot = d.reduce([meets, len(rep.requests)])
    ids = [r.id for r in mine.requests]
    gathered = [None] * world
    dist.all_gather_object(gathered, ids)
    out[rank] = (tot, sorted(i for g in gathered for i in g), len(ids))
    d.close()


def test_two_rank_sharding_and_reduction():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    (t0, ids0, n0), (t1, ids1, n1) = out[0], out[1]
    assert t0 == t1                                  # both ranks see the same totals
    assert t0[1] == 80 and n0 == n1 == 40             # every request exactly once
    assert ids0 == ids1 and len(set(ids0)) == 80
    assert 0 <= t0[0] <= 80
