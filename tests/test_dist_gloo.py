"""Multi-process (world_size 2, gloo, CPU) test of the N>1 bench plumbing.

``bench.py --gpus N`` under torchrun: the serving cluster is one event loop (the
reference's), so rank 0 drives every GPU -- instance k of the deployment on GPU k -- and
the other ranks only wait for it at a barrier.  Checked here without a GPU:
  * every rank derives the same deployment and workload config for N (SURVEY.md 8e:
    EP:1,D:1 on 2 GPUs), and the reference arm reports the identical config;
  * the placement puts one instance per GPU slot in the reference's construction order;
  * rank 0's work (here: the reference replay of the deployment on the trace, with every
    migration planned by ``plan_transfer`` and moving exactly the job's bytes) completes
    while rank 1 waits, and both ranks leave the barrier."""

import os
import socket
import types

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
    from paper_2505_12658_b200 import get_shape
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import copy_bytes, instance_devices, plan_transfer
    d = bench.Dist()
    args = types.SimpleNamespace(gpus=1, method=None, model="llava-1.5-7b", requests=20,
                                 trace="textcaps",
                                 rate_lo=16.0, rate_hi=128.0)
    n = bench.n_gpus(args, d)
    cfg = bench.workload_config(args, n)
    cfgs = [None] * world
    dist.all_gather_object(cfgs, cfg)
    res = {"n": n, "cfg_equal": all(c == cfg for c in cfgs), "method": cfg["method"]}
    if rank == 0:
        spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(cfg["method"]))
        shape = get_shape(args.model)
        base, slo = bench.base_trace(E, cfg["requests"])
        cl = C.Cluster(spec, shape.profile(), E.DEFAULT_HARDWARE, slo)
        place = instance_devices(list(cl.instances), [f"cuda:{i}" for i in range(n)])
        res["placement"] = {iid: dv.index for iid, dv in place.items()}
        moved = []
        orig = C.Cluster._start_migration

        def start(self, r, inst, kind):
            orig(self, r, inst, kind)
            job = self.jobs[r.rid]
            pools = {k: types.SimpleNamespace(ids={r.rid: list(range(b))}, slot={r.rid: 0})
                     for k, b in (("kv", job.kv_blocks), ("img", job.image_blocks))}
            plan = plan_transfer(job, r, shape, pools["kv"], pools["kv"], pools["img"],
                                 pools["img"])
            moved.append((sum(copy_bytes(len(a), *x) for w, a, _, *x in plan
                              if w != "last_tok"), job.kv_bytes + job.image_bytes))
        C.Cluster._start_migration = start
        try:
            rep = cl.run(E.scale_to_rate(base, 10.0))
        finally:
            C.Cluster._start_migration = orig
        res["finished"] = rep.aggregates["n_finished"]
        res["moved"] = moved
    d.barrier()  # rank 1 waits here for rank 0, as in bench.run_ours
    out[rank] = res
    d.close()


def test_two_rank_disaggregated_plumbing():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, r1 = out[0], out[1]
    assert r0["n"] == r1["n"] == 2 and r0["method"] == r1["method"] == "EP:1,D:1"
    assert r0["cfg_equal"] and r1["cfg_equal"]
    assert r0["placement"] == {"D0": 0, "EP0": 1}  # construction order E, P, D, EP, ...
    assert r0["finished"] == 40
    assert len(r0["moved"]) == 40  # every request migrates EP0 -> D0 once (PD)
    assert all(a == b for a, b in r0["moved"])
