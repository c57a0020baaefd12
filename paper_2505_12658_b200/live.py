"""Live asynchronous serving loop.

``GpuCluster.run`` replays a trace as a discrete-event simulation: each batch executes on
the GPU, but virtual time jumps by the batch's measured latency and only one batch is in
flight in the whole cluster at any moment (the reference's event loop, cluster.py:231-259).
``run_live`` drives the same cluster in wall-clock time instead:

* requests arrive when the wall clock reaches ``arrival_time + preprocess_delay`` (scaled by
  ``time_scale``: 2.0 replays the trace twice as fast);
* every idle instance launches its next batch asynchronously on its own V/L streams
  (``InstanceRuntime.launch_batch``), so instances on different GPUs -- or sharing one -- run
  concurrently, each with at most one batch in flight (the reference's ``busy`` flag);
* a batch completes when its CUDA events do (``batch_done`` polls them); its measured latency
  is charged to the requests and the reference's own ``_on_batch_done`` runs at the wall
  time of completion, so token timestamps, TTFT and TBT are real;
* migration control / completion events keep the reference's handlers
  (``_on_mig_control`` / ``_on_mig_done``); the block copy is launched asynchronously on the
  target's copy stream when the target reserves the blocks (``GpuMigrationJob``), and
  ``_on_mig_done`` runs when the copy's completion event fires, charged with the copy's
  measured device time (the loop never blocks on a copy).

The scheduler, admission, budgets, migration protocol and report are the reference's code,
unchanged; only the clock and the overlap differ.  One driver thread polls every instance
(launches are asynchronous, so a thread per GPU is not needed to keep the GPUs busy).
"""

from __future__ import annotations

import heapq
import time

from ._epdsim import C


def run_live(cluster, trace, *, time_scale: float = 1.0, check_invariants: bool = False,
             idle_sleep_s: float = 1e-4, timeout_s: float = 3600.0):
    """Serve ``trace`` on ``cluster`` (a ``GpuCluster``) in wall-clock time; returns the
    reference ``SimReport``.  ``cluster.batch_log`` entries carry the measured latency."""
    if time_scale <= 0:
        raise ValueError("time_scale must be positive")
    cluster.check_invariants = check_invariants
    for req in trace.requests:
        plan = C.plan_stages(req, cluster.spec.preprocess_delay)
        cluster.reqs[req.id] = C.RequestState(spec=req, plan=plan)
        cluster._push(req.arrival_time + plan.preprocess_delay, C._ARRIVAL, req.id)
    cluster._live = {}
    copies = []  # MIG_DONE events whose copy is still running on the device
    t0 = time.perf_counter()

    def now() -> float:
        return (time.perf_counter() - t0) * time_scale

    try:
        while cluster._heap or cluster._live or copies:
            progressed = False
            for iid in list(cluster._live):
                rt = cluster.runtimes[iid]
                if not rt.batch_done():
                    continue
                h = cluster._live.pop(iid)
                latency = rt.complete_batch(h)
                inst = cluster.instances[iid]
                inst.current_latency = latency
                if cluster.batch_log is not None:
                    b = inst.current_batch
                    cluster.batch_log.append((iid, tuple(b.decode_entries),
                                              tuple(b.prefill_chunks),
                                              tuple(b.encode_entries), repr(latency)))
                cluster.now = now()
                cluster._on_batch_done(iid)
                progressed = True
            for rid in list(copies):
                job = cluster.jobs[rid]
                if cluster.copy_done(job):
                    copies.remove(rid)
                    cluster._finish_copy(job)
                    cluster.now = now()
                    cluster._on_mig_done(rid)
                    progressed = True
            t = now()
            while cluster._heap and cluster._heap[0][0] <= t:
                _, _, kind, payload = heapq.heappop(cluster._heap)
                cluster.now = t
                if kind == C._ARRIVAL:
                    cluster._on_arrival(payload)
                elif kind == C._MIG_CONTROL:
                    cluster._on_mig_control(payload)
                elif kind == C._MIG_DONE:
                    job = cluster.jobs[payload]
                    if getattr(job, "_copy", None) is not None:
                        copies.append(payload)  # delivered when the copy completes
                    else:
                        cluster._on_mig_done(payload)
                else:
                    raise AssertionError(f"unexpected event {kind} in live mode")
                progressed = True
            if check_invariants and progressed:
                cluster._assert_invariants()
            if not progressed:
                if t / time_scale > timeout_s:
                    raise TimeoutError(f"live run exceeded {timeout_s} s")
                time.sleep(idle_sleep_s)
    finally:
        live = cluster._live
        cluster._live = None
        for iid, h in (live or {}).items():  # error path: do not leave work in flight
            cluster.runtimes[iid].complete_batch(h)
    if cluster.finished != cluster.arrived:
        cluster._raise_deadlock()
    report = C.metrics_mod.build_report([cluster.reqs[r.id] for r in trace.requests],
                                        meta=cluster._meta(trace),
                                        migrations=cluster.completed_migrations)
    cluster._collect_generated()
    return report
