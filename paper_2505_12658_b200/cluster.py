"""Drop-in cluster: epdsim's own event loop with the GPU executor underneath.

``GpuCluster`` subclasses the reference ``Cluster`` (cluster.py:168-488) and keeps its
event loop, router, stage-level batching, admission and migration protocol.  Three
seams change:

  S1  ``_try_schedule`` (cluster.py:287-299): the batch formed by the reference
      ``form_batch`` runs on the instance's GPU via ``InstanceRuntime.run_batch``; its
      latency is epdsim's own ``batch_latency`` (clock="oracle") or measured
      (clock="device" | "wall").
  S2  each instance's ``kv_pool`` / ``image_pool`` is replaced, before any request
      arrives, by a ``PhysicalCachePool`` with the same capacity.
  S3  ``_start_migration`` (cluster.py:392-421) wraps the job in ``GpuMigrationJob``
      whose ``transfer_seconds`` (migration.py:63-64) performs the block copy -- KV
      blocks for PD, image-cache blocks for EP -- when the target reserves its blocks
      (first call, cluster.py:323) and returns the cached value on the accounting call
      (cluster.py:437).

Instances map to devices in construction order (E, P, D, EP, ED, PD, EPD;
cluster.py:180-190): instance k -> devices[k % len(devices)].  Copies between
instances on different GPUs read the source pool through a peer (NVLink) pointer.
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._epdsim import C, EN, MC, MG
from .executor import CLOCKS, InstanceRuntime
from .inputs import ImageStore
from .shapes import MllmShape
from .weights import DeviceWeights
from .wire import BlockMap, MigrationMessage


class GpuMigrationJob(MG.MigrationJob):
    """MigrationJob whose transfer is a real block copy; the measured (or oracle)
    duration is computed once and cached, because the loop asks twice."""

    def bind(self, cluster: "GpuCluster") -> "GpuMigrationJob":
        self._cluster = cluster
        self._seconds = None
        return self

    def transfer_seconds(self, hw) -> float:
        if self._seconds is None:
            self._seconds = self._cluster._execute_transfer(self, hw)
        return self._seconds


class GpuCluster(C.Cluster):
    def __init__(self, spec, shape: MllmShape, hw, slo, *, devices: Sequence = None,
                 clock: str = "device", seed: int = 0, resident_inputs: bool = True,
                 probe_image_tokens: int = MC.IMAGE_BLOCK_TOKENS, max_slots: Optional[int] = None,
                 max_seq_tokens: int = 16384, record_batches: bool = False,
                 weights: Optional[Dict] = None, capture: bool = False,
                 pool_bytes_limit: Optional[int] = None, profile_override=None,
                 budgets: str = "roofline", emulated_link_gbs: Optional[float] = None):
        if clock not in CLOCKS:
            raise ValueError(f"clock must be one of {CLOCKS}")
        if not torch.cuda.is_available():
            raise RuntimeError("GpuCluster needs a CUDA device (there is no CPU fallback)")
        # the scheduler normally sees exactly the executed shape; parity tests that run a
        # depth-reduced model under the full model's decisions pass the full profile
        profile = profile_override if profile_override is not None else shape.profile()
        super().__init__(spec, profile, hw, slo, probe_image_tokens)
        self.shape = shape
        self.clock = clock
        self.seed = seed
        devices = [torch.device(d) for d in (devices or [torch.device("cuda", 0)])]
        self.devices = devices
        self.images = ImageStore(seed, shape.patch)
        self.weights: Dict[torch.device, DeviceWeights] = dict(weights or {})
        self.runtimes: Dict[str, InstanceRuntime] = {}
        place = instance_devices(list(self.instances), devices)
        for iid, inst in self.instances.items():
            dev = place[iid]
            if dev not in self.weights:
                self.weights[dev] = DeviceWeights(shape, dev, seed)
            self.runtimes[iid] = InstanceRuntime(
                inst, shape, self.weights[dev], seed=seed, images=self.images,
                resident_inputs=resident_inputs, max_slots=max_slots,
                max_seq_tokens=max_seq_tokens, capture=capture,
                pool_bytes_limit=pool_bytes_limit)
        if len({d.index for d in devices}) > 1:
            for a in devices:
                for b in devices:
                    if a != b:
                        _lib.check(_lib.load().hy_enable_peer_access(a.index, b.index),
                                   "hy_enable_peer_access")
        self.capture = capture
        # Emulating separate GPUs with instances co-located on one device (the DES runs one
        # batch at a time, so each batch's device time is what a dedicated GPU would
        # measure): a migration between two instances is then an HBM->HBM copy, and its
        # charged time is max(measured, bytes / link) with the link's measured bandwidth.
        self.emulated_link_gbs = emulated_link_gbs
        self.exec_order: List = []
        self.batch_log: Optional[List] = [] if record_batches else None
        self.migration_log: List = []
        self.transfer_stats = {"count": 0, "bytes": 0.0, "copied_bytes": 0, "seconds": 0.0}
        self._live = None  # {iid: in-flight batch} while live.run_live drives the cluster
        self.generated: Dict[str, List[int]] = {}
        # per-batch budgets: the reference's roofline search (decisions identical to the
        # reference) or the same search over GPU-timed probe batches
        if budgets == "measured":
            from .budgets import measured_budgets
            measured_budgets(self)
        elif budgets != "roofline":
            raise ValueError("budgets must be 'roofline' or 'measured'")

    # ------------------------------------------------------------------ S1
    def _try_schedule(self, iid: str) -> None:
        inst = self.instances[iid]
        if inst.busy:
            return
        self._admit_migrations(inst)
        batch = inst.form_batch(self.reqs)
        if not batch:
            return
        if self._live is not None:  # live.run_live: launch, complete on the CUDA events
            self._live[iid] = self.runtimes[iid].launch_batch(batch, self.reqs, self.clock,
                                                             self.model, self.hw)
            if self.capture:
                self.exec_order.append((iid, len(self.runtimes[iid].exec_log)))
            inst.busy = True
            inst.current_batch = batch
            inst.current_latency = 0.0
            return
        latency = self.runtimes[iid].run_batch(batch, self.reqs, self.clock, self.model,
                                               self.hw)
        if self.capture:
            self.exec_order.append((iid, len(self.runtimes[iid].exec_log) - 1))
        if self.batch_log is not None:
            self.batch_log.append((iid, tuple(batch.decode_entries),
                                   tuple(batch.prefill_chunks),
                                   tuple(batch.encode_entries), repr(latency)))
        inst.busy = True
        inst.current_batch = batch
        inst.current_latency = latency
        self._push(self.now + latency, C._BATCH_DONE, iid)

    # ------------------------------------------------------------------ S3
    def _start_migration(self, r, inst, kind: str) -> None:
        super()._start_migration(r, inst, kind)
        job = self.jobs[r.rid]
        fields = {f.name: getattr(job, f.name) for f in dataclasses.fields(job)}
        self.jobs[r.rid] = GpuMigrationJob(**fields).bind(self)

    def _execute_transfer(self, job: GpuMigrationJob, hw) -> float:
        """Launch the job's block copy on the target's copy stream (pull: the target GPU's
        SMs read the source pool, through a peer NVLink pointer when the instances sit on
        different GPUs) and return its duration under the cluster clock.

        Token-exact: whole blocks except the last one, of which only the valid tokens (KV)
        or rows (image) move, so the bytes copied equal ``job.kv_bytes + job.image_bytes``
        (cluster.py:411-413).  Ordering is by events, never a device-wide sync: the copy
        waits for the source's last batch; both instances' next batches wait for the copy
        (the target reads the blocks, the source may reuse them once it releases them at
        MIG_DONE).  clock="device" waits for the copy's completion event to charge the
        measured time; in live mode (live.py) nothing waits here -- MIG_DONE is delivered
        when the completion event fires."""
        src = self.runtimes[job.source]
        dst = self.runtimes[job.target]
        r = self.reqs[job.rid]
        lib = _lib.load()
        bases = {"kv": (src.kv, dst.kv), "image": (src.img, dst.img),
                 "last_tok": (src.last_tok, dst.last_tok)}
        maps = [(w, a, b_) + bases[w] + (blk, grp, tail) for w, a, b_, blk, grp, tail in
                plan_transfer(job, r, self.shape, src.kv_pool, dst.kv_pool, src.image_pool,
                              dst.image_pool)]
        dev = dst.device
        st = dst.copy_stream()
        ids_host = np.concatenate([np.asarray(list(m[1]) + list(m[2]), dtype=np.int32)
                                   for m in maps]) if maps else np.zeros(0, np.int32)
        with torch.cuda.device(dev), torch.cuda.stream(st):
            ids = torch.from_numpy(ids_host).to(dev)  # ordered on the copy stream
            for ev in src.last_events():
                st.wait_event(ev)
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(st)
            copied = 0
            off = 0
            for what, s_ids, d_ids, s_pool, d_pool, block, group, tail in maps:
                n = len(s_ids)
                _lib.check(lib.hy_copy_blocks_tail(
                    s_pool.data_ptr(), d_pool.data_ptr(), ids.data_ptr() + 4 * off,
                    ids.data_ptr() + 4 * (off + n), n, block, group, tail, st.cuda_stream),
                    "hy_copy_blocks_tail")
                off += 2 * n
                if what != "last_tok":
                    copied += copy_bytes(n, block, group, tail)
            ev1.record(st)
        dst.launches += len(maps)
        for rt in (src, dst):
            rt.wait_before_next_batch(ev1)
        job._copy = (ev0, ev1, ids)
        self.transfer_stats["count"] += 1
        self.transfer_stats["bytes"] += job.kv_bytes + job.image_bytes
        self.transfer_stats["copied_bytes"] += copied
        kind = self.transfer_stats.setdefault(job.kind, {"count": 0, "bytes": 0, "seconds": 0.0})
        kind["count"] += 1
        kind["bytes"] += copied
        self.migration_log.append([job.kind, job.source, job.target, job.rid,
                                   [(w, list(a), list(b_)) for w, a, b_, *_ in maps
                                    if w != "last_tok"], None])
        job._log_entry = self.migration_log[-1]
        # the control message a separate-process target would receive (wire.py, f4)
        iids = list(self.instances)
        msg = MigrationMessage(
            job.kind, job.rid, iids.index(job.source), iids.index(job.target), r.kv_len,
            -1, int(job.kv_bytes + job.image_bytes), self.seed,
            tuple(BlockMap(w, bb, tuple(a), tuple(b_), gb, tb)
                  for w, a, b_, _, _, bb, gb, tb in maps if w != "last_tok"),
            tuple(int(t) for t in src.prompt(r)) if job.kind == "ep" else ())
        self.transfer_stats["control_bytes"] = (self.transfer_stats.get("control_bytes", 0) +
                                                len(msg.to_bytes()))
        self.last_migration_message = msg
        if self._live is not None:
            return 0.0  # provisional: live.py charges the measured time at completion
        if self.clock == "oracle":
            return MG.MigrationJob.transfer_seconds(job, hw)
        return self._finish_copy(job)

    def copy_done(self, job) -> bool:
        """True once the job's copy has completed on the device (live mode polls this)."""
        c = getattr(job, "_copy", None)
        return c is None or c[1].query()

    def _finish_copy(self, job) -> float:
        """Wait for the job's copy, record its measured time; returns seconds."""
        ev0, ev1, _ = job._copy
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1)
        if self.emulated_link_gbs:
            ms = max(ms, (job.kv_bytes + job.image_bytes) / (self.emulated_link_gbs * 1e6))
        job._copy = None
        job._seconds = ms * 1e-3
        job._log_entry[5] = ms
        self.transfer_stats["seconds"] += ms * 1e-3
        self.transfer_stats[job.kind]["seconds"] += ms * 1e-3
        return ms * 1e-3

    # ------------------------------------------------------------------ results
    def _finish(self, r, inst) -> None:
        super()._finish(r, inst)
        self.runtimes[inst.id].forget(r.rid)

    def run(self, trace, check_invariants: bool = False):
        report = super().run(trace, check_invariants=check_invariants)
        self._collect_generated()
        return report

    def _collect_generated(self) -> None:
        merged: Dict[str, List] = {}
        for rt in self.runtimes.values():
            rt.collect_tokens(rt.generated)
            for rid, toks in rt.generated.items():
                merged.setdefault(rid, []).extend(toks)
            rt.generated.clear()
        for rid, toks in merged.items():
            self.generated[rid] = [t for _, t in sorted(toks)]

    def _assert_invariants(self) -> None:
        super()._assert_invariants()
        for iid, rt in self.runtimes.items():
            for pool in (rt.kv_pool, rt.image_pool):
                if not pool.consistent():
                    raise AssertionError(f"physical pool of {iid} disagrees with its counts")

    def close(self) -> None:
        """Drop every device buffer of this cluster (pools, tables, workspaces) so the
        next cluster on the same GPU can reuse the memory; shared weights stay."""
        for rt in self.runtimes.values():
            rt.close()
        self.runtimes = {}
        self.jobs.clear()
        import gc
        gc.collect()

    def gpu_launch_count(self) -> int:
        return sum(rt.launches for rt in self.runtimes.values())


def copy_bytes(n: int, block: int, group: int, tail: int) -> int:
    """Bytes ``hy_copy_blocks_tail`` moves for n blocks (the last one token-exact)."""
    return 0 if n <= 0 else (n - 1) * block + (block // group) * tail


def plan_transfer(job, r, shape: MllmShape, src_kv, dst_kv, src_img, dst_img) -> List:
    """The block copies of one migration job: [(pool, src ids, dst ids, block bytes, group
    bytes, tail bytes per group)].  KV: the ``kv_blocks_needed(kv_len)`` blocks holding the
    request's tokens, the last one token-exact; image: the blocks holding its
    ``visual_tokens`` rows (packed contiguously from its first block), the last one
    row-exact; PD jobs also carry the 4-byte last sampled token of the request's slot.
    The copied bytes therefore equal ``job.kv_bytes + job.image_bytes`` (cluster.py:411-413).
    Pure host logic (CPU-tested)."""
    out = []
    if job.kv_bytes > 0:
        kv_n = MC.kv_blocks_needed(r.kv_len)
        valid = r.kv_len - (kv_n - 1) * MC.KV_BLOCK_TOKENS
        grp = MC.KV_BLOCK_TOKENS * shape.head_dim * 2
        out.append(("kv", list(src_kv.ids[job.rid][:kv_n]), list(dst_kv.ids[job.rid][:kv_n]),
                    shape.kv_block_elems * 2, grp, valid * shape.head_dim * 2))
    if job.image_bytes > 0:
        vt = r.plan.visual_tokens
        img_n = min(job.image_blocks, MC.image_blocks_needed(vt))
        blk = shape.image_block_elems * 2
        valid = vt - (img_n - 1) * MC.IMAGE_BLOCK_TOKENS
        out.append(("image", list(src_img.ids[job.rid][:img_n]),
                    list(dst_img.ids[job.rid][:img_n]), blk, blk, valid * shape.hidden * 2))
    if job.kind == "pd":
        out.append(("last_tok", [src_kv.slot[job.rid]], [dst_kv.slot[job.rid]], 4, 4, 4))
    return out


def instance_devices(instance_ids: Sequence[str], devices: Sequence) -> Dict[str, "torch.device"]:
    """Placement: instance k, in the reference's construction order
    (cluster.py:180-190), runs on devices[k % len(devices)]."""
    devs = [torch.device(d) for d in devices]
    return {iid: devs[k % len(devs)] for k, iid in enumerate(instance_ids)}


def batch_log_digest(log) -> str:
    """sha256[:16] of a batch log, the recipe in BASELINE.md section 2."""
    return hashlib.sha256(json.dumps(log).encode()).hexdigest()[:16]


def run_trace_gpu(spec, shape: MllmShape, hw, slo, trace, *, check_invariants: bool = False,
                  **kw):
    """GPU counterpart of ``epdsim.run_trace`` (cluster.py:491-497)."""
    cluster = GpuCluster(spec, shape, hw, slo, **kw)
    report = cluster.run(trace, check_invariants=check_invariants)
    return cluster, report
