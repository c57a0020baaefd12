"""The path on the CPU: epdsim batches executed by the fp32 port -- TEST / BASELINE ONLY.

``bench.py --impl reference`` (and its ``cpu_baseline`` leg) time the reference's own CPU
implementation of the hot path.  The reference (epdsim) prices a batch analytically and
executes no model, so the CPU implementation of the path is this
port: the unmodified reference scheduler forms every batch (Algorithm 1, engine.py:333-404)
and ``CpuPathExecutor`` is bound at the executor seam the reference exposes for it --
``batch_latency`` is looked up as a module global of ``epdsim.cluster`` at cluster.py:295
 -- executing the batch on ``OracleMLLM`` and returning the measured
seconds (a measured-clock replay, like the GPU arm's).

Depth sampling: a 7B-shaped model in fp32 on host cores is slow, so the port runs
``sample_layers`` decoder / ``sample_v_layers`` ViT layers at full width and charges the
time spent inside the layer loops scaled to the full depth; embedding, projector, final
norm and lm_head are charged once, as measured.  Migration copies are host memcpys of the
same bytes (timed).  Nothing here is on the product path.
"""

from __future__ import annotations

import time
from typing import Dict

import numpy as np
import torch

from .mllm_fp32 import OracleMLLM


class CpuPathExecutor:
    def __init__(self, shape, *, seed: int = 0, sample_layers: int = 2,
                 sample_v_layers: int = 2):
        import dataclasses
        from paper_2505_12658_b200.inputs import ImageStore
        from paper_2505_12658_b200.weights import weight_specs
        self.full = shape
        self.sample = dataclasses.replace(shape, n_layers=min(sample_layers, shape.n_layers),
                                          v_layers=min(sample_v_layers, shape.v_layers))
        self.lang_scale = shape.n_layers / self.sample.n_layers
        self.vit_scale = shape.v_layers / self.sample.v_layers
        self.seed = seed
        self.o = OracleMLLM.random_for_timing(self.sample.asdict(), weight_specs(self.sample),
                                              seed)
        self.images = ImageStore(seed, shape.patch)
        self.last_tok: Dict[str, int] = {}
        self.prompts: Dict[str, np.ndarray] = {}
        self.batches = 0
        self.busy_s = 0.0

    def _prompt(self, r):
        from paper_2505_12658_b200.inputs import prompt_tokens
        p = self.prompts.get(r.rid)
        if p is None:
            p = self.prompts[r.rid] = prompt_tokens(self.seed, r.rid, r.spec.prompt_tokens,
                                                    self.full.vocab)
        return p

    def batch_seconds(self, batch, reqs) -> float:
        """Execute one epdsim ``Batch`` (pre-batch cursors, engine.py:243-265) and return its
        full-depth CPU time.  Reads ``batch``/``reqs``; never mutates them."""
        o, s = self.o, self.full
        l0 = dict(o.layer_s)
        t0 = time.perf_counter()
        for rid, k, _counts in batch.encode_entries:
            r = reqs[rid]
            counts = r.spec.image_token_counts
            for ii in range(r.images_done, r.images_done + k):
                gh, gw = s.patch_grid(counts[ii])
                px = self.images.request_image(rid, ii, gh, gw)
                o.add_image_rows(rid, o.encode_image(px, gh, gw))
        for rid, kv_len in batch.decode_entries:
            lg = o.decode(rid, self.last_tok[rid], kv_len)
            self.last_tok[rid] = int(lg.argmax())
        for rid, c in batch.prefill_chunks:
            r = reqs[rid]
            lg = o.prefill_chunk(rid, self._prompt(r), r.plan.visual_tokens, r.prefill_done, c)
            if r.prefill_done + c >= r.plan.prefill_total_tokens:
                self.last_tok[rid] = int(lg.argmax())
                o.image_rows.pop(rid, None)
        wall = time.perf_counter() - t0
        dv = o.layer_s["vit"] - l0["vit"]
        dl = o.layer_s["lang"] - l0["lang"]
        sec = wall + (self.vit_scale - 1.0) * dv + (self.lang_scale - 1.0) * dl
        self.batches += 1
        self.busy_s += sec
        return sec

    def drop(self, rid: str) -> None:
        self.o.drop(rid)
        self.last_tok.pop(rid, None)
        self.prompts.pop(rid, None)


def replay_on_cpu(epdsim, spec, shape, hw, slo, trace, executor: CpuPathExecutor):
    """Measured-clock replay of ``trace`` through the unmodified reference ``Cluster`` with
    every batch executed by ``executor`` (bound at the cluster.py:295 seam for the duration
    of the call) and every migration charged the time of a host copy of its bytes."""
    C = epdsim.cluster
    MG = epdsim.migration
    orig = C.batch_latency
    orig_tx = MG.MigrationJob.transfer_seconds
    cache: Dict[str, float] = {}

    def lat(batch, reqs, _model, _hw):
        return executor.batch_seconds(batch, reqs)

    def tx(job, _hw):
        if job.rid not in cache:
            n = int(job.kv_bytes + job.image_bytes)
            a = torch.empty(n, dtype=torch.uint8)
            b = torch.empty_like(a)
            t0 = time.perf_counter()
            b.copy_(a)
            cache[job.rid] = time.perf_counter() - t0
        return cache[job.rid]

    C.batch_latency = lat
    MG.MigrationJob.transfer_seconds = tx
    try:
        cluster = C.Cluster(spec, shape.profile(), hw, slo)
        rep = cluster.run(trace)
    finally:
        C.batch_latency = orig
        MG.MigrationJob.transfer_seconds = orig_tx
    for rid in list(executor.last_tok):
        executor.drop(rid)
    return cluster, rep
