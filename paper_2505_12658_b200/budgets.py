"""Measured-probe budget search.

The reference sizes each instance type's per-batch token budget tau_t and image budget
tau_e by binary search against a latency cap, probing its roofline model
(``search_budgets``, engine.py:105-153; caps from ``derive_latency_cap``, engine.py:70-77;
per type via ``budgets_for_type``, cluster.py:147-158).  The roofline assumes 2.25 PF/s
and 8 TB/s with no launch, norm or lm_head cost, so on real hardware its budgets produce
batches that overrun the cap (and the TBT SLO).

``measured_budgets`` keeps the reference's search -- same caps, same 50/50 split of the
cap between the towers of a mixed instance, same monotone largest-true bisection over
[1, ceiling] -- but each probe is a real batch executed on the instance's GPU (a single
prefill chunk of n tokens, or e encode images of 576 tokens), timed with CUDA events.
The paper profiles the same way at initialisation.
"""

from __future__ import annotations

import statistics
from typing import Callable, Dict

from ._epdsim import EN, MC, E


_largest_true = EN._largest_true  # the reference's own bisection (engine.py:91-102)


class RooflineProber:
    """The reference's analytic probe latencies (engine.py:128-132): with this prober
    ``search_with_prober`` reproduces ``search_budgets`` exactly (tests/test_planner.py)."""

    def __init__(self, model, hw):
        self.model, self.hw = model, hw

    def tokens(self, n: int) -> float:
        return MC.roofline_latency(MC.language_work([n], [], self.model), self.hw)

    def images(self, e: int, tokens: int) -> float:
        return MC.roofline_latency(MC.vision_work([tokens] * e, self.model), self.hw)


def search_with_prober(itype, slo, spec, prober, token_prober=None,
                       probe_image_tokens: int = MC.IMAGE_BLOCK_TOKENS):
    """``budgets_for_type`` (cluster.py:147-158) -> ``search_budgets`` (engine.py:105-153)
    with the probe latencies supplied by ``prober`` (``tokens(n)``, ``images(e, T)``): the
    same cap (``derive_latency_cap``), the same 50/50 split of the cap between the towers
    of a mixed instance, the same largest-true bisection over [1, ceiling], the same floor
    budgets and feasibility flags.  ``token_prober`` (default ``prober``) answers the
    token probes; instances without a language tower still run the reference's token
    search, whose result their batches never use."""
    tp = token_prober or prober
    cap = EN.derive_latency_cap(itype, slo, spec.alpha)
    if cap <= 0:
        raise ValueError("cap must be > 0")
    has_language = itype.can_prefill or itype.can_decode
    has_encode = itype.can_encode
    both = has_language and has_encode
    token_cap = cap * (1.0 - spec.vision_cap_share) if both else cap
    vision_cap = cap * spec.vision_cap_share if both else cap
    feasible = True
    if tp.tokens(1) <= token_cap:
        token_budget = _largest_true(1, spec.token_budget_ceiling,
                                     lambda n: tp.tokens(n) <= token_cap)
    else:
        token_budget = 1
        if has_language:
            feasible = False
    image_budget = 0
    if has_encode:
        if prober.images(1, probe_image_tokens) <= vision_cap:
            image_budget = _largest_true(
                1, spec.image_budget_ceiling,
                lambda e: prober.images(e, probe_image_tokens) <= vision_cap)
        else:
            image_budget = 1
            feasible = False
    return EN.BudgetPair(token_budget, image_budget, feasible)


class _Prober:
    def __init__(self, rt, shape, repeats: int = 5):
        self.rt = rt
        self.shape = shape
        self.repeats = repeats
        self.cache: Dict = {}
        self.n = 0

    def _time(self, batch, reqs) -> float:
        self.rt.run_batch(batch, reqs, "device")  # warm (workspace growth, I-cache)
        ts = [self.rt.run_batch(batch, reqs, "device") for _ in range(self.repeats)]
        return statistics.median(ts)

    def tokens(self, n: int) -> float:
        key = ("t", n)
        if key not in self.cache:
            self.n += 1
            rid = f"__probe_t{self.n}"
            spec = E.RequestSpec(rid, 0.0, (), n, 2, E.SloSpec(1.0, 1.0))
            r = EN.RequestState(spec=spec, plan=E.plan_stages(spec))
            r.stage = EN.PREFILL
            pool = self.rt.kv_pool
            pool.allocate(rid, MC.kv_blocks_needed(n))
            try:
                self.cache[key] = self._time(EN.Batch(prefill_chunks=[(rid, n)]), {rid: r})
            finally:
                pool.release(rid)
                self.rt.forget(rid)
        return self.cache[key]

    def images(self, e: int, tokens: int) -> float:
        key = ("e", e, tokens)
        if key not in self.cache:
            self.n += 1
            rid = f"__probe_e{self.n}"
            counts = (tokens,) * e
            spec = E.RequestSpec(rid, 0.0, counts, 1, 2, E.SloSpec(1.0, 1.0))
            r = EN.RequestState(spec=spec, plan=E.plan_stages(spec))
            pool = self.rt.image_pool
            pool.allocate(rid, MC.image_blocks_needed(tokens * e))
            try:
                self.cache[key] = self._time(
                    EN.Batch(encode_entries=[(rid, e, counts)]), {rid: r})
            finally:
                pool.release(rid)
        return self.cache[key]


_CACHE: Dict = {}


def measured_budgets(cluster, probe_image_tokens: int = MC.IMAGE_BLOCK_TOKENS,
                     prober_factory: Callable = None):
    """Re-run the reference budget search for every instance type of ``cluster`` with
    probes from ``prober_factory(runtime, shape)`` -- by default GPU-timed batches on an
    instance of that type (``_Prober``); instances without a language tower answer the
    (unused) token probes from the roofline, as the reference computes them.  Installs and
    returns {InstanceType: BudgetPair}.  GPU results are cached per (model shape, device,
    instance type, caps) for the life of the process."""
    spec = cluster.spec
    factory = prober_factory or (lambda rt, shape: _Prober(rt, shape))
    roof = RooflineProber(cluster.model, cluster.hw)
    out = {}
    for itype in cluster.type_budgets:
        rt = next(cluster.runtimes[iid] for iid, inst in cluster.instances.items()
                  if inst.itype == itype)
        key = (cluster.shape, str(rt.device), itype.name, cluster.slo, spec.alpha,
               spec.vision_cap_share, spec.token_budget_ceiling, spec.image_budget_ceiling,
               probe_image_tokens)
        cache = prober_factory is None
        if cache and key in _CACHE:
            out[itype] = _CACHE[key]
            continue
        pr = factory(rt, cluster.shape)
        has_language = itype.can_prefill or itype.can_decode
        out[itype] = search_with_prober(itype, cluster.slo, spec, pr,
                                        token_prober=pr if has_language else roof,
                                        probe_image_tokens=probe_image_tokens)
        if cache:
            _CACHE[key] = out[itype]
        if isinstance(pr, _Prober):  # the probes ran real batches: reset the counters
            rt.tok_records.clear()
            rt.tok_cursor = 0
            for k in rt.stats:
                rt.stats[k] = 0 if isinstance(rt.stats[k], int) else 0.0
    for inst in cluster.instances.values():
        inst.budgets = out[inst.itype]
    cluster.type_budgets = dict(out)
    return out
