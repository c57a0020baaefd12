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


def _largest_true(lo: int, hi: int, pred: Callable[[int], bool]) -> int:
    """Largest n in [lo, hi] with pred(n) for a monotone-decreasing predicate with
    pred(lo) true (restates engine.py:91-102)."""
    if pred(hi):
        return hi
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if pred(mid):
            lo = mid
        else:
            hi = mid
    return lo


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


def measured_budgets(cluster, probe_image_tokens: int = MC.IMAGE_BLOCK_TOKENS):
    """Re-run the reference budget search for every instance type of ``cluster`` with
    GPU-timed probes; installs and returns {InstanceType: BudgetPair}.  Results are cached
    per (model shape, device, instance type, caps) for the life of the process."""
    spec = cluster.spec
    out = {}
    for itype in cluster.type_budgets:
        key = (cluster.shape, str(cluster.runtimes[next(
            iid for iid, inst in cluster.instances.items() if inst.itype == itype)].device),
            itype.name, cluster.slo, spec.alpha, spec.vision_cap_share,
            spec.token_budget_ceiling, spec.image_budget_ceiling, probe_image_tokens)
        if key in _CACHE:
            out[itype] = _CACHE[key]
            continue
        rt = next(cluster.runtimes[iid] for iid, inst in cluster.instances.items()
                  if inst.itype == itype)
        pr = _Prober(rt, cluster.shape)
        cap = EN.derive_latency_cap(itype, cluster.slo, spec.alpha)
        has_language = itype.can_prefill or itype.can_decode
        has_encode = itype.can_encode
        both = has_language and has_encode
        token_cap = cap * (1.0 - spec.vision_cap_share) if both else cap
        vision_cap = cap * spec.vision_cap_share if both else cap
        feasible = True
        token_budget = 1
        if has_language:
            if pr.tokens(1) <= token_cap:
                token_budget = _largest_true(1, spec.token_budget_ceiling,
                                             lambda n: pr.tokens(n) <= token_cap)
            else:
                feasible = False
        image_budget = 0
        if has_encode:
            if pr.images(1, probe_image_tokens) <= vision_cap:
                image_budget = _largest_true(
                    1, spec.image_budget_ceiling,
                    lambda e: pr.images(e, probe_image_tokens) <= vision_cap)
            else:
                image_budget = 1
                feasible = False
        out[itype] = _CACHE[key] = EN.BudgetPair(token_budget, image_budget, feasible)
        rt.tok_records.clear()
        rt.tok_cursor = 0
        for k in rt.stats:
            rt.stats[k] = 0 if isinstance(rt.stats[k], int) else 0.0
    for inst in cluster.instances.values():
        inst.budgets = out[inst.itype]
    cluster.type_budgets = dict(out)
    return out
