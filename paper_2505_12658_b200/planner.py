"""Algorithm 2 on measured stage speeds.

The reference's offline disaggregation profiler (``plan_partition``, profiler.py:167-177)
summarises a trace, searches per-stage batch budgets under the SLO
(``stage_budgets``, profiler.py:86-112), converts them to stage throughputs
(``estimate_throughputs``, profiler.py:115-127), and splits N instances proportionally to the
stage times (``partition``, profiler.py:142-164), from which ``candidate_methods``
(profiler.py:180-191) builds the E+P+D, EP+D and ED+P deployments.  Every latency in that
pipeline comes from the analytic roofline.

``measured_plan_partition`` runs the same pipeline with the three latency probes supplied by
the caller -- on hardware, GPU-timed batches of this executor (``gpu_stage_timers``): a
prefill chunk of n tokens, an encode of e images, a decode step of n requests at the
workload's mean context.  With the roofline as the timer it reproduces the reference's
``plan_partition`` exactly (tests/test_planner.py), so the only difference on hardware is
where the seconds come from.  The budget searches keep the reference's caps (alpha / beta
shares of the TTFT bound for encode / prefill, the TBT bound for decode), its
largest-true bisection and its memory cap on decode concurrency.
"""

from __future__ import annotations

from typing import Callable, Tuple

from ._epdsim import EN, MC, E

TimeFn = Callable[..., float]


_largest_true = EN._largest_true  # the reference's own bisection (engine.py:91-102)


def measured_stage_budgets(slo, model, hw, summary, t_prefill: TimeFn, t_encode: TimeFn,
                           alpha: float = 0.5, beta: float = 0.5, gamma: float = 0.9,
                           ceilings: Tuple[int, int] = (EN.DEFAULT_TOKEN_CEILING,
                                                        EN.DEFAULT_IMAGE_CEILING)
                           ) -> Tuple[int, int, int]:
    """(tau_e images, tau_p tokens, tau_d tokens) as in profiler.stage_budgets, with the
    reference's single-tower ``search_budgets`` probes replaced by ``t_encode(e, T)`` and
    ``t_prefill(n)`` (seconds)."""
    P = _profiler()
    token_ceiling, image_ceiling = ceilings
    T = max(1, round(summary.avg_image_tokens))

    def tokens_budget(cap: float) -> int:
        if t_prefill(1) > cap:
            return 1  # the reference's floor budget (infeasible flag is not used here)
        return _largest_true(1, token_ceiling, lambda n: t_prefill(n) <= cap)

    if t_encode(1, T) <= alpha * slo.ttft_max:
        tau_e = _largest_true(1, image_ceiling, lambda e: t_encode(e, T) <= alpha * slo.ttft_max)
    else:
        tau_e = 1
    tau_p = tokens_budget(beta * slo.ttft_max)
    tau_d = tokens_budget(slo.tbt_max)
    mem_cap = P.decode_concurrency_cap(summary, model, hw, gamma)
    if mem_cap < 1:
        raise P.ProfilerError(f"decode memory infeasible: concurrency cap {mem_cap} < 1")
    return tau_e, tau_p, min(tau_d, mem_cap)


def measured_plan_partition(trace, N: int, slo, model, hw, t_prefill: TimeFn,
                            t_encode: TimeFn, t_decode: TimeFn):
    """profiler.plan_partition with measured probes; returns the reference PartitionResult.
    ``t_decode(n, ctx)`` times one decode step of n requests at context ctx."""
    P = _profiler()
    summary = P.summarize_workload(trace)
    tau_e, tau_p, tau_d = measured_stage_budgets(slo, model, hw, summary, t_prefill, t_encode)
    T = max(1, round(summary.avg_image_tokens))
    ctx = max(1, round(summary.avg_context_tokens))
    tp_e = tau_e * T / t_encode(tau_e, T) if tau_e > 0 else 0.0
    tp_p = tau_p / t_prefill(tau_p)
    tp_d = tau_d / t_decode(tau_d, ctx)
    t_e = summary.W_e / tp_e if tp_e > 0 else 0.0
    t_p = summary.W_p / tp_p
    t_d = summary.W_d / tp_d
    N_e, N_p, N_d = P.partition(N, t_e, t_p, t_d)
    return P.PartitionResult(N_e, N_p, N_d, t_e, t_p, t_d, tp_e, tp_p, tp_d)


def roofline_timers(model, hw):
    """The reference's analytic latencies as timer callables (parity tests, CPU)."""
    def t_prefill(n: int) -> float:
        return MC.roofline_latency(MC.language_work([n], [], model), hw)

    def t_encode(e: int, T: int) -> float:
        return MC.roofline_latency(MC.vision_work([T] * e, model), hw)

    def t_decode(n: int, ctx: int) -> float:
        return MC.roofline_latency(MC.language_work([], [ctx] * n, model), hw)
    return t_prefill, t_encode, t_decode


def gpu_stage_timers(runtime, shape, repeats: int = 3):
    """Timer callables backed by GPU-timed batches on ``runtime`` (an InstanceRuntime whose
    instance can prefill, encode and decode -- e.g. the EPD instance of a GpuCluster).  The
    decode probe allocates n requests of ctx cached tokens in the instance's KV pool."""
    from .budgets import _Prober
    pr = _Prober(runtime, shape, repeats=repeats)
    cache = {}

    def t_decode(n: int, ctx: int) -> float:
        key = (n, ctx)
        if key in cache:
            return cache[key]
        pool = runtime.kv_pool
        nblk = MC.kv_blocks_needed(ctx + 1)
        n = max(1, min(n, (pool.free_blocks // nblk) if nblk else n))
        reqs, entries = {}, []
        for i in range(n):
            rid = f"__probe_d{i}"
            spec = E.RequestSpec(rid, 0.0, (), ctx, 2, E.SloSpec(1.0, 1.0))
            r = EN.RequestState(spec=spec, plan=E.plan_stages(spec))
            r.stage = EN.DECODE
            pool.allocate(rid, nblk)
            reqs[rid] = r
            entries.append((rid, ctx))
        try:
            cache[key] = pr._time(EN.Batch(decode_entries=entries), reqs) * (key[0] / n)
        finally:
            for rid in reqs:
                pool.release(rid)
                runtime.forget(rid)
        return cache[key]

    return pr.tokens, pr.images, t_decode


def _profiler():
    import epdsim.profiler as P  # the reference package is already on sys.path (._epdsim)
    return P


def measured_select_method(trace, N: int, slo, model, hw, goodput_of: Callable,
                           timers=None):
    """profiler.select_method (profiler.py:242-270) on measured quantities: Algorithm 2's
    partition from the measured stage speeds (``timers`` = (t_prefill, t_encode,
    t_decode); the roofline when None), the three candidate deployments of that partition
    (``candidate_methods``, profiler.py:180-191), each scored by ``goodput_of(method)`` --
    on hardware, the replayed goodput of the deployment on N GPUs -- and the argmax with
    the reference's tie rule (first in candidate order).  Returns the reference's
    ``SelectionResult``."""
    P = _profiler()
    t_prefill, t_encode, t_decode = timers or roofline_timers(model, hw)
    plan = measured_plan_partition(trace, N, slo, model, hw, t_prefill, t_encode, t_decode)
    candidates = P.candidate_methods(plan.N_e, plan.N_p, plan.N_d)
    table = tuple((m, goodput_of(m)) for m in candidates)
    if all(g == 0.0 for _, g in table):
        rows = "; ".join(f"{m.label}: goodput 0" for m, _ in table)
        raise P.ProfilerError(f"all candidate methods infeasible ({rows})")
    best = max(g for _, g in table)
    first = next(m for m, g in table if g == best)
    return P.SelectionResult(best=first, table=table, partition=plan)
