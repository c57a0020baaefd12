#!/usr/bin/env python
"""bench.py -- HydraInfer serving hot path on B200 (BASELINE.json metric).

Metric: req/s at P90 TTFT+TPOT SLO (SLO attainment >= 0.9, metrics.py:57-68,214-262),
with decode tok/s and KV-migration GB/s reported beside it.

Workload: LLaVA-1.5-7B shape (CLIP ViT-L/14-336 + Llama-2-7B, random-init bf16) on a
TextCaps-shaped synthetic trace ``synth_trace(seed=7, 1 image x 576 tokens, prompt
{25,35,45}, output {90,110,130})`` (SURVEY.md 8d config 4 shape), SLO (4.0 s, 0.08 s),
``--requests`` requests per GPU (weak scaling).  The deployment follows the GPU count
(SURVEY.md 8e): N=1 colocated ``EPD:1`` (BASELINE config 2); N=2 ``EP:1,D:1``; N=4
``EP:2,D:2``; N=8 ``E:2,P:3,D:3`` (config 4) -- one instance per GPU, instance k on
``cuda:k`` in the reference's construction order (cluster.py:180-190), every EP / PD
migration a block copy pulled by the target GPU over NVLink (peer pointers).  One process
drives all N GPUs (the reference's scheduler is one event loop); under torchrun, rank 0
drives them and the other ranks only wait.

One "step" = one goodput probe: a full replay of the trace, scaled to the probe rate,
through the reference scheduler (epdsim) with every batch executed on the GPU(s) and the
virtual clock advanced by each batch's CUDA-event time (inputs resident in HBM).  K steps
= K geometric-bisection probes of ``find_goodput`` (metrics.py:214-262); W warm-up
replays precede them.  ``value`` = the largest probed rate with attainment >= 0.9.

e2e: the same metric through the same public API with the images copied from pinned host
memory every batch, the new tokens read back every batch, and each batch's latency the
host wall time of the whole call.  live: the asynchronous wall-clock server (live.py) at
the found rate and below.

--impl reference: the reference's CPU implementation of the path on the host cores -- the
unmodified reference scheduler (epdsim) with each batch executed by the fp32 CPU port
(oracle/cpu_executor.py, depth-sampled) on a bounded sample of the same trace; one step =
one measured-clock goodput probe, same metric, unit, config and SLO as our arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "req/s at P90 TTFT+TPOT SLO on 8×B200; decode tok/s; KV-migration GB/s"
UNIT = "req/s"
# the deployment for each GPU count
METHOD_BY_N = {1: "EPD:1", 2: "EP:1,D:1", 4: "EP:2,D:2", 8: "E:2,P:3,D:3"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6, help="goodput bisection probes")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llava-1.5-7b")
    ap.add_argument("--method", default=None,
                    help="deployment; default by GPU count: " + json.dumps(METHOD_BY_N))
    ap.add_argument("--devices", default=None,
                    help="comma list of CUDA device indices, one per GPU slot (default "
                         "0..N-1); repeating an index co-locates instances (functional tests)")
    # >= 30 s of arrivals at the goodput rate, so a burst cannot drain inside the
    # 4 s TTFT bound and pass a rate the GPU cannot sustain (finite-trace artifact, BASELINE.md
    # 2): 2,400 requests = 34 s at 71 req/s (1,500 gave 18 s at 84 req/s, with the device busy
    # 24 s -- a backlog the 4 s TTFT allowance absorbed)
    ap.add_argument("--requests", type=int, default=2400, help="trace requests per GPU")
    ap.add_argument("--rate-lo", type=float, default=16.0, help="per-GPU req/s")
    ap.add_argument("--rate-hi", type=float, default=128.0, help="per-GPU req/s")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-live", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=3,
                    help="requests of the trace the CPU port replays per step")
    ap.add_argument("--trace", default="textcaps", choices=sorted(TRACES))
    ap.add_argument("--emulate-link-gbs", type=float, default=770.0,
                    help="with co-located GPU slots (--devices 0,0,...), charge each migration "
                         "max(measured copy, bytes / this link bandwidth) (measured NVLink peer "
                         "copy, B200_PROFILING.md)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--budgets", default="measured", choices=["measured", "roofline"],
                    help="per-batch token/image budgets: reference search over GPU-timed "
                         "probes (SURVEY 8f f2) or over the reference roofline")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def log(msg):
    print(f"[bench] {msg}", file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


TRACES = {
    # BASELINE configs 2 / 4: TextCaps-shaped, one 576-token image (LLaVA)
    "textcaps": dict(seed=7, image_count_dist=1, visual_token_choices=576,
                     prompt_dist=[25, 35, 45], output_dist=[90, 110, 130], slo=(4.0, 0.08),
                     desc="TextCaps-shaped synth_trace(seed=7): 1 image x 576 tokens, "
                          "prompt {25,35,45}, output {90,110,130}; SLO TTFT 4 s / TBT 0.08 s"),
    # BASELINE config 3: dynamic-resolution images (Qwen2-VL), SLO qwen2-vl-7b/textcaps
    "dynres": dict(seed=11, image_count_dist=1, visual_token_choices=[256, 576, 1024, 1600, 2916],
                   prompt_dist=[25, 35, 45], output_dist=[90, 110, 130], slo=(8.0, 0.10),
                   desc="dynamic-resolution synth_trace(seed=11): 1 image x {256,576,1024,1600,"
                        "2916} tokens, prompt {25,35,45}, output {90,110,130}; SLO TTFT 8 s / "
                        "TBT 0.10 s (presets.py:55)"),
}
TRACE = "textcaps"


def base_trace(E, n, seed=None):
    t = TRACES[TRACE]
    slo = E.SloSpec(*t["slo"])
    return E.synth_trace(seed=t["seed"] if seed is None else seed, n_requests=n, rate=1.0,
                         image_count_dist=t["image_count_dist"],
                         visual_token_choices=t["visual_token_choices"],
                         prompt_dist=t["prompt_dist"], output_dist=t["output_dist"], slo=slo,
                         name=TRACE), slo


def n_gpus(args, d) -> int:
    return d.world if d.world > 1 else args.gpus


def method_for(args, n: int) -> str:
    return args.method or METHOD_BY_N.get(n, f"EPD:{n}")


def workload_config(args, n: int) -> dict:
    """The workload both arms run (identical dict in both JSON lines)."""
    method = method_for(args, n)
    return {"workload": f"{args.model} shape, {method} on {n} GPU(s), "
                        f"{TRACES[args.trace]['desc']} (P90 attainment)",
            "model": args.model, "method": method, "trace": args.trace,
            "requests": args.requests * n,
            "requests_per_gpu": args.requests,
            "rate_bounds_per_gpu": [args.rate_lo, args.rate_hi],
            "parallelism": (f"disaggregated {method}: one instance per GPU, EP/PD migrations "
                            "as NVLink block copies" if n > 1 else "colocated EPD:1"),
            "l2": "inputs larger than L2: 14 GB weights + paged KV streamed per step"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices):
        self.indices = sorted(set(indices))
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(map(str, self.indices)), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s, p in zip(sm, power) if p > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "samples_under_load": len(loaded),
                "power_w_max": max(power) if power else None}


class Dist:
    """torchrun plumbing (gloo, scalars only).  The serving cluster is one event loop, so
    rank 0 drives every GPU and the other ranks wait for it at a barrier."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            import datetime
            import torch.distributed as dist
            dist.init_process_group("gloo", timeout=datetime.timedelta(hours=3))
            self.dist = dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def geometric_bisect(probe, lo, hi, steps, threshold=0.9):
    """find_goodput (metrics.py:214-262) with a geometric midpoint and a fixed probe
    count; returns (rate, probes).  Every probe is one timed step."""
    probes = []
    best = None
    for _ in range(steps):
        mid = math.sqrt(lo * hi)
        att = probe(mid)
        probes.append((mid, att))
        if att >= threshold:
            lo, best = mid, mid
        else:
            hi = mid
    return best, probes


def attainment(P, rep) -> float:
    return sum(1 for m in rep.requests if P.epdsim.meets_slo(m)) / max(1, len(rep.requests))


# ----------------------------------------------------------------------------- ours
def run_ours(args, d: Dist):
    import torch
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200 import _lib
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    from paper_2505_12658_b200.live import run_live
    from paper_2505_12658_b200.profiling import KernelSampler
    from paper_2505_12658_b200.weights import DeviceWeights

    n = n_gpus(args, d)
    cfg = workload_config(args, n)
    if d.rank != 0:  # rank 0 drives all N GPUs (one scheduler event loop)
        d.barrier()
        return
    idx = ([int(x) for x in args.devices.split(",")] if args.devices else list(range(n)))
    if len(idx) != n:
        raise SystemExit(f"--devices lists {len(idx)} slots for {n} GPUs")
    if max(idx) >= torch.cuda.device_count():
        raise SystemExit(f"{n} GPU slots need devices {idx}; this box has "
                         f"{torch.cuda.device_count()}")
    devs = [torch.device("cuda", i) for i in idx]
    phys = sorted(set(idx))
    dev0 = devs[0]
    torch.cuda.set_device(dev0)
    peaks, peak_src = measured_peaks()
    shape = P.get_shape(args.model)
    hw = P.b200_hardware()
    # co-located instances (repeated --devices entries) split the device's memory; the
    # reference's pool accounting (pool_capacities, cluster.py:127-144) is then given the
    # same per-instance share, so every block it admits exists physically
    share = max(idx.count(i) for i in phys)
    pool_limit = None if share == 1 else int(130e9 / share / 1.1)
    emulated = share > 1 and n > 1  # several GPU slots on one device (see GpuCluster)
    if share > 1:
        hw = P.b200_hardware(gpu_memory_bytes=hw.model_weight_bytes + pool_limit)
    method = cfg["method"]
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(method))
    n_inst = sum(c for _, c in spec.method.counts)
    if n_inst != n:
        log(f"note: {method} has {n_inst} instances on {n} GPU slots (round-robin)")
    lib = _lib.load()
    weights = {torch.device("cuda", i): DeviceWeights(shape, torch.device("cuda", i), args.seed)
               for i in phys}
    base, slo = base_trace(E, args.requests * n)
    sampler = KernelSampler(dev0, every=4)
    budgets_seen = {}

    def replay(rate_total, clock="device", resident=True, sample=False, trace=None,
               live=False):
        tr = E.scale_to_rate(trace or base, rate_total)
        cl = GpuCluster(spec, shape, hw, slo, devices=devs, clock=clock, seed=args.seed,
                        resident_inputs=resident, weights=weights, budgets=args.budgets,
                        pool_bytes_limit=pool_limit,
                        emulated_link_gbs=args.emulate_link_gbs if emulated else None)
        budgets_seen.update({t.name: [b.token_budget, b.image_budget]
                             for t, b in cl.type_budgets.items()})
        if sample:
            for rt in cl.runtimes.values():
                if rt.device == dev0:
                    rt.sampler = sampler
        rep = run_live(cl, tr, timeout_s=1800) if live else cl.run(tr)
        return cl, rep

    def mig_summary(cl):
        ts = cl.transfer_stats
        out = {"count": ts["count"], "bytes": ts["bytes"], "copied_bytes": ts["copied_bytes"],
               "seconds": ts["seconds"],
               "gbs": ts["copied_bytes"] / ts["seconds"] / 1e9 if ts["seconds"] > 0 else None}
        for kind in ("ep", "pd"):
            k = ts.get(kind)
            if k:
                out[kind] = dict(k, gbs=k["bytes"] / k["seconds"] / 1e9 if k["seconds"] else None)
        return out

    # ---- warm-up (untimed): short replays exercise every kernel shape class
    warm = E.Trace(base.requests[:24 * n], name="warm")
    for i in range(args.warmup):
        replay(50.0 * n * (i + 1), trace=warm)[0].close()
    for dv in phys:
        torch.cuda.synchronize(dv)
    log(f"warm-up done; {method} on devices {idx}; budgets {budgets_seen}")

    # ---- timed goodput search: K probes
    probe_info = []
    clocks = ClockSampler(phys)
    launches0 = lib.hy_launch_count()
    for dv in phys:
        torch.cuda.synchronize(dv)
    clocks.start()
    t_all0 = time.perf_counter()

    def probe(rate_per_gpu):
        total = rate_per_gpu * n
        t0 = time.perf_counter()
        cl, rep = replay(total, sample=True)
        for dv in phys:
            torch.cuda.synchronize(dv)
        dt = time.perf_counter() - t0
        a = rep.aggregates
        att = attainment(P, rep)
        span = (max(s.t_done for s in cl.reqs.values()) -
                min(s.spec.arrival_time for s in cl.reqs.values()))
        tokens = sum(r.tokens_out for r in cl.reqs.values())
        probe_info.append({
            "rate": total, "attainment": att, "wall_s": dt, "virtual_span_s": span,
            "tokens": tokens, "decode_tok_s": tokens / span if span > 0 else 0.0,
            "device_busy_s": sum(rt.stats["device_ms"] for rt in cl.runtimes.values()) / 1e3,
            "batches": sum(rt.stats["batches"] for rt in cl.runtimes.values()),
            "vision_critical": [sum(rt.stats["vision_critical"] for rt in cl.runtimes.values()),
                                sum(rt.stats["mixed_batches"] for rt in cl.runtimes.values())],
            "ttft_p90": a["ttft_percentiles_s"].get("p90"),
            "tbt_p90": a["tbt_percentiles_s"].get("p90"),
            "migration": mig_summary(cl) if cl.transfer_stats["count"] else None})
        cl.close()
        log(f"probe rate {total:.1f}: attainment {att:.3f}, {probe_info[-1]['batches']} "
            f"batches, wall {dt:.1f} s")
        return att

    best, probes = geometric_bisect(probe, args.rate_lo, args.rate_hi, args.steps)
    for dv in phys:
        torch.cuda.synchronize(dv)
    t_all = time.perf_counter() - t_all0
    clk = clocks.stop()
    launches = int(lib.hy_launch_count() - launches0)
    value = (best or 0.0) * n
    best_probe = max((p for p in probe_info if p["attainment"] >= 0.9),
                     key=lambda p: p["rate"], default=None)

    # ---- roofline of the dominant kernel, timed live inside the probes
    summ = sampler.summary()
    dominant = max(summ, key=lambda k: summ[k]["share_of_batch_time"]) if summ else None

    def traffic_of(name):
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                return json.load(fh).get(name)
        except OSError:
            return None

    def roof(name):
        s = summ[name]
        if name == "decode_attn":
            ach = s["work_per_ms"] / 1e6  # bytes/ms -> GB/s
            return {"kernel": "attn_decode_kernel (K8)", "bound": "hbm", "achieved": ach,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                    "traffic": traffic_of("decode_attn"), "launches_timed": s["launches"],
                    "avg_launch_ms": s["avg_ms"], "share_of_step": s["share_of_batch_time"],
                    "peak_source": f"{peak_src} hbm_gbs",
                    # batches without vision work (no cross-stream contention)
                    "solo_achieved": s["solo_work_per_ms"] / 1e6, "solo_launches": s["solo_launches"]}
        ach = s["work_per_ms"] / 1e9  # flop/ms -> TFLOP/s
        pk = peaks["bf16_tflops_sustained"]
        busy = s["work_per_union_ms"] / 1e9
        return {"kernel": {"gemm": "gemm_tc_kernel + gemm_pair_kernel (K1, tcgen05)",
                           "prefill_attn": "attn_tc_kernel<128,paged> (K7, tcgen05)",
                           "vit_attn": "attn_tc_kernel<64,varlen> (K3, tcgen05)"}[name],
                "bound": "tensor", "achieved": ach, "peak": pk, "unit": "TFLOP/s",
                "frac": ach / pk, "traffic": traffic_of(name), "launches_timed": s["launches"],
                "avg_launch_ms": s["avg_ms"], "share_of_step": s["share_of_batch_time"],
                "peak_source": f"{peak_src} bf16_tflops_sustained",
                # the same flops over the time any launch of the class was running (the V and
                # L streams overlap their kernels; per-launch durations count that time twice)
                "achieved_over_busy_time": busy, "frac_over_busy_time": busy / pk,
                "solo_achieved": s["solo_work_per_ms"] / 1e9, "solo_launches": s["solo_launches"]}

    roofline = roof(dominant) if dominant else None
    if roofline is not None and dominant == "gemm":
        roofline["by_shape"] = sampler.gemm_breakdown()
    others = {k: roof(k) for k in summ if k != dominant}

    # ---- end-to-end through host buffers (wall clock per batch)
    e2e = None
    if not args.no_e2e and best:
        e2e_rate = None
        e2e_probes = []
        img_bytes = shape.patch_grid(576)[0] * shape.patch_grid(576)[1] * shape.patch ** 2 * 3
        n_img = n_tok = 0
        for f in (1.0, 0.96, 0.92, 0.88, 0.8, 0.6):
            r = best * n * f
            cl, rep = replay(r, clock="wall", resident=False)
            att = attainment(P, rep)
            e2e_probes.append((r, att))
            log(f"e2e probe rate {r:.1f}: attainment {att:.3f}")
            n_img = sum(rt.stats["images"] for rt in cl.runtimes.values())
            n_tok = sum(r_.tokens_out for r_ in cl.reqs.values())
            cl.close()
            if att >= 0.9:
                e2e_rate = r
                break
        e2e = {"value": e2e_rate or 0.0, "unit": UNIT,
               "h2d_bytes_per_step": None, "d2h_bytes_per_step": None, "probes": e2e_probes,
               "clock": "host wall time per batch (lowering + H2D pixels + GPU + D2H tokens)"}
        if e2e_rate:
            # a step is one replay; bytes are this replay's pixel uploads and token
            # read-backs (int32 per generated token)
            e2e["h2d_bytes_per_step"] = n_img * img_bytes
            e2e["d2h_bytes_per_step"] = n_tok * 4

    # ---- live asynchronous serving (live.py): wall-clock arrivals, concurrent instances
    live = None
    if emulated and not args.no_live:
        # co-located GPU slots share one device in wall-clock time: a live run would measure
        # that contention, not N GPUs (the replay times each batch alone instead)
        live = {"skipped": "emulated GPU slots share one device in wall-clock time"}
    elif not args.no_live and best:
        lp = []
        live_rate = None
        for f in (1.0, 0.9, 0.8):
            r = best * n * f
            cl, rep = replay(r, live=True)
            att = attainment(P, rep)
            a = rep.aggregates
            lp.append({"rate": r, "attainment": att, "ttft_p90": a["ttft_percentiles_s"].get("p90"),
                       "tbt_p90": a["tbt_percentiles_s"].get("p90")})
            log(f"live probe rate {r:.1f}: attainment {att:.3f}")
            cl.close()
            if att >= 0.9:
                live_rate = r
                break
        live = {"value": live_rate or 0.0, "unit": UNIT, "probes": lp,
                "clock": "wall clock; arrivals in real time; batches asynchronous on the V/L "
                         "streams; migrations complete on their copy events"}

    # ---- KV-block migration copy (K10) at the config-5 payload; NVLink pairs when N > 1
    mig = kv_migration_probe(devs, shape, peaks)

    # ---- CPU baseline: the reference's CPU implementation of the path (bounded sample)
    cpu = None
    if n == 1 and not args.no_cpu_baseline:
        cpu = cpu_path_probe(args, shape, base, slo, spec, args.rate_lo)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_all * 1e3 / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, synthetic pixels/prompt ids)",
        "config": cfg,
        "arm": {"executor": "libhydra_sm100.so (sm_100a) under the reference scheduler",
                "devices": idx,
                "emulated_gpus": (f"{n} GPU slots co-located on {len(phys)} device(s): each "
                                  "batch is timed alone on the device (one batch in flight in "
                                  "the replay), migrations charged max(measured copy, bytes / "
                                  f"{args.emulate_link_gbs:g} GB/s); each slot has "
                                  f"{hw.gpu_memory_bytes / 1e9:.0f} GB (weights + its pool "
                                  "share) in the reference's pool accounting")
                if emulated else None,
                "clock": "virtual clock advanced by the CUDA-event time of each batch",
                "budgets": {"mode": args.budgets, "tau_t_tau_e": budgets_seen}},
        "decode_tok_s": best_probe["decode_tok_s"] if best_probe else 0.0,
        "kv_migration_gbs": mig.get("gbs") if mig else None,
        "kv_migration": mig,
        "serving_migrations": best_probe["migration"] if best_probe else None,
        "probes": probe_info,
        "roofline": roofline, "roofline_other_kernels": others,
        "cpu_baseline": cpu, "e2e": e2e, "live": live, "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line))
    d.barrier()


def kv_migration_probe(devs, shape, peaks, n_blocks=869, valid_tail=7, reps=5):
    """The prefill->decode KV migration copy (migration.py:63-64) at the config-5 payload:
    869 KV blocks (8 MiB each for LLaVA-7B; the multi-image stress trace's largest job,
    SURVEY.md 8d) with shuffled block ids and a 7-token tail (token-exact,
    hy_copy_blocks_tail).  One GPU: HBM -> HBM on cuda:k.  Two or more physical GPUs: pairs
    (0->1), (2->3), ... pull concurrently over NVLink through peer pointers (1, 2, 4 pairs),
    next to NCCL's broadcast of the same gathered payload (the send/recv baseline)."""
    import numpy as np
    import torch
    from paper_2505_12658_b200 import _lib
    lib = _lib.load()
    bb = shape.kv_block_elems * 2  # bf16
    grp = 16 * shape.head_dim * 2
    tail = valid_tail * shape.head_dim * 2
    payload = (n_blocks - 1) * bb + (bb // grp) * tail
    phys = sorted({d.index for d in devs})
    rng = np.random.default_rng(0)
    perm_s = rng.permutation(n_blocks).astype(np.int32)
    perm_d = rng.permutation(n_blocks).astype(np.int32)

    def timed(fns, streams):
        for f in fns:
            f()
        for s in streams:
            s.synchronize()
        ts = []
        for _ in range(reps):
            evs = []
            for f, s in zip(fns, streams):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(s.device):
                    a.record(s)
                    f()
                    b.record(s)
                evs.append((a, b))
            for _, b in evs:
                b.synchronize()
            ts.append(max(a.elapsed_time(b) for a, b in evs))  # max over pairs
        return statistics.median(ts)

    out = {"unit": "GB/s of token-exact payload (job.kv_bytes) per copy", "blocks": n_blocks,
           "block_bytes": bb, "payload_bytes": payload}
    try:
        d0 = torch.device("cuda", phys[0])
        src = torch.empty(n_blocks * bb, dtype=torch.uint8, device=d0)
        dst = torch.empty_like(src)
        sid = torch.from_numpy(perm_s).to(d0)
        did = torch.from_numpy(perm_d).to(d0)
        st = torch.cuda.current_stream(d0)

        def once():
            _lib.check(lib.hy_copy_blocks_tail(src.data_ptr(), dst.data_ptr(), sid.data_ptr(),
                                               did.data_ptr(), n_blocks, bb, grp, tail,
                                               st.cuda_stream), "hy_copy_blocks_tail")
        t = timed([once], [st])
        t_ref = timed([lambda: dst.copy_(src)], [st])
        gbs = payload / t / 1e6
        out.update({"gbs": gbs, "ms": t, "path": f"same-device HBM->HBM on cuda:{phys[0]}",
                    "hbm_achieved_gbs": 2 * gbs, "hbm_peak_gbs": peaks["hbm_gbs"],
                    "hbm_frac": 2 * gbs / peaks["hbm_gbs"],
                    "contiguous_memcpy_gbs": n_blocks * bb / t_ref / 1e6})
        del src, dst
        torch.cuda.empty_cache()
        log(f"kv migration copy: {gbs:.0f} GB/s payload ({2 * gbs:.0f} GB/s HBM)")
    except Exception as e:  # noqa: BLE001  (reported, never fatal to the bench line)
        out["error"] = f"{type(e).__name__}: {e}"[:300]
    if len(phys) >= 2:
        out["nvlink"] = nvlink_pairs(phys, n_blocks, bb, grp, tail, payload, perm_s, perm_d,
                                     timed)
        best = max((r for r in out["nvlink"] if r.get("p2p_gbs")),
                   key=lambda r: r["pairs"], default=None)
        if best:
            out["gbs"] = best["p2p_gbs"]
            out["path"] = (f"cross-GPU pull over NVLink, {best['pairs']} concurrent pair(s): the "
                           "destination GPU's copy kernel reads the source pool through a "
                           "peer pointer")
    return out


def nvlink_pairs(phys, n_blocks, bb, grp, tail, payload, perm_s, perm_d, timed):
    """P2P pull vs NCCL for 1, 2, 4 concurrent GPU pairs (max time over pairs)."""
    import torch
    from paper_2505_12658_b200 import _lib
    lib = _lib.load()
    rows = []
    max_pairs = len(phys) // 2
    for pairs in (1, 2, 4):
        if pairs > max_pairs:
            break
        row = {"pairs": pairs}
        try:
            bufs = []
            for p in range(pairs):
                s_dev = torch.device("cuda", phys[2 * p])
                d_dev = torch.device("cuda", phys[2 * p + 1])
                _lib.check(lib.hy_enable_peer_access(d_dev.index, s_dev.index), "peer")
                src = torch.empty(n_blocks * bb, dtype=torch.uint8, device=s_dev).random_(0, 255)
                dst = torch.empty(n_blocks * bb, dtype=torch.uint8, device=d_dev)
                sid = torch.from_numpy(perm_s).to(d_dev)
                did = torch.from_numpy(perm_d).to(d_dev)
                bufs.append((s_dev, d_dev, src, dst, sid, did))
            fns, sts = [], []
            for s_dev, d_dev, src, dst, sid, did in bufs:
                st = torch.cuda.current_stream(d_dev)

                def pull(src=src, dst=dst, sid=sid, did=did, st=st):
                    _lib.check(lib.hy_copy_blocks_tail(src.data_ptr(), dst.data_ptr(),
                                                       sid.data_ptr(), did.data_ptr(), n_blocks,
                                                       bb, grp, tail, st.cuda_stream),
                               "hy_copy_blocks_tail(peer)")
                fns.append(pull)
                sts.append(st)
            t = timed(fns, sts)
            row.update({"p2p_ms": t, "p2p_gbs": payload / t / 1e6,
                        "p2p_aggregate_gbs": pairs * payload / t / 1e6})
            # NCCL baseline: gather on the source, broadcast (send/recv), scatter on the target
            try:
                import torch.cuda.nccl as nccl
                seqs = {}
                for s_dev, d_dev, src, dst, sid, did in bufs:
                    seqs[s_dev.index] = torch.arange(n_blocks, dtype=torch.int32, device=s_dev)
                    seqs[d_dev.index] = torch.arange(n_blocks, dtype=torch.int32, device=d_dev)
                stage = [(torch.empty(payload, dtype=torch.uint8, device=s_dev),
                          torch.empty(payload, dtype=torch.uint8, device=d_dev))
                         for s_dev, d_dev, *_ in bufs]
                t0 = time.perf_counter()
                for r in range(reps + 1):
                    if r == 1:
                        for s_dev, d_dev, *_ in bufs:
                            torch.cuda.synchronize(s_dev)
                            torch.cuda.synchronize(d_dev)
                        t0 = time.perf_counter()
                    for (s_dev, d_dev, src, dst, sid, did), (a, b) in zip(bufs, stage):
                        with torch.cuda.device(s_dev):
                            _lib.check(lib.hy_copy_blocks_tail(
                                src.data_ptr(), a.data_ptr(), sid.data_ptr(),
                                seqs[s_dev.index].data_ptr(), n_blocks, bb, grp, tail,
                                torch.cuda.current_stream(s_dev).cuda_stream), "gather")
                    for a, b in stage:
                        nccl.broadcast([a, b], root=0)
                    for (s_dev, d_dev, src, dst, sid, did), (a, b) in zip(bufs, stage):
                        with torch.cuda.device(d_dev):
                            _lib.check(lib.hy_copy_blocks_tail(
                                b.data_ptr(), dst.data_ptr(), seqs[d_dev.index].data_ptr(),
                                did.data_ptr(), n_blocks, bb, grp, tail,
                                torch.cuda.current_stream(d_dev).cuda_stream), "scatter")
                for s_dev, d_dev, *_ in bufs:
                    torch.cuda.synchronize(s_dev)
                    torch.cuda.synchronize(d_dev)
                t_n = (time.perf_counter() - t0) / reps * 1e3
                row.update({"nccl_ms": t_n, "nccl_gbs": payload / t_n / 1e6,
                            "nccl_clock": "host wall time per round (synchronised)"})
            except Exception as e:  # noqa: BLE001
                row["nccl_error"] = f"{type(e).__name__}: {e}"[:200]
            del bufs
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001
            row["p2p_error"] = f"{type(e).__name__}: {e}"[:200]
        rows.append(row)
        log(f"nvlink migration: {row}")
    return rows


def cpu_path_probe(args, shape, base, slo, spec, rate_per_gpu):
    """One measured-clock replay of the first ``--cpu-sample`` requests of the trace (at
    the trace's rate scaled to ``rate_per_gpu``) through the unmodified reference
    scheduler, every batch executed by the fp32 CPU port on all host cores."""
    import torch
    from oracle.cpu_executor import CpuPathExecutor, replay_on_cpu
    from paper_2505_12658_b200._epdsim import E
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    ex = CpuPathExecutor(shape, seed=args.seed)
    hw = E.HardwareProfile(2.25e15, 8.0e12, 160e9, 14e9, 900e9)
    tr = E.scale_to_rate(E.Trace(base.requests[:args.cpu_sample], name="cpu_sample"),
                         rate_per_gpu)
    t0 = time.perf_counter()
    _cl, rep = replay_on_cpu(E, spec, shape, hw, slo, tr, ex)
    wall = time.perf_counter() - t0
    att = sum(1 for m in rep.requests if E.meets_slo(m)) / len(rep.requests)
    a = rep.aggregates
    span = max(r.t_done for r in _cl.reqs.values()) - min(
        r.spec.arrival_time for r in _cl.reqs.values())
    return {"value": rate_per_gpu if att >= 0.9 else 0.0, "unit": UNIT, "cores": cores,
            "kind": "port", "attainment": att, "probe_rate": rate_per_gpu,
            "throughput_rps": len(tr.requests) / span if span > 0 else 0.0,
            "ttft_p90": a["ttft_percentiles_s"].get("p90"),
            "tbt_p90": a["tbt_percentiles_s"].get("p90"),
            "decode_tok_s": sum(r.tokens_out for r in _cl.reqs.values()) / span if span else 0,
            "batches": ex.batches, "wall_s": wall,
            "sample": (f"first {len(tr.requests)} requests of the same trace at "
                       f"{rate_per_gpu:g} req/s through the unmodified epdsim scheduler; "
                       f"batches executed by oracle/cpu_executor (fp32 port, "
                       f"{ex.sample.n_layers}/{shape.n_layers} decoder + "
                       f"{ex.sample.v_layers}/{shape.v_layers} ViT layers at full width, "
                       "layer time scaled to full depth), measured-clock")}


# ----------------------------------------------------------------------------- reference
def analytic_reference(args, method, shape_name, slo_trace):
    """The reference's own model of the path -- epdsim's analytic batch_latency /
    transfer_seconds on a B200 HardwareProfile built from the measured peaks -- searched for
    goodput on the same trace.  A simulated ideal (perfect compute/memory overlap), reported
    for context only; it executes no model."""
    from paper_2505_12658_b200._epdsim import C, E
    peaks, src = measured_peaks()
    hw = E.HardwareProfile(peaks["bf16_tflops_sustained"] * 1e12, peaks["hbm_gbs"] * 1e9,
                           160e9, 14e9, 770e9)
    model = E.MODEL_PRESETS[shape_name] if shape_name in E.MODEL_PRESETS else None
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(method))
    base, slo = slo_trace
    t0 = time.perf_counter()

    def probe(rate):
        rep = C.run_trace(spec, model, hw, slo, E.scale_to_rate(base, rate))
        return sum(1 for m in rep.requests if E.meets_slo(m)) / len(rep.requests)

    best, _ = geometric_bisect(probe, args.rate_lo, 4 * args.rate_hi, 8)
    return {"goodput_rps": best, "wall_s": time.perf_counter() - t0,
            "executor": f"epdsim analytic roofline, B200 profile from {src} peaks (simulated)"}


def run_reference(args, d: Dist):
    """--impl reference: the reference's CPU implementation of the path, timed on this box's
    host cores.  The reference scheduler (epdsim, unmodified) forms every batch of the same
    trace; each batch is executed by the fp32 CPU port (oracle/cpu_executor.py) on all host
    threads and charged its measured time (measured-clock replay, the reference's
    batch_latency seam).  A step is one goodput probe over a bounded sample (the first
    ``--cpu-sample`` requests of the trace), bisecting the same per-GPU rate range as our
    arm; ``value`` is the largest probed rate meeting the SLO (0 when none does)."""
    if d.rank != 0:
        return
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    n = n_gpus(args, d)
    cfg = workload_config(args, n)
    shape = P.get_shape(args.model)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(cfg["method"]))
    base, slo = base_trace(E, args.requests * n)
    for _ in range(args.warmup):
        cpu_path_probe(args, shape, base, slo, spec, args.rate_lo * n)
    samples = []
    t0 = time.perf_counter()

    def probe(rate):
        r = cpu_path_probe(args, shape, base, slo, spec, rate * n)
        samples.append(r)
        log(f"reference probe {rate * n:.1f} req/s: attainment {r['attainment']:.3f}, "
            f"ttft p90 {r['ttft_p90']}")
        return r["attainment"]

    best, _ = geometric_bisect(probe, args.rate_lo, args.rate_hi, args.steps)
    dt = time.perf_counter() - t0
    value = (best or 0.0) * n
    last = samples[-1]
    analytic = analytic_reference(args, cfg["method"], args.model, base_trace(E, args.requests * n))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, synthetic pixels/prompt ids)",
            "impl": "reference", "config": cfg,
            "arm": {"executor": "unmodified epdsim scheduler + oracle/cpu_executor (fp32 CPU "
                                "port of the path), all host threads",
                    "clock": "measured-clock replay (CPU time of each batch)"},
            "probes": [{k: s_[k] for k in ("probe_rate", "attainment", "ttft_p90", "tbt_p90",
                                           "throughput_rps", "wall_s")} for s_ in samples],
            "decode_tok_s": last["decode_tok_s"], "throughput_rps": last["throughput_rps"],
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "port",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "analytic_epdsim": analytic}
    print(json.dumps(line))


def main():
    global TRACE
    args = parse()
    TRACE = args.trace
    d = Dist()
    try:
        if args.impl == "reference":
            run_reference(args, d)
        else:
            run_ours(args, d)
    finally:
        d.close()


if __name__ == "__main__":
    main()
