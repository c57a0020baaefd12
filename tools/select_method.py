"""Algorithm 2 + replayed-goodput selection on hardware.

    python tools/select_method.py [--model qwen2-vl-7b] [--trace dynres] [--N 3]
                                  [--requests-per-gpu 300] [--probes 4] [--json out.json]

1. Stage speeds measured on one B200 (planner.gpu_stage_timers on an EPD instance: a prefill
   chunk of n tokens, an encode of e images, a decode step of n requests) feed the
   reference's partition (profiler.plan_partition restated by measured_plan_partition).
2. The three candidate deployments of that partition (profiler.candidate_methods: E+P+D,
   EP+D, ED+P) are each replayed on N GPU slots -- co-located on this one B200 (bench.py's
   emulated slots: each batch timed alone, migrations charged max(copy, bytes / 770 GB/s),
   each slot's pool accounting sized to its memory share) -- and scored by goodput
   (geometric bisection, attainment >= 0.9).
3. measured_select_method returns the argmax with the reference's tie rule.
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2-vl-7b")
    ap.add_argument("--trace", default="dynres")
    ap.add_argument("--N", type=int, default=3)
    ap.add_argument("--requests-per-gpu", type=int, default=300)
    ap.add_argument("--probes", type=int, default=4)
    ap.add_argument("--rate-lo", type=float, default=4.0, help="per GPU")
    ap.add_argument("--rate-hi", type=float, default=64.0, help="per GPU")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    from paper_2505_12658_b200.planner import gpu_stage_timers, measured_select_method
    from paper_2505_12658_b200.weights import DeviceWeights
    bench.TRACE = args.trace
    N = args.N
    shape = P.get_shape(args.model)
    model = shape.profile()
    dev = torch.device("cuda", 0)
    weights = {dev: DeviceWeights(shape, dev, 0)}
    base, slo = bench.base_trace(E, args.requests_per_gpu * N)
    pool_limit = int(130e9 / N / 1.1)
    hw_slot = P.b200_hardware(gpu_memory_bytes=14e9 + pool_limit)
    hw_full = P.b200_hardware()
    t0 = time.time()
    # (1) measured stage speeds on a full-memory EPD instance
    epd = GpuCluster(C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1")), shape,
                     hw_full, slo, devices=[dev], clock="device", weights=weights)
    timers = gpu_stage_timers(next(iter(epd.runtimes.values())), shape)
    log = []

    def goodput_of(method):
        spec = C.ClusterSpec(method=method)
        lo, hi, best = args.rate_lo, args.rate_hi, 0.0
        probes = []
        for _ in range(args.probes):
            mid = math.sqrt(lo * hi)
            cl = GpuCluster(spec, shape, hw_slot, slo, devices=[dev] * N, clock="device",
                            weights=weights, pool_bytes_limit=pool_limit,
                            budgets="measured", emulated_link_gbs=770.0)
            rep = cl.run(E.scale_to_rate(base, mid * N))
            att = sum(1 for m in rep.requests if E.meets_slo(m)) / len(rep.requests)
            probes.append((mid * N, att, cl.transfer_stats["count"]))
            cl.close()
            if att >= 0.9:
                lo, best = mid, mid * N
            else:
                hi = mid
        log.append({"method": method.label, "goodput_rps": best, "probes": probes})
        print(json.dumps(log[-1]), flush=True)
        return best

    sel = measured_select_method(base, N, slo, model, hw_slot, goodput_of, timers=timers)
    p = sel.partition
    out = {"model": args.model, "trace": args.trace, "N": N,
           "partition": {"N_e": p.N_e, "N_p": p.N_p, "N_d": p.N_d, "tp_e_tok_s": p.tp_e,
                         "tp_p_tok_s": p.tp_p, "tp_d_tok_s": p.tp_d},
           "candidates": log, "selected": sel.best.label,
           "slots": f"{N} GPU slots co-located on one B200 (bench.py emulated slots)",
           "wall_s": time.time() - t0}
    print(json.dumps(out), flush=True)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
