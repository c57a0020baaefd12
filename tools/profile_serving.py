"""Short LLaVA-1.5-7B serving replay for ncu captures (profiles/).

    python tools/profile_serving.py [--requests 48] [--rate 60]

Runs the same path as bench.py (epdsim scheduler + GPU executor, device clock) on a short
TextCaps-shaped trace, so `ncu --metrics gpu__time_duration.sum` gives the launch list
of a real serving mix and `ncu --set full -k regex:<kernel>` captures representative
launches.  Never a source of bench numbers (ncu serialises and replays kernels).
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=48)
    ap.add_argument("--rate", type=float, default=60.0)
    ap.add_argument("--model", default="llava-1.5-7b")
    ap.add_argument("--trace", default="textcaps", choices=["textcaps", "dynres"],
                    help="dynres: bench.py's Qwen2-VL dynamic-resolution trace (config 3)")
    ap.add_argument("--budgets", default="roofline", choices=["roofline", "measured"])
    ap.add_argument("--clock", default="device", choices=["device", "wall"])
    ap.add_argument("--watchdog", type=float, default=0.0,
                    help="dump Python stacks and exit after this many seconds (hang triage)")
    args = ap.parse_args()
    if args.watchdog:
        import faulthandler
        faulthandler.dump_traceback_later(args.watchdog, exit=True)
    import torch
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    shape = P.get_shape(args.model)
    if args.trace == "dynres":
        slo = E.SloSpec(8.0, 0.10)
        tr = E.synth_trace(seed=11, n_requests=args.requests, rate=args.rate, image_count_dist=1,
                           visual_token_choices=[256, 576, 1024, 1600, 2916],
                           prompt_dist=[25, 35, 45], output_dist=[90, 110, 130], slo=slo)
    else:
        slo = E.SloSpec(4.0, 0.08)
        tr = E.synth_trace(seed=7, n_requests=args.requests, rate=args.rate, image_count_dist=1,
                           visual_token_choices=576, prompt_dist=[25, 35, 45],
                           output_dist=[90, 110, 130], slo=slo)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    cl = GpuCluster(spec, shape, P.b200_hardware(), slo, clock=args.clock,
                    budgets=args.budgets, resident_inputs=args.clock == "device")
    rep = cl.run(tr)
    torch.cuda.synchronize()
    rt = next(iter(cl.runtimes.values()))
    nb = max(1, rt.stats["batches"])
    print("batches", rt.stats["batches"], "device_ms", round(rt.stats["device_ms"], 1),
          "attainment", rep.aggregates["slo_attainment"], "vision_critical",
          rt.stats["vision_critical"], "of mixed", rt.stats["mixed_batches"])
    print("per batch ms: device %.2f host %.2f prep(lang lowering) %.2f lang-launch-done %.2f"
          % (rt.stats["device_ms"] / nb, rt.stats["host_ms"] / nb, rt.stats["prep_ms"] / nb,
             rt.stats["launch_ms"] / nb))


if __name__ == "__main__":
    main()
