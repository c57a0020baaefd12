"""Live (wall-clock) serving of the LLaVA-1.5-7B TextCaps-shaped trace on one B200, next to
the measured-clock replay of the same trace (paper_2505_12658_b200/live.py).

    python tools/live_serving.py [--requests 600] [--rates 60,75,85] [--json out.json]

For each rate: SLO attainment, P90 TTFT / TBT and the wall span of the live run, and the
same figures from ``GpuCluster.run`` (device clock, one batch in flight at a time) on the
same trace.  Budgets are the measured ones (bench.py's default)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _summary(rep, span):
    a = rep.aggregates
    return {"attainment": a["slo_attainment"],
            "ttft_p90": a["ttft_percentiles_s"].get("p90"),
            "tbt_p90": a["tbt_percentiles_s"].get("p90"), "span_s": span}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=600)
    ap.add_argument("--rates", default="60,75,85")
    ap.add_argument("--json", default=None)
    ap.add_argument("--idle-sleep", type=float, default=1e-4, help="live loop poll sleep (s)")
    ap.add_argument("--live-only", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    from paper_2505_12658_b200.live import run_live
    shape = P.get_shape("llava-1.5-7b")
    slo = E.SloSpec(4.0, 0.08)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    out = []
    for rate in (float(x) for x in args.rates.split(",")):
        tr = E.synth_trace(seed=7, n_requests=args.requests, rate=rate, image_count_dist=1,
                           visual_token_choices=576, prompt_dist=[25, 35, 45],
                           output_dist=[90, 110, 130], slo=slo)
        row = {"rate": rate, "requests": args.requests}
        for mode in (("live",) if args.live_only else ("replay", "live")):
            cl = GpuCluster(spec, shape, P.b200_hardware(), slo, clock="device",
                            budgets="measured", resident_inputs=True)
            t0 = time.perf_counter()
            if mode == "live":
                rep = run_live(cl, tr, timeout_s=1800, idle_sleep_s=args.idle_sleep)
                span = time.perf_counter() - t0
            else:
                rep = cl.run(tr)
                span = max(r.token_times[-1] for r in cl.reqs.values() if r.token_times)
            torch.cuda.synchronize()
            row[mode] = _summary(rep, span)
            row[mode]["device_busy_s"] = sum(rt.stats["device_ms"] for rt in cl.runtimes.values()) / 1e3
            row[mode]["host_ms_per_batch"] = (sum(rt.stats["host_ms"] for rt in cl.runtimes.values()) /
                                              max(1, sum(rt.stats["batches"] for rt in cl.runtimes.values())))
            cl.close()
        out.append(row)
        print(json.dumps(row), flush=True)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
