"""Algorithm 2 (the reference's disaggregation planner) on GPU-measured stage speeds.

    python tools/plan_disaggregation.py [--model llava-1.5-7b] [--N 2 4 8]

Times prefill / encode / decode probe batches on one B200 (the EPD instance of a GpuCluster),
runs planner.measured_plan_partition, and prints it beside the reference's roofline plan
(epdsim.profiler.plan_partition) and the three candidate deployments for each cluster size
(the replayed-goodput selection over candidates needs N GPUs)."""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llava-1.5-7b")
    ap.add_argument("--N", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import paper_2505_12658_b200 as H  # puts the reference package on sys.path
    import epdsim.profiler as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    from paper_2505_12658_b200.planner import gpu_stage_timers, measured_plan_partition
    shape = H.get_shape(args.model)
    hw = H.b200_hardware()
    slo = E.SloSpec(4.0, 0.08)
    tr = E.synth_trace(seed=7, n_requests=400, rate=4.0, image_count_dist=1,
                       visual_token_choices=576, prompt_dist=[25, 35, 45],
                       output_dist=[90, 110, 130], slo=slo)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    cl = GpuCluster(spec, shape, hw, slo, clock="device", budgets="roofline")
    rt = next(iter(cl.runtimes.values()))
    timers = gpu_stage_timers(rt, shape)
    out = {}
    for N in args.N:
        if N < 3:
            continue
        ref = P.plan_partition(tr, N, slo, shape.profile(), hw)
        got = measured_plan_partition(tr, N, slo, shape.profile(), hw, *timers)
        out[N] = {"roofline": ref.__dict__, "measured": got.__dict__,
                  "candidates_measured": [m.label for m in P.candidate_methods(
                      got.N_e, got.N_p, got.N_d)]}
        print(f"N={N}: roofline E/P/D = {ref.N_e}/{ref.N_p}/{ref.N_d} "
              f"(tp tok/s e {ref.tp_e:.0f} p {ref.tp_p:.0f} d {ref.tp_d:.0f}); "
              f"measured E/P/D = {got.N_e}/{got.N_p}/{got.N_d} "
              f"(tp e {got.tp_e:.0f} p {got.tp_p:.0f} d {got.tp_d:.0f}); candidates "
              f"{out[N]['candidates_measured']}", flush=True)
    cl.close()
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
