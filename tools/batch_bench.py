"""Device time of single batches on the LLaVA-1.5-7B EPD instance (budget-probe batches):
a prefill chunk of n tokens and an encode of e images.  For A/B comparisons of kernel
changes without the serving-loop noise.   python tools/batch_bench.py [--reps 7]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.budgets import _Prober
    from paper_2505_12658_b200.cluster import GpuCluster
    shape = P.get_shape("llava-1.5-7b")
    slo = E.SloSpec(4.0, 0.08)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    cl = GpuCluster(spec, shape, P.b200_hardware(), slo, clock="device", budgets="roofline")
    rt = next(iter(cl.runtimes.values()))
    pr = _Prober(rt, shape, repeats=args.reps)
    for n in (512, 1024, 2048, 2560, 2816, 4096):
        ms = pr.tokens(n) * 1e3
        print(f"prefill {n:5d} tokens: {ms:7.2f} ms  ({n / ms:6.0f} tok/ms)", flush=True)
    for e in (1, 8, 32, 64):
        ms = pr.images(e, 576) * 1e3
        print(f"encode  {e:5d} images: {ms:7.2f} ms", flush=True)
    cl.close()


if __name__ == "__main__":
    main()
