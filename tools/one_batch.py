"""Run one prefill batch of n tokens (single request) on the LLaVA EPD instance -- for ncu
launch lists of the budget-probe batch.   python tools/one_batch.py [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2816
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.budgets import _Prober
    from paper_2505_12658_b200.cluster import GpuCluster
    shape = P.get_shape("llava-1.5-7b")
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    cl = GpuCluster(spec, shape, P.b200_hardware(), E.SloSpec(4.0, 0.08), clock="device",
                    budgets="roofline")
    rt = next(iter(cl.runtimes.values()))
    pr = _Prober(rt, shape, repeats=reps)
    print(f"prefill {n}: {pr.tokens(n) * 1e3:.2f} ms")
    cl.close()


if __name__ == "__main__":
    main()
