"""Device time of mixed decode + prefill batches on the LLaVA-1.5-7B EPD instance, for A/B
comparisons of environment knobs read per call (e.g. HY_LANG_SPLIT=16).
    python tools/mixed_batch.py [--reps 7] [--variants 'HY_LANG_SPLIT=16;...']"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--variants", default="HY_LANG_SPLIT=16")
    ap.add_argument("--lib", default=None, help="lab build of the library (HY_LIB_PATH)")
    ap.add_argument("--mixes", default="64x700x512,128x700x1024,256x700x2048,128x300x2816",
                    help="decodes x context x prefill-chunk list")
    args = ap.parse_args()
    if args.lib:
        os.environ["HY_LIB_PATH"] = args.lib
    import paper_2505_12658_b200 as P
    from paper_2505_12658_b200._epdsim import C, E, EN, MC
    from paper_2505_12658_b200.budgets import _Prober
    from paper_2505_12658_b200.cluster import GpuCluster
    shape = P.get_shape("llava-1.5-7b")
    slo = E.SloSpec(4.0, 0.08)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"))
    cl = GpuCluster(spec, shape, P.b200_hardware(), slo, clock="device", budgets="roofline")
    rt = next(iter(cl.runtimes.values()))
    pr = _Prober(rt, shape, repeats=args.reps)
    pool = rt.kv_pool
    variants = [{}] + [dict(kv.split("=") for kv in v.split(","))
                       for v in filter(None, args.variants.split(";"))]
    mixes = [tuple(int(v) for v in m.split("x")) for m in args.mixes.split(",")]
    for nd, ctx, npf in mixes:
        reqs, entries = {}, []
        nblk = MC.kv_blocks_needed(ctx + 1)
        for i in range(nd):
            rid = f"__mix_d{i}"
            s = E.RequestSpec(rid, 0.0, (), ctx, 2, E.SloSpec(1.0, 1.0))
            r = EN.RequestState(spec=s, plan=E.plan_stages(s))
            r.stage = EN.DECODE
            pool.allocate(rid, nblk)
            reqs[rid] = r
            entries.append((rid, ctx))
        rid = "__mix_p"
        s = E.RequestSpec(rid, 0.0, (), npf, 2, E.SloSpec(1.0, 1.0))
        r = EN.RequestState(spec=s, plan=E.plan_stages(s))
        r.stage = EN.PREFILL
        pool.allocate(rid, MC.kv_blocks_needed(npf + 1))
        reqs[rid] = r
        batch = EN.Batch(decode_entries=entries, prefill_chunks=[(rid, npf)])
        out = []
        for v in variants:
            old = {k: os.environ.get(k) for k in v}
            os.environ.update(v)
            try:
                out.append((",".join(f"{k}={x}" for k, x in v.items()) or "default",
                            pr._time(batch, reqs) * 1e3))
            finally:
                for k, x in old.items():
                    if x is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = x
        print(f"decode {nd:4d} x ctx {ctx:4d} + prefill {npf:5d}: "
              + "  ".join(f"[{k}: {ms:.3f} ms]" for k, ms in out), flush=True)
        for rid in reqs:
            pool.release(rid)
            rt.forget(rid)


if __name__ == "__main__":
    main()
