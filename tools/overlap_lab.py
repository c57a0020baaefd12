"""Can decode attention (HBM-bound) run on the same SMs as a prefill GEMM (tensor-bound)?

    python tools/overlap_lab.py [--lib path/to/libhydra_variant.so]

Times, on one B200, a pair GEMM of a mixed batch's prefill rows (M x 12288 x 4096, the QKV
projection) and the paged decode attention of its decode rows (n seqs x ctx keys, 32 heads
x 128) -- each alone, then issued on two streams at once.  If the GEMM's CTAs leave enough
shared memory and registers for a decode-attention CTA per SM, the concurrent time drops
toward max(gemm, attention) instead of their sum.  Lab variants of the library with smaller
GEMM operand rings (compile-time HY_PAIR_SMEM_KB / HY_GEMM_SMEM_KB) are loaded with --lib.
Never a bench number.
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--M", type=int, default=3000)
    ap.add_argument("--seqs", type=int, default=400)
    ap.add_argument("--ctx", type=int, default=700)
    ap.add_argument("--bulk", default="0,0", help="decode kernel: nw,spw of the bulk kernel (0,0 = K8)")
    ap.add_argument("--co", action="store_true", help="co-resident decode kernel (K8c)")
    ap.add_argument("--delay", type=int, default=0,
                    help="spin cycles on the attention stream before its launch, so the GEMM's "
                    "CTAs are resident first")
    args = ap.parse_args()
    if args.lib:
        os.environ["HY_LIB_PATH"] = args.lib
    import torch
    from paper_2505_12658_b200 import _lib
    lib = _lib.load()
    nw, spw = (int(x) for x in args.bulk.split(","))
    assert lib.hy_set_decode_kernel(nw, spw) == 0, lib.hy_last_error()
    lib.hy_set_decode_coresident(1 if args.co else 0)
    dev = "cuda:0"
    M, N, K = args.M, 12288, 4096
    A = torch.randn(M, K, device=dev).bfloat16()
    W = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    e = _lib.HyGemmEpilogue(0, 0, 0, 0, 0, C.data_ptr(), N, 0)
    nh, d, L = 32, 128, 1
    n, ctx = args.seqs, args.ctx
    nbs = -(-ctx // 16)
    blk = L * 2 * nh * 16 * d
    kv = torch.randn(n * nbs + 1, blk, device=dev).bfloat16()
    bt = torch.randperm(n * nbs, device=dev).int().view(n, nbs)
    q = torch.randn(n, nh * d, device=dev).bfloat16()
    o = torch.empty_like(q)
    slots = torch.arange(n, dtype=torch.int32, device=dev)
    ctxs = torch.full((n,), ctx, dtype=torch.int32, device=dev)
    wsb = lib.hy_attn_decode_workspace_bytes(n, nh, d, ctx)
    dws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(dev)
    s2 = torch.cuda.Stream(dev)

    def gemm(s):
        rc = lib.hy_gemm_bf16(A.data_ptr(), K, W.data_ptr(), K, M, N, K, e, ws.data_ptr(),
                              ws.numel(), s.cuda_stream)
        assert rc == 0, lib.hy_last_error()

    def attn(s):
        rc = lib.hy_attn_decode_paged(q.data_ptr(), nh * d, n, nh, nh, d, slots.data_ptr(),
                                      ctxs.data_ptr(), ctx, bt.data_ptr(), nbs, kv.data_ptr(),
                                      blk, 1 / math.sqrt(d), o.data_ptr(), nh * d,
                                      dws.data_ptr(), dws.numel(), s.cuda_stream)
        assert rc == 0, lib.hy_last_error()

    def timed(fn, reps=20):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        gemm(s1)
        if args.delay:
            with torch.cuda.stream(s2):
                torch.cuda._sleep(args.delay)
        attn(s2)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    cur = torch.cuda.current_stream()
    tg = timed(lambda: gemm(cur))
    ta = timed(lambda: attn(cur))
    tb = timed(both)
    kv_bytes = n * ctx * 2 * nh * d * 2
    print(f"lib {os.path.basename(_lib.LIB_PATH)} bulk {args.bulk} co {int(args.co)} "
          f"slim {os.environ.get('HY_GEMM_SLIM', 0)} M={M}: gemm {tg:.1f} us "
          f"({2 * M * N * K / tg / 1e6:.0f} TF/s) | decode attn {n}x{ctx} {ta:.1f} us "
          f"({kv_bytes / ta / 1e3:.0f} GB/s) | both {tb:.1f} us (sum {tg + ta:.1f}, "
          f"max {max(tg, ta):.1f}, overlap {(tg + ta - tb) / min(tg, ta):.0%})", flush=True)


if __name__ == "__main__":
    main()
