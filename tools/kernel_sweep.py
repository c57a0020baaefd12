"""Per-shape microbenchmarks of the serving kernels (LLaVA-1.5-7B shapes) on one B200.

    python tools/kernel_sweep.py [--what gemm,attn,copy] [--json out.json]

GEMM: hy_gemm_bf16 vs torch.matmul (cuBLAS) on the decoder / ViT / projector shapes
the serving mix produces (decode M 1..256, mixed prefill M ~ tau_t, ViT M = 577 x images).
Every timing: CUDA events on the launching stream, warm-up first, median of repeats,
and the weights rotated through a set larger than L2 so each launch streams from HBM.
Attention: decode (K8), paged prefill (K7), ViT varlen (K3) at serving shapes, reported
as GB/s (decode) or TFLOP/s (4*d*keys per head).  Copy: hy_copy_blocks on 8 MiB KV blocks
(same device; the peer-pointer path needs two GPUs).
Never a source of bench numbers; it explains them.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

DEV = "cuda:0"


def lib():
    return _lib.load()


def st():
    return torch.cuda.current_stream().cuda_stream


def timeit(fn, reps=5, per_graph=20, warm=3):
    """GPU time per launch: `per_graph` launches captured in one CUDA graph (no host
    launch overhead in the measurement), replayed `reps` times, median."""
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(per_graph):
                fn(i)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    cur = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        g.replay()
        b.record(cur)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / per_graph)
    ts.sort()
    return ts[len(ts) // 2]


VARIANTS = []
RESIDUAL = []
ONLY = []
EXTRA = []


def gemm_sweep(out):
    H, F, V = 4096, 11008, 32000
    shapes = []
    for M in (1, 16, 64, 128, 256, 512, 1024, 1600, 2304, 4096):
        shapes += [("qkv", M, 3 * H, H), ("o", M, H, H), ("gate_up", M, 2 * F, H),
                   ("down", M, H, F)]
    shapes += [("lm_head", 64, V, H), ("lm_head", 256, V, H)]
    for n_img in (1, 2, 3, 8, 56):
        T = 577 * n_img
        shapes += [("vit_qkv", T, 3072, 1024), ("vit_o", T, 1024, 1024),
                   ("vit_fc1", T, 4096, 1024), ("vit_fc2", T, 1024, 4096),
                   ("proj1", 576 * n_img, 4096, 1024), ("proj2", 576 * n_img, 4096, 4096)]
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=DEV)
    shapes += EXTRA
    if ONLY:
        shapes = [x for x in shapes if x[0] in ONLY]
    for name, M, N, K in shapes:
        nw = max(2, int(400e6 // (N * K * 2)) + 1)  # > L2 of weights in rotation
        Ws = [torch.randn(N, K, device=DEV).mul_(0.02).bfloat16() for _ in range(nw)]
        A = torch.randn(M, K, device=DEV).bfloat16()
        C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
        # in-place residual (the serving o / down projections: x += GEMM) when --residual
        # names this shape; x rotates through buffers larger than L2 like the weights
        if name in RESIDUAL or "all" in RESIDUAL:
            R = torch.randn(M, N, device=DEV).bfloat16()
            e = _lib.HyGemmEpilogue(0, R.data_ptr(), N, 0, 0, R.data_ptr(), N, 0)
        else:
            e = _lib.HyGemmEpilogue(0, 0, 0, 0, 0, C.data_ptr(), N, 0)

        def ours(i):
            W = Ws[i % nw]
            rc = lib().hy_gemm_bf16(A.data_ptr(), K, W.data_ptr(), K, M, N, K, e,
                                    ws.data_ptr(), ws.numel(), st())
            assert rc == 0, lib().hy_last_error()

        def cublas(i):
            torch.matmul(A, Ws[i % nw].t(), out=C)

        t0 = timeit(ours)
        t1 = timeit(cublas)
        var = {}
        for v in VARIANTS:
            old = {k: os.environ.get(k) for k in v}
            os.environ.update(v)
            try:
                var[",".join(f"{k}={x}" for k, x in v.items())] = timeit(ours) * 1e3
            except AssertionError:
                pass
            for k, x in old.items():
                if x is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = x
        fl = 2.0 * M * N * K
        wb = N * K * 2 + M * K * 2 + M * N * 2
        r = {"name": name, "M": M, "N": N, "K": K, "ours_us": t0 * 1e3, "cublas_us": t1 * 1e3,
             "ours_tflops": fl / t0 / 1e9, "cublas_tflops": fl / t1 / 1e9,
             "ours_gbs": wb / t0 / 1e6, "speedup_vs_cublas": t1 / t0, "variants_us": var}
        out.append(r)
        print(f"{name:8s} M={M:6d} N={N:6d} K={K:6d}  ours {t0*1e3:8.1f} us "
              f"{r['ours_tflops']:7.1f} TF {r['ours_gbs']:7.0f} GB/s | cublas {t1*1e3:8.1f} us "
              f"{r['cublas_tflops']:7.1f} TF | x{r['speedup_vs_cublas']:.2f} "
              + " ".join(f"[{k}: {x:.1f}]" for k, x in var.items()), flush=True)
        del Ws


def attn_sweep(out):
    """ViT varlen (K3) and paged prefill (K7) attention vs flash_attn (library, reference
    speed only -- never on the product path)."""
    import math
    import numpy as np
    try:
        from flash_attn import flash_attn_varlen_func
    except Exception:  # noqa: BLE001
        flash_attn_varlen_func = None
    # ViT: n images x T tokens: LLaVA 16 heads x 64 (577 tokens), Qwen2-VL 16 heads x 80
    # (dynamic resolution)
    vit = ((1, 577, 64), (3, 577, 64), (8, 577, 64), (32, 577, 64), (1, 2916, 80),
           (4, 1024, 80), (8, 576, 80))
    if os.environ.get("ATTN_VIT_SHAPES"):  # "images/tokens/head_dim;..."
        vit = [tuple(int(v) for v in x.split("/")) for x in os.environ["ATTN_VIT_SHAPES"].split(";")]
    for n_img, T, d in vit:
        nh = 16
        tot = n_img * T
        qkv = torch.randn(tot, 3 * nh * d, device=DEV).bfloat16()
        o = torch.empty(tot, nh * d, device=DEV, dtype=torch.bfloat16)
        seg = torch.arange(0, tot + 1, T, dtype=torch.int32, device=DEV)

        def ours(i):
            rc = lib().hy_attn_varlen(qkv.data_ptr(), 3 * nh * d, tot, n_img, seg.data_ptr(), T, nh, d,
                                      1 / math.sqrt(d), o.data_ptr(), nh * d, st())
            assert rc == 0, lib().hy_last_error()
        t0 = timeit(ours)
        t1 = None
        if flash_attn_varlen_func is not None:
            q3 = qkv.view(tot, 3, nh, d)
            q, k, v = q3[:, 0], q3[:, 1], q3[:, 2]

            def fa(i):
                flash_attn_varlen_func(q, k, v, seg, seg, T, T)
            t1 = timeit(fa)
        fl = 4.0 * d * nh * n_img * T * T
        r = {"name": "vit_attn", "images": n_img, "T": T, "d": d, "ours_us": t0 * 1e3,
             "ours_tflops": fl / t0 / 1e9, "fa_us": t1 * 1e3 if t1 else None,
             "fa_tflops": fl / t1 / 1e9 if t1 else None}
        out.append(r)
        print(f"vit_attn images={n_img:3d} x {T:4d} d={d}  ours {t0*1e3:8.1f} us {r['ours_tflops']:7.1f} TF | "
              f"flash_attn {r['fa_us'] or 0:8.1f} us {r['fa_tflops'] or 0:7.1f} TF", flush=True)
    # prefill: chunks (offset, len) over paged KV, 32 heads x 128
    for chunks in ([(0, 616)], [(0, 616)] * 4, [(0, 1024), (1024, 1024)], [(0, 2304)]):
        nh, d = 32, 128
        n = len(chunks)
        ctxs = [a + b for a, b in chunks]
        nblk = [-(-c // 16) for c in ctxs]
        block_elems = 2 * nh * 16 * d
        kv = torch.randn(sum(nblk) + 1, block_elems, device=DEV).bfloat16()
        bts = max(nblk)
        bt = torch.zeros(n, bts, dtype=torch.int32)
        u = 0
        for i, nb in enumerate(nblk):
            bt[i, :nb] = torch.arange(u, u + nb, dtype=torch.int32)
            u += nb
        bt = bt.to(DEV)
        rows = sum(c for _, c in chunks)
        q = torch.randn(rows, nh * d, device=DEV).bfloat16()
        o = torch.empty_like(q)
        qstart = torch.tensor(np.cumsum([0] + [c for _, c in chunks]), dtype=torch.int32,
                              device=DEV)
        offs = torch.tensor([a for a, _ in chunks], dtype=torch.int32, device=DEV)
        slots = torch.arange(n, dtype=torch.int32, device=DEV)
        mq = max(c for _, c in chunks)

        def ours(i):
            rc = lib().hy_attn_prefill_paged(q.data_ptr(), nh * d, rows, n, qstart.data_ptr(),
                                             offs.data_ptr(), slots.data_ptr(), mq, nh, nh, d,
                                             bt.data_ptr(), bts, kv.data_ptr(), block_elems,
                                             1 / math.sqrt(d), o.data_ptr(), nh * d, st())
            assert rc == 0, lib().hy_last_error()
        t0 = timeit(ours)
        keys = sum(c * a + c * (c + 1) // 2 for a, c in chunks)
        fl = 4.0 * d * nh * keys
        r = {"name": "prefill_attn", "chunks": chunks, "ours_us": t0 * 1e3,
             "ours_tflops": fl / t0 / 1e9}
        out.append(r)
        print(f"prefill_attn {chunks}  ours {t0*1e3:8.1f} us {r['ours_tflops']:7.1f} TF",
              flush=True)


def overlap_probe(out):
    """Can HBM-bound decode attention overlap tensor-bound prefill GEMMs on separate
    streams?  Times each alone and both concurrently (decode attention of 256 sequences x
    660 context, LLaVA 32x128 heads; gate_up GEMM 2304 x 22016 x 4096)."""
    import math
    n, ctx, nh, d = 256, 660, 32, 128
    nb = -(-ctx // 16)
    block_elems = 2 * nh * 16 * d  # one layer
    kv = torch.randn(n * nb + 1, block_elems, device=DEV).bfloat16()
    bt = torch.arange(n * nb, dtype=torch.int32, device=DEV).view(n, nb).contiguous()
    q = torch.randn(n, nh * d, device=DEV).bfloat16()
    o = torch.empty_like(q)
    slots = torch.arange(n, dtype=torch.int32, device=DEV)
    ctxs = torch.full((n,), ctx, dtype=torch.int32, device=DEV)
    wsb = lib().hy_attn_decode_workspace_bytes(n, nh, d, ctx)
    dws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=DEV)
    M, N, K = 2304, 22016, 4096
    A = torch.randn(M, K, device=DEV).bfloat16()
    W = (torch.randn(N, K, device=DEV) * 0.02).bfloat16()
    C = torch.empty(M, N // 2, device=DEV, dtype=torch.bfloat16)
    gws = torch.zeros(64 << 20, dtype=torch.uint8, device=DEV)
    e = _lib.HyGemmEpilogue(0, 0, 0, _lib.HY_ACT_SWIGLU, 0, C.data_ptr(), N // 2, 0)
    s_att = torch.cuda.Stream(priority=-1)
    s_gemm = torch.cuda.Stream()

    def att(stream):
        rc = lib().hy_attn_decode_paged(q.data_ptr(), nh * d, n, nh, nh, d, slots.data_ptr(),
                                        ctxs.data_ptr(), ctx, bt.data_ptr(), nb, kv.data_ptr(),
                                        block_elems, 1 / math.sqrt(d), o.data_ptr(), nh * d,
                                        dws.data_ptr(), dws.numel(), stream.cuda_stream)
        assert rc == 0, lib().hy_last_error()

    def gemm(stream):
        rc = lib().hy_gemm_bf16(A.data_ptr(), K, W.data_ptr(), K, M, N, K, e, gws.data_ptr(),
                                gws.numel(), stream.cuda_stream)
        assert rc == 0, lib().hy_last_error()

    def run(which, reps=20):
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        ev0.record(cur)
        s_att.wait_stream(cur)
        s_gemm.wait_stream(cur)
        for _ in range(reps):
            if "a" in which:
                att(s_att)
            if "g" in which:
                gemm(s_gemm)
        cur.wait_stream(s_att)
        cur.wait_stream(s_gemm)
        ev1.record(cur)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    for w in ("a", "g", "ag"):
        run(w, 3)
    ta, tg, tb = run("a"), run("g"), run("ag")
    r = {"name": "overlap", "attn_ms": ta, "gemm_ms": tg, "both_ms": tb,
         "sum_ms": ta + tg, "max_ms": max(ta, tg)}
    out.append(r)
    print(f"overlap: attn {ta:.3f} ms ({n * ctx * block_elems * 2 / ta / 1e9:.0f} GB/s), "
          f"gemm {tg:.3f} ms, concurrent {tb:.3f} ms (sum {ta + tg:.3f}, max {max(ta, tg):.3f})",
          flush=True)


def decode_sweep(out):
    """Paged decode attention (K8) bandwidth for MHA (LLaVA) and GQA (Qwen2-VL 28/4)."""
    import math
    shapes = ((32, 32, 256, 660, 0), (32, 32, 256, 660, 1), (32, 32, 128, 700, 1),
              (32, 32, 64, 700, 1), (32, 32, 32, 700, 1), (28, 4, 256, 660, 0),
              (28, 4, 64, 4000, 0), (32, 8, 256, 660, 0), (32, 32, 16, 8000, 0))
    if os.environ.get("DECODE_SHAPES"):  # "nh/nkv/seqs/ctx/shuffled;..." (ctx "lo-hi": random)
        shapes = [tuple(v if "-" in v else int(v) for v in x.split("/"))
                  for x in os.environ["DECODE_SHAPES"].split(";")]
    if os.environ.get("DECODE_CO"):
        lib().hy_set_decode_coresident(1)
    for nh, nkv, n, ctx, shuffled in shapes:
        d = 128
        if isinstance(ctx, str):  # per-sequence contexts drawn from [lo, hi]
            lo, hi = (int(v) for v in ctx.split("-"))
            cl = torch.randint(lo, hi + 1, (n,), generator=torch.Generator().manual_seed(0))
            ctx = int(cl.max())
        else:
            cl = torch.full((n,), ctx)
        nb = -(-ctx // 16)
        be = 2 * nkv * 16 * d
        # DECODE_POOL_GB: a serving-sized pool -- blocks of DECODE_LAYERS layers (block stride
        # = layers x the one-layer slice) scattered over that many GB, as in a 122 GB KV pool
        pool_gb = float(os.environ.get("DECODE_POOL_GB", "0"))
        layers = int(os.environ.get("DECODE_LAYERS", "1"))
        n_blk = n * nb + 1
        if pool_gb > 0:
            n_blk = max(n_blk, int(pool_gb * 1e9 // (be * layers * 2)))
            kv = torch.empty(n_blk, be * layers, device=DEV, dtype=torch.bfloat16)
            kv[:, :be].normal_()  # layer 0 (the one read) only
        else:
            kv = torch.randn(n_blk, be, device=DEV).bfloat16()
        # shuffled: blocks scattered over the pool as the free list hands them out in serving
        ids = (torch.randperm(n_blk - 1, device=DEV)[:n * nb] if shuffled
               else torch.arange(n * nb, device=DEV))
        bt = ids.to(torch.int32).view(n, nb).contiguous()
        be = be * layers if pool_gb > 0 else be
        q = torch.randn(n, nh * d, device=DEV).bfloat16()
        o = torch.empty_like(q)
        slots = torch.arange(n, dtype=torch.int32, device=DEV)
        ctxs = cl.to(torch.int32).to(DEV)
        wsb = lib().hy_attn_decode_workspace_bytes(n, nh, d, ctx)
        ws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=DEV)

        def ours(i):
            rc = lib().hy_attn_decode_paged(q.data_ptr(), nh * d, n, nh, nkv, d, slots.data_ptr(),
                                            ctxs.data_ptr(), ctx, bt.data_ptr(), nb, kv.data_ptr(),
                                            be, 1 / math.sqrt(d), o.data_ptr(), nh * d,
                                            ws.data_ptr(), ws.numel(), st())
            assert rc == 0, lib().hy_last_error()
        t = timeit(ours)
        byt = int(cl.sum()) * 2 * nkv * d * 2
        r = {"name": "decode_attn", "n_heads": nh, "n_kv": nkv, "seqs": n, "ctx": ctx,
             "shuffled_blocks": bool(shuffled), "us": t * 1e3, "gbs": byt / t / 1e6}
        out.append(r)
        print(f"decode_attn heads {nh}/{nkv} seqs {n} ctx {ctx}{' shuffled' if shuffled else ''}: {t*1e3:8.1f} us "
              f"{r['gbs']:7.0f} GB/s", flush=True)
        del kv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="gemm")
    ap.add_argument("--json", default=None)
    ap.add_argument("--variants", default="",
                    help="';'-separated env settings, e.g. 'HY_GEMM_NOSK=1;HY_GEMM_BN=128'")
    ap.add_argument("--only", default="", help="comma list of shape names")
    ap.add_argument("--residual", default="", help="shape names run with an in-place residual "
                    "epilogue ('all' for every shape)")
    ap.add_argument("--shapes", default="", help="extra MxNxK list, e.g. 128x128x64,577x1024x1024")
    args = ap.parse_args()
    for v in filter(None, args.variants.split(";")):
        VARIANTS.append(dict(kv.split("=") for kv in v.split(",")))
    ONLY.extend(filter(None, args.only.split(",")))
    RESIDUAL.extend(filter(None, args.residual.split(",")))
    for x in filter(None, args.shapes.split(",")):
        M, N, K = (int(v) for v in x.split("x"))
        EXTRA.append(("custom", M, N, K))
    res = {}
    if "gemm" in args.what:
        res["gemm"] = []
        gemm_sweep(res["gemm"])
    if "attn" in args.what:
        res["attn"] = []
        attn_sweep(res["attn"])
    if "decode" in args.what:
        res["decode"] = []
        decode_sweep(res["decode"])
    if "overlap" in args.what:
        res["overlap"] = []
        overlap_probe(res["overlap"])
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
