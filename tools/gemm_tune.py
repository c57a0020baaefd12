"""Measured GEMM dispatch table for the served models (writes csrc/gemm_table.inc).

    python tools/gemm_tune.py [--models llava-1.5-7b,qwen2-vl-7b] [--out PATH] [--quick]

For every (N, K) GEMM of the models (language tower, lm_head, ViT tower, projector, patch
embedding) and a grid of token counts M, times each kernel configuration the library has
-- swap-AB (tokens on MMA-N) at BN 32..256, single-CTA 128xBN tiles at BN 64/128/256, CTA
pairs at BN 128/256, each with and without stream-K -- with weights rotated through more
than L2 and CUDA-graph replay (no launch overhead), and keeps the fastest.  The table entry
for grid point M covers token counts in (previous point, M].  The chosen configuration,
its time, the heuristic's time and cuBLAS's time are written beside each entry.

Run on a B200 (gpurun); commit the generated table.  Never a bench number.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2505_12658_b200 import _lib, get_shape  # noqa: E402

DEV = "cuda:0"
LANG_M = [1, 8, 16, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 512, 576, 640,
          768, 896, 1024, 1152, 1280, 1408, 1536, 1792, 2048, 2304, 2560, 2816, 3072, 3328,
          3584, 4096]
HEAD_M = [1, 8, 16, 32, 64, 96, 128, 192, 256, 384, 512]


def model_gemms(name):
    s = get_shape(name)
    H, F = s.hidden, s.ffn
    out = [("qkv", s.qkv_cols, H, LANG_M), ("o", H, s.n_heads * s.head_dim, LANG_M),
           ("gate_up", 2 * F, H, LANG_M), ("down", H, F, LANG_M),
           ("lm_head", s.vocab, H, HEAD_M)]
    Hv = s.v_hidden
    if s.merge == 1:  # LLaVA: 577-token images
        vit_m = [577 * k for k in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32, 48, 64, 80)]
        proj_m = [576 * k for k in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32, 48, 64, 80)]
        pin = Hv
    else:  # Qwen2-VL: dynamic resolution, 2x2 merge
        vit_m = [256, 576, 1024, 1600, 2048, 2916, 4096, 5832, 8192, 11664, 16384, 23328]
        proj_m = [m // 4 for m in vit_m]
        pin = 4 * Hv
    out += [("vit_qkv", 3 * Hv, Hv, vit_m), ("vit_o", Hv, Hv, vit_m),
            ("vit_fc1", s.v_mlp, Hv, vit_m), ("vit_fc2", Hv, s.v_mlp, vit_m),
            ("patch", Hv, s.k_pad, vit_m),
            ("proj1", s.proj_hidden, pin, proj_m), ("proj2", H, s.proj_hidden, proj_m)]
    return out


def configs(M, N):
    """(label, mode, env, kind, bn, sk) candidates valid for this shape."""
    c = []
    if M <= 256:
        for bn in (32, 64, 128, 256):
            if bn >= 2 * max(M, 32) and bn > 32:
                continue  # more than half the token tile empty
            for sk in (0, 1):
                c.append((f"swap{bn}{'+sk' if sk else ''}", 1,
                          {"HY_GEMM_BN": str(bn), "HY_GEMM_SK" if sk else "HY_GEMM_NOSK": "1"},
                          1, bn, sk))
    if M >= 96:
        for bn in (64, 128, 256):
            if N % bn or N % 128:
                continue
            for sk in (0, 1):
                c.append((f"single{bn}{'+sk' if sk else ''}", 2,
                          {"HY_GEMM_BN": str(bn), "HY_GEMM_SK" if sk else "HY_GEMM_NOSK": "1"},
                          2, bn, sk))
    if M >= 192:
        for bn in (128, 256):
            if N % bn:
                continue
            for sk in (0, 1):
                env = {"HY_PAIR_BN": str(bn)}
                if sk:
                    env["HY_PAIR_SK"] = "1"
                c.append((f"pair{bn}{'+sk' if sk else ''}", 3, env, 3, bn, sk))
    return c


def timeit(fn, reps=5, per_graph=10, warm=2):
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
    return ts[len(ts) // 2] * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="llava-1.5-7b,qwen2-vl-7b")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "paper_2505_12658_b200", "csrc", "gemm_table.inc"))
    ap.add_argument("--quick", action="store_true", help="a few shapes only (smoke)")
    args = ap.parse_args()
    os.environ["HY_GEMM_NOTABLE"] = "1"  # the heuristic is the baseline being replaced
    lib = _lib.load()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=DEV)
    st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    seen = set()
    lines = ["// generated by tools/gemm_tune.py on a B200: {N, K, m_max, kind (1 swap, 2 single, "
             "3 pair), bn, stream-K}", "// M grid point: best config us | heuristic us | cuBLAS us"]
    gains = []
    for model in args.models.split(","):
        for name, N, K, grid in model_gemms(model):
            if (N, K) in seen:
                continue
            seen.add((N, K))
            if args.quick:
                grid = grid[::8]
            nw = max(2, int(400e6 // (N * K * 2)) + 1)  # weights rotate through > L2
            Ws = [torch.empty(N, K, device=DEV, dtype=torch.bfloat16).normal_(0, 0.02)
                  for _ in range(nw)]
            A = torch.randn(max(grid), K, device=DEV).bfloat16()
            C = torch.empty(max(grid), N, device=DEV, dtype=torch.float32)
            f32 = name == "lm_head"
            for M in grid:
                e = _lib.HyGemmEpilogue(0, 0, 0, 0, 0, C.data_ptr(), N, 1 if f32 else 0)

                def run(mode):
                    def f(i):
                        rc = lib.hy_gemm_bf16_mode(A.data_ptr(), K, Ws[i % nw].data_ptr(), K, M, N,
                                                   K, e, ws.data_ptr(), ws.numel(), mode, st())
                        assert rc == 0, lib.hy_last_error()
                    return f

                t_auto = timeit(run(0))
                best = None
                for label, mode, env, kind, bn, sk in configs(M, N):
                    old = {k: os.environ.get(k) for k in env}
                    os.environ.update(env)
                    try:
                        t = timeit(run(mode))
                    except AssertionError:
                        t = None
                    finally:
                        for k, v in old.items():
                            if v is None:
                                os.environ.pop(k, None)
                            else:
                                os.environ[k] = v
                    if t is not None and (best is None or t < best[0]):
                        best = (t, label, kind, bn, sk)
                Av = A[:M]
                Cb = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)  # (bf16 out for lm_head too)
                t_cb = timeit(lambda i: torch.matmul(Av, Ws[i % nw].t(), out=Cb))
                if best is None or best[0] > t_auto * 0.98:  # keep the heuristic unless it loses
                    best = (t_auto, "auto", 0, 0, 0)
                gains.append((name, M, N, K, t_auto, best[0], t_cb))
                print(f"{model:12s} {name:8s} M={M:6d} N={N:6d} K={K:6d}  best {best[1]:12s} "
                      f"{best[0]:8.1f} us | auto {t_auto:8.1f} | cublas {t_cb:8.1f} "
                      f"| x{t_cb / best[0]:.2f} of cuBLAS", flush=True)
                if best[2]:
                    lines.append(f"    {{{N}, {K}, {M}, {best[2]}, {best[3]}, {best[4]}}},  "
                                 f"// {name} M={M}: {best[1]} {best[0]:.1f} | {t_auto:.1f} | "
                                 f"{t_cb:.1f}")
                else:  # heuristic kept: an entry that defers to it (kind 0)
                    lines.append(f"    {{{N}, {K}, {M}, 0, 0, 0}},  // {name} M={M}: auto "
                                 f"{t_auto:.1f} | cuBLAS {t_cb:.1f}")
            del Ws, A, C
            torch.cuda.empty_cache()
    with open(args.out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tot_auto = sum(g[4] for g in gains)
    tot_best = sum(g[5] for g in gains)
    print(f"wrote {args.out}: {len(lines) - 2} entries; sum over the grid: heuristic "
          f"{tot_auto:.0f} us -> table {tot_best:.0f} us")


if __name__ == "__main__":
    main()
