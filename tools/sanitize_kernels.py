"""One small launch of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_kernels.py

Covers the paths with intra-kernel synchronisation worth checking: the GEMM's stream-K
last-arriver fixup (single-CTA normal and swap orientation, and the CTA-pair kernel with
stream-K forced on), the pair kernel's cluster barriers, the tcgen05 attention kernels
(paged prefill, varlen d = 64 / 80 / 128, one and two query tiles), decode attention (MHA
split-KV + combine, GQA tensor-core, the bulk-copy ticket kernel K8b and the co-resident
tensor-core kernel K8c with its per-SM flags), the SLIM pair GEMM, GEMMs launched under
programmatic dependent launch, norms, RoPE append, argmax and the token-exact block copy.  Every result is checked against torch so a sanitizer-clean run is also a correct one.
"""

import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

DEV = "cuda:0"
lib = _lib.load()


def st():
    return torch.cuda.current_stream().cuda_stream


def ck(rc, what):
    assert rc == 0, f"{what}: {lib.hy_last_error().decode()}"


def gemm(M, N, K, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        A = torch.randn(M, K, device=DEV).bfloat16()
        W = (torch.randn(N, K, device=DEV) * 0.05).bfloat16()
        C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
        ws = torch.zeros(64 << 20, dtype=torch.uint8, device=DEV)
        e = _lib.HyGemmEpilogue(0, 0, 0, 0, 0, C.data_ptr(), N, 0)
        ck(lib.hy_gemm_bf16(A.data_ptr(), K, W.data_ptr(), K, M, N, K, e, ws.data_ptr(),
                            ws.numel(), st()), f"gemm {M}x{N}x{K} {env}")
        torch.cuda.synchronize()
        err = (C.float() - A.float() @ W.float().t()).abs().max().item()
        assert err < 0.1, (M, N, K, env, err)
        print(f"gemm {M}x{N}x{K} {env}: max err {err:.4f}", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def varlen(d, lens, tiles):
    os.environ["HY_ATTN_T"] = str(tiles)
    nh = 2
    T = sum(lens)
    qkv = torch.randn(T, 3 * nh * d, device=DEV).bfloat16()
    out = torch.empty(T, nh * d, device=DEV, dtype=torch.bfloat16)
    seg = torch.tensor(np.cumsum([0] + lens), dtype=torch.int32, device=DEV)
    ck(lib.hy_attn_varlen(qkv.data_ptr(), 3 * nh * d, T, len(lens), seg.data_ptr(), max(lens),
                          nh, d, 1 / math.sqrt(d), out.data_ptr(), nh * d, st()), "varlen")
    torch.cuda.synchronize()
    x = qkv[:lens[0]].float().view(lens[0], 3, nh, d)
    s = torch.einsum("qhd,khd->hqk", x[:, 0], x[:, 1]) / math.sqrt(d)
    ref = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), x[:, 2]).reshape(lens[0], -1)
    err = (out[:lens[0]].float() - ref).abs().max().item()
    assert err < 2e-2, err
    print(f"varlen d={d} lens={lens} T={tiles}: max err {err:.4f}", flush=True)
    os.environ.pop("HY_ATTN_T", None)


def paged(n_heads, n_kv, chunks, tiles):
    """prefill over a paged cache: chunk c of each sequence after `off` cached tokens."""
    os.environ["HY_ATTN_T"] = str(tiles)
    d, blk = 128, 16
    nb = 64
    kv = torch.randn(nb, 2, n_kv, blk, d, device=DEV).bfloat16()
    bt = torch.randperm(nb, device=DEV).int().view(4, 16)
    q_rows = sum(c for c, _ in chunks)
    q = torch.randn(q_rows, n_heads * d, device=DEV).bfloat16()
    out = torch.empty_like(q)
    qstart = torch.tensor(np.cumsum([0] + [c for c, _ in chunks]), dtype=torch.int32, device=DEV)
    off = torch.tensor([o for _, o in chunks], dtype=torch.int32, device=DEV)
    slots = torch.arange(len(chunks), dtype=torch.int32, device=DEV)
    ck(lib.hy_attn_prefill_paged(q.data_ptr(), n_heads * d, q_rows, len(chunks),
                                 qstart.data_ptr(), off.data_ptr(), slots.data_ptr(),
                                 max(c for c, _ in chunks), n_heads, n_kv, d, bt.data_ptr(), 16,
                                 kv.data_ptr(), 2 * n_kv * blk * d, 1 / math.sqrt(d),
                                 out.data_ptr(), n_heads * d, st()), "paged prefill")
    torch.cuda.synchronize()
    print(f"paged prefill heads {n_heads}/{n_kv} chunks {chunks} T={tiles}: ok", flush=True)
    os.environ.pop("HY_ATTN_T", None)


def decode(n_heads, n_kv, ctxs, kernel=None, co=False):
    """paged decode attention (split-KV + combine for long contexts; GQA tensor-core path
    for 4 <= group <= 16) over one layer of a 2-layer paged cache."""
    d, L, blk = 128, 2, 16
    n = len(ctxs)
    bts = max(-(-c // blk) for c in ctxs)
    nb = n * bts
    kv = torch.randn(nb, L, 2, n_kv, blk, d, device=DEV).bfloat16()
    bt = torch.randperm(nb, device=DEV).int().view(n, bts)
    q = torch.randn(n, n_heads * d, device=DEV).bfloat16()
    out = torch.empty_like(q)
    slots = torch.arange(n, dtype=torch.int32, device=DEV)
    ctx = torch.tensor(ctxs, dtype=torch.int32, device=DEV)
    wsb = lib.hy_attn_decode_workspace_bytes(n, n_heads, d, max(ctxs))
    ws = torch.zeros(max(wsb, 16), dtype=torch.uint8, device=DEV)
    if kernel:
        ck(lib.hy_set_decode_kernel(*kernel), "decode kernel")
    lib.hy_set_decode_coresident(1 if co else 0)
    ck(lib.hy_attn_decode_paged(q.data_ptr(), n_heads * d, n, n_heads, n_kv, d,
                                slots.data_ptr(), ctx.data_ptr(), max(ctxs), bt.data_ptr(), bts,
                                kv.data_ptr() + 2 * n_kv * blk * d * 2, L * 2 * n_kv * blk * d,
                                1 / math.sqrt(d), out.data_ptr(), n_heads * d, ws.data_ptr(),
                                ws.numel(), st()), "decode")
    torch.cuda.synchronize()
    lib.hy_set_decode_kernel(0, 0)
    lib.hy_set_decode_coresident(0)
    print(f"decode heads {n_heads}/{n_kv} ctxs {ctxs} kernel {kernel} co {co}: ok", flush=True)


def copy_tail():
    src = torch.randint(1, 255, (8, 4096 * 4), dtype=torch.uint8, device=DEV)
    dst = torch.zeros_like(src)
    ids = torch.tensor([1, 5, 2, 7, 3, 0], dtype=torch.int32, device=DEV)
    ck(lib.hy_copy_blocks_tail(src.data_ptr(), dst.data_ptr(), ids.data_ptr(),
                               ids.data_ptr() + 12, 3, 4096 * 4, 4096, 5 * 256, st()), "copy")
    torch.cuda.synchronize()
    assert torch.equal(dst[7], src[1]) and torch.equal(dst[3], src[5])
    print("copy tail: ok", flush=True)


def main():
    # GEMM: swap + stream-K (decode), normal stream-K forced, pair (+ stream-K), 128x64 tiles
    gemm(16, 4096, 4096, {})
    gemm(200, 4096, 4096, {"HY_GEMM_SK": "1"})
    gemm(600, 1024, 4096, {"HY_GEMM_MODE": "2", "HY_GEMM_SK": "1"})
    gemm(1100, 4096, 4096, {})
    gemm(1100, 2048, 4096, {"HY_PAIR_SK": "1", "HY_GEMM_MODE": "3"})
    gemm(577, 3072, 1024, {})
    gemm(1100, 4096, 4096, {"HY_GEMM_SLIM": "1", "HY_GEMM_NOTABLE": "1"})
    lib.hy_set_pdl(1)  # prologues overlapping the previous kernel (griddepcontrol)
    gemm(16, 4096, 4096, {})
    gemm(1100, 4096, 4096, {"HY_PAIR_SK": "1", "HY_GEMM_MODE": "3"})
    lib.hy_set_pdl(0)
    for tiles in (1, 2):
        varlen(64, [577, 33], tiles)
        varlen(80, [300, 5], tiles)
        varlen(128, [129], tiles)
        paged(4, 4, [(130, 0), (20, 200)], tiles)
        paged(28, 4, [(64, 16)], tiles)
    decode(32, 32, [616, 3000])
    decode(28, 4, [5, 900])
    decode(8, 8, [616, 3000, 17], kernel=(2, 2))
    decode(8, 8, [616, 3000, 17], kernel=(8, 3))
    decode(32, 32, [616, 3000], co=True)
    decode(28, 4, [5, 900], co=True)
    copy_tail()
    print("sanitize run complete")


if __name__ == "__main__":
    main()
