"""One launch (after warm-up) of a single kernel at a serving shape, for ncu captures.

    python tools/one_kernel.py vit_attn N_IMAGES        # attn_tc_kernel<64, varlen>, LLaVA ViT
    python tools/one_kernel.py qwen_vit_attn N_TOKENS   # attn_tc_kernel<128(80), varlen>, Qwen ViT
    python tools/one_kernel.py copy N_BLOCKS            # copy_blocks_kernel, 8 MiB KV blocks
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

lib = _lib.load()
what, n = sys.argv[1], int(sys.argv[2])
st = torch.cuda.current_stream().cuda_stream


def ck(rc):
    assert rc == 0, lib.hy_last_error()


if what in ("vit_attn", "qwen_vit_attn"):
    nh, d = (16, 64) if what == "vit_attn" else (16, 80)
    lens = [577] * n if what == "vit_attn" else [n]
    T = sum(lens)
    qkv = torch.randn(T, 3 * nh * d, device="cuda").bfloat16()
    out = torch.empty(T, nh * d, device="cuda", dtype=torch.bfloat16)
    seg = torch.tensor(np.cumsum([0] + lens), dtype=torch.int32, device="cuda")
    for _ in range(3):
        ck(lib.hy_attn_varlen(qkv.data_ptr(), 3 * nh * d, T, len(lens), seg.data_ptr(),
                              max(lens), nh, d, 1 / math.sqrt(d), out.data_ptr(), nh * d, st))
elif what == "copy":
    bb = 8 << 20
    src = torch.empty(n * bb, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    rng = np.random.default_rng(0)
    sid = torch.from_numpy(rng.permutation(n).astype(np.int32)).cuda()
    did = torch.from_numpy(rng.permutation(n).astype(np.int32)).cuda()
    for _ in range(3):
        ck(lib.hy_copy_blocks_tail(src.data_ptr(), dst.data_ptr(), sid.data_ptr(), did.data_ptr(),
                                   n, bb, 4096, 7 * 256, st))
else:
    raise SystemExit(f"unknown kernel {what}")
torch.cuda.synchronize()
print("ok")
