"""One paged decode-attention call (for ncu): python tools/decode_once.py n_heads n_kv seqs ctx"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

nh, nkv, n, ctx = (int(x) for x in sys.argv[1:5])
lib = _lib.load()
if os.environ.get("HY_CO"):  # co-resident kernel (K8c)
    lib.hy_set_decode_coresident(1)
d = 128
nb = -(-ctx // 16)
be = 2 * nkv * 16 * d
kv = torch.randn(n * nb + 1, be, device="cuda").bfloat16()
bt = torch.arange(n * nb, dtype=torch.int32, device="cuda").view(n, nb).contiguous()
q = torch.randn(n, nh * d, device="cuda").bfloat16()
o = torch.empty_like(q)
slots = torch.arange(n, dtype=torch.int32, device="cuda")
ctxs = torch.full((n,), ctx, dtype=torch.int32, device="cuda")
ws = torch.zeros(max(lib.hy_attn_decode_workspace_bytes(n, nh, d, ctx), 16), dtype=torch.uint8,
                 device="cuda")
for _ in range(3):
    rc = lib.hy_attn_decode_paged(q.data_ptr(), nh * d, n, nh, nkv, d, slots.data_ptr(),
                                  ctxs.data_ptr(), ctx, bt.data_ptr(), nb, kv.data_ptr(), be,
                                  1 / math.sqrt(d), o.data_ptr(), nh * d, ws.data_ptr(), ws.numel(),
                                  torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.hy_last_error()
torch.cuda.synchronize()
print("ok", n * ctx * 2 * nkv * d * 2 / 1e6, "MB of K+V")
