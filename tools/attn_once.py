"""One paged prefill attention call (LLaVA 32 heads x 128, one 2304-token chunk), for ncu."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

lib = _lib.load()
nh, d, c = 32, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 2304
nb = -(-c // 16)
be = 2 * nh * 16 * d
kv = torch.randn(nb + 1, be, device="cuda").bfloat16()
bt = torch.arange(nb, dtype=torch.int32, device="cuda").view(1, nb)
q = torch.randn(c, nh * d, device="cuda").bfloat16()
o = torch.empty_like(q)
qs = torch.tensor([0, c], dtype=torch.int32, device="cuda")
offs = torch.zeros(1, dtype=torch.int32, device="cuda")
slots = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    rc = lib.hy_attn_prefill_paged(q.data_ptr(), nh * d, c, 1, qs.data_ptr(), offs.data_ptr(),
                                   slots.data_ptr(), c, nh, nh, d, bt.data_ptr(), nb, kv.data_ptr(),
                                   be, 1 / math.sqrt(d), o.data_ptr(), nh * d,
                                   torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.hy_last_error()
torch.cuda.synchronize()
print("ok")
