"""Run one hy_gemm_bf16 shape a few times (for ncu captures).
    python tools/gemm_once.py M N K [reps] [mode]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_12658_b200 import _lib  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
mode = int(sys.argv[5]) if len(sys.argv) > 5 else 0
lib = _lib.load()
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
e = _lib.HyGemmEpilogue(0, 0, 0, 0, 0, C.data_ptr(), N, 0)
for _ in range(reps):
    rc = lib.hy_gemm_bf16_mode(A.data_ptr(), K, W.data_ptr(), K, M, N, K, e, ws.data_ptr(),
                               ws.numel(), mode, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.hy_last_error()
torch.cuda.synchronize()
ref = A.float() @ W.float().t()
print("max err", (C.float() - ref).abs().max().item())
